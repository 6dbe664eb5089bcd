/*
 * sig.h -- C ABI of libsig.so, the B200 (sm_100a) hot path of Signatory (arXiv 2001.00706):
 * batched truncated signature / logsignature transforms of piecewise-linear paths, their
 * handwritten reversible backward passes, and the group-like product.
 *
 * Citations "P:Lnnn" are lines of the paper's LaTeX source (reference PAPER.md).
 *
 * Conventions for every call
 *  - Tensors are DEVICE pointers to contiguous, row-major float32 arrays, owned by the caller
 *    (allocated through PyTorch in the Python binding).  The library never allocates device
 *    memory on these calls and writes only to the output / gradient / workspace arguments.
 *  - Every call is asynchronous on the given CUDA stream (cudaStream_t, may be NULL = legacy
 *    default stream).  Errors in the arguments are detected on the host BEFORE anything is
 *    launched and reported as SIG_ERR_INVALID_ARG / SIG_ERR_SHAPE; a (C, depth) pair for which
 *    no kernel is compiled returns SIG_ERR_UNSUPPORTED (there is no CPU fallback); a failed
 *    launch returns SIG_ERR_CUDA.  NaN/Inf inputs are not checked and propagate.  A detail
 *    string for the last error of the calling thread is available from sig_last_error().
 *  - Truncated tensor layout: levels k = 1..depth back to back; inside
 *    level k the word (j_1..j_k) (0-based channel letters) is at offset sum_m j_m C^(k-m).
 *    The scalar level 0 is not stored: it is 1 for signatures, 0 for logsignatures.
 *    S = sig_signature_channels(C, depth) = sum_{k=1}^{depth} C^k floats per path.
 *  - Paths are [B, L, C]: B streams of L points in R^C.  The path is the
 *    piecewise-linear interpolation of its points; increments z_t = x_{t+1} - x_t.
 *  - basepoint (reading R4): SIG_BP_NONE uses the points as given;
 *    SIG_BP_ZERO prepends the origin; SIG_BP_GIVEN prepends basepoint[b] ([B, C] device array).
 *    With a basepoint the stream has L+1 points (so L >= 1 suffices); without, L >= 2.
 *    M = L - 1 (+1 with a basepoint) is the number of increments.
 *  - stream: 0 returns Sig of the whole path, [B, S]; 1 returns every expanding
 *    prefix Sig(x_1..x_{j+1}), j = 1..M, as [B, M, S].
 *  - Results are deterministic: every reduction has a fixed order.
 */
#ifndef SIG_B200_H
#define SIG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* sig_cuda_stream_t; /* identical to cudaStream_t */

typedef enum {
    SIG_OK = 0,
    SIG_ERR_INVALID_ARG = 1, /* null pointer, C < 1, depth < 1, bad enum */
    SIG_ERR_SHAPE = 2,       /* too few points, sizes overflow int64, workspace too small */
    SIG_ERR_UNSUPPORTED = 3, /* no sm_100a kernel instantiated for (C, depth) or path too long */
    SIG_ERR_CUDA = 4,        /* a CUDA launch or runtime call failed */
    SIG_ERR_WORKSPACE = 5    /* ws_bytes smaller than the size the *_workspace_size query gave */
} sig_status_t;

typedef enum { SIG_BP_NONE = 0, SIG_BP_ZERO = 1, SIG_BP_GIVEN = 2 } sig_basepoint_t;

/* Logsignature bases (Appendix A.2):
 *  EXPAND   -- log Sig itself in the tensor basis, S floats.
 *  BRACKETS -- coefficients alpha_l of the Lyndon basis phi(l): sum_l alpha_l phi(l) = log Sig
 *              (eq-linearsystem), w(C, depth) floats.
 *  WORDS    -- the paper's new basis z = psi(log Sig): the coefficients of the Lyndon words
 *              (P:L561-575), w(C, depth) floats.  Lyndon words are ordered by (length, lex).   */
typedef enum { SIG_LOGSIG_EXPAND = 0, SIG_LOGSIG_BRACKETS = 1, SIG_LOGSIG_WORDS = 2 } sig_logsig_mode_t;

/* ---------------------------------------------------------------- sizes and diagnostics */

/* S = sum_{k=1}^{depth} C^k; -1 if C < 1, depth < 1 or the sum overflows int64. */
int64_t sig_signature_channels(int64_t C, int32_t depth);

/* Output width of the logsignature: S for EXPAND, Witt's formula w(C, depth) for
 * BRACKETS and WORDS; -1 on invalid arguments. */
int64_t sig_logsignature_channels(int64_t C, int32_t depth, sig_logsig_mode_t mode);

/* 1 if sm_100a kernels exist for (C, depth) -- forward (backward = 0) or backward (backward = 1);
 * 0 otherwise. */
int32_t sig_is_supported(int64_t C, int32_t depth, int32_t backward);

/* Number of CUDA kernels this library has launched in this process (all devices and threads) --
 * a diagnostic used by the benchmark to report how many of its own kernels ran. */
uint64_t sig_launch_count(void);

const char* sig_status_string(sig_status_t status);
/* Detail of the last failed call on this host thread ("" if none).  Valid until the next call. */
const char* sig_last_error(void);

/* ---------------------------------------------------------------- signature (K1 + K3) */

/* Bytes of device workspace sig_signature needs for this problem (0 when the whole path of every
 * stream is scanned by one unit; > 0 when long paths are split into time chunks whose
 * signatures are then folded in order with Chen's identity). */
size_t sig_signature_workspace_size(int64_t B, int64_t L, int64_t C, int32_t depth, int32_t stream,
                                    sig_basepoint_t bp);

/* Forward signature by the fused multiply-exponentiate scan (eq-fusedterm).
 *   path      [B, L, C]
 *   basepoint [B, C] if bp == SIG_BP_GIVEN, else ignored (may be NULL)
 *   out       [B, S] (stream = 0) or [B, M, S] (stream = 1); fully overwritten
 *   ws        device workspace of at least sig_signature_workspace_size(...) bytes (NULL if 0) */
sig_status_t sig_signature(const float* path, int64_t B, int64_t L, int64_t C, int32_t depth, int32_t stream,
                           sig_basepoint_t bp, const float* basepoint, float* out, void* ws, size_t ws_bytes,
                           sig_cuda_stream_t s);

/* Reversible backward (Appendix C): gradients of <grad_out, Sig(path)>.
 *   grad_out       [B, S] or [B, M, S] (stream), the upstream gradient
 *   out_saved      the forward's `out` for the same arguments (its final signature seeds the
 *                  reversal eq-reverse); consistency with `path` is NOT checked
 *   grad_path      [B, L, C], overwritten
 *   grad_basepoint [B, C] (bp == SIG_BP_GIVEN) or NULL; overwritten when given
 * One CTA reverses one path, staging its increments in shared memory tile by tile, so any path
 * length works here (no workspace, no time chunks).  Small batches and long paths run faster
 * through sig_signature_backward_ex with sig_signature_backward_ex_workspace_size(...) bytes of
 * workspace: the path is then split into time chunks reversed in parallel. */
sig_status_t sig_signature_backward(const float* grad_out, const float* path, const float* out_saved, int64_t B,
                                    int64_t L, int64_t C, int32_t depth, int32_t stream, sig_basepoint_t bp,
                                    const float* basepoint, float* grad_path, float* grad_basepoint,
                                    sig_cuda_stream_t s);

/* ---------------------------------------------------------------- forward with saved chunk states */

/* The time-parallel backward (sig_signature_backward_ex with workspace; Chen's
 * identity P:L84-87 over time chunks) starts chunk j's reversal (eq-reverse)
 * from the product of the chunks before it and needs the products after it for the chunk-end
 * gradients; without saved state it recomputes every chunk's signature (one forward pass over the
 * whole path) first.  This pair keeps them instead: sig_signature_save computes the chunk
 * signatures S_j and their inclusive prefix products P_{j+1} = S_0 [x] .. [x] S_j (the signature
 * is the last one, copied to `out`), and sig_signature_backward_saved reverses every chunk in
 * parallel from them.  Plain calls only (no stream, inverse or initial).  When the batch fills the
 * GPU without chunks (sig_signature_saved_bytes(...) == 0) both are the plain forward / reversal.
 *   saved  device buffer of sig_signature_saved_bytes(...) bytes: [2][B, m, S] floats, m chunks;
 *          written by sig_signature_save, read by sig_signature_backward_saved for the SAME path,
 *          B, L, C, depth and basepoint (not checked); owned by the caller
 *   ws     sig_signature_save_workspace_size(...) resp. sig_signature_backward_saved_workspace_size
 *          bytes (scan scratch; suffix products, chunk-end gradients and the shared-point buffer)
 * Errors: as sig_signature / sig_signature_backward; WORKSPACE when saved or ws is too small. */
size_t sig_signature_saved_bytes(int64_t B, int64_t L, int64_t C, int32_t depth, sig_basepoint_t bp);
size_t sig_signature_save_workspace_size(int64_t B, int64_t L, int64_t C, int32_t depth, sig_basepoint_t bp);
sig_status_t sig_signature_save(const float* path, int64_t B, int64_t L, int64_t C, int32_t depth, sig_basepoint_t bp,
                                const float* basepoint, float* out, float* saved, size_t saved_bytes, void* ws,
                                size_t ws_bytes, sig_cuda_stream_t s);
size_t sig_signature_backward_saved_workspace_size(int64_t B, int64_t L, int64_t C, int32_t depth,
                                                   sig_basepoint_t bp);
sig_status_t sig_signature_backward_saved(const float* grad_out, const float* path, const float* out_saved,
                                          const float* saved, size_t saved_bytes, int64_t B, int64_t L, int64_t C,
                                          int32_t depth, sig_basepoint_t bp, const float* basepoint, float* grad_path,
                                          float* grad_basepoint, void* ws, size_t ws_bytes, sig_cuda_stream_t s);

/* ---------------------------------------------------------------- host-resident batches */

/* Signature forward + reversible backward of a batch that lives in HOST memory (the training step
 * of BASELINE config c2 fed from the host): the batch is cut into `chunks` slices; per slice the
 * host->device copies of path and grad_out run on an internal copy stream, the forward and
 * backward kernels (sig_signature, sig_signature_backward) on `s` once the slice has arrived, and
 * the device->host copy of its grad_path on a second internal stream -- so copies of one slice
 * overlap the kernels of another.  Work on `s` issued before the call is ordered before the copies,
 * and `s` waits for the last read-back, so the host results are valid once `s` completes.
 *   path_h       [B, L, C] host, read   (pinned memory for the copies to overlap)
 *   grad_out_h   [B, S] host, read      (the upstream gradient of the final signature)
 *   grad_path_h  [B, L, C] host, written
 *   ws           device workspace of sig_signature_fwd_bwd_host_workspace_size(...) bytes (holds the
 *                device copies of the inputs, the signatures, the gradients; caller-owned)
 * No basepoint, no stream mode; each path must fit the plain backward (see sig_signature_backward).
 * Returns the first failing call's status. */
size_t sig_signature_fwd_bwd_host_workspace_size(int64_t B, int64_t L, int64_t C, int32_t depth, int32_t chunks);
sig_status_t sig_signature_fwd_bwd_host(const float* path_h, const float* grad_out_h, int64_t B, int64_t L, int64_t C,
                                        int32_t depth, float* grad_path_h, int32_t chunks, void* ws, size_t ws_bytes,
                                        sig_cuda_stream_t s);

/* ---------------------------------------------------------------- signature options */

/* The `inverse` and `initial` options (reading R18).
 *   inverse = 0: out = I [x] Sig(x)              (I = initial, or the identity when NULL)
 *   inverse = 1: out = Sig(x)^{-1} [x] I, where Sig(x)^{-1} = Sig(x reversed); with
 *                stream = 1, row t is the inverse of the prefix signature, [x] I.
 * `initial` [B, S] (device) is the signature of the data seen before (inverse = 0), or its inverse
 * (inverse = 1) -- the update case of P:L252-258: feed the new points with basepoint = the last
 * old point.  Any [B, S] tensor is accepted; it is not checked to be group-like.
 * Everything else as sig_signature.  Implementation: inverse scans the negated path from
 * alpha(I) and reverses the words of the output (alpha = word reversal); it needs
 * sig_signature_ex_workspace_size(...) bytes of workspace (B * S floats more than the plain
 * scan when initial is given). */
size_t sig_signature_ex_workspace_size(int64_t B, int64_t L, int64_t C, int32_t depth, int32_t stream,
                                       sig_basepoint_t bp, int32_t inverse, int32_t has_initial);
sig_status_t sig_signature_ex(const float* path, int64_t B, int64_t L, int64_t C, int32_t depth, int32_t stream,
                              sig_basepoint_t bp, const float* basepoint, int32_t inverse, const float* initial,
                              float* out, void* ws, size_t ws_bytes, sig_cuda_stream_t s);

/* Backward of sig_signature_ex (reversible, as sig_signature_backward).
 *   grad_initial [B, S] or NULL: overwritten with the gradient w.r.t. `initial` (the scan's start
 *                state) when given
 *   ws           sig_signature_backward_ex_workspace_size(...) bytes: for inverse = 1 the alpha
 *                images of grad_out, the final state, initial and grad_initial ((rows + up to 3 B)
 *                * S floats, rows = B or B*M); then, when the batch alone cannot fill the GPU
 *                (fewer paths than one resident wave of the backward), the time-chunk buffers
 *                (5 B m S + B m C floats for m chunks).  With a smaller ws (or NULL) the call runs
 *                without time chunks.
 * Errors as sig_signature_backward; WORKSPACE when ws is too small. */
size_t sig_signature_backward_ex_workspace_size(int64_t B, int64_t L, int64_t C, int32_t depth, int32_t stream,
                                                sig_basepoint_t bp, int32_t inverse, int32_t has_initial,
                                                int32_t want_grad_initial);
sig_status_t sig_signature_backward_ex(const float* grad_out, const float* path, const float* out_saved, int64_t B,
                                       int64_t L, int64_t C, int32_t depth, int32_t stream, sig_basepoint_t bp,
                                       const float* basepoint, int32_t inverse, const float* initial,
                                       float* grad_path, float* grad_basepoint, float* grad_initial, void* ws,
                                       size_t ws_bytes, sig_cuda_stream_t s);

/* ---------------------------------------------------------------- combine (K3) */

/* out[b] = a[b] [x] b[b] for b < B; all [B, S]. out must not alias a or b.  Any B >= 0
 * (the batch is grid-strided; no 65535 limit). */
sig_status_t sig_signature_combine(const float* a, const float* b, int64_t B, int64_t C, int32_t depth, float* out,
                                   sig_cuda_stream_t s);

/* VJP of sig_signature_combine: grad_a, grad_b [B, S] overwritten (either may be NULL). */
sig_status_t sig_signature_combine_backward(const float* grad_out, const float* a, const float* b, int64_t B,
                                            int64_t C, int32_t depth, float* grad_a, float* grad_b,
                                            sig_cuda_stream_t s);

size_t sig_multi_signature_combine_workspace_size(int64_t n, int64_t B, int64_t C, int32_t depth);

/* out[b] = sigs[0, b] [x] sigs[1, b] [x] ... [x] sigs[n-1, b]   (sigs [n, B, S] in time order;
 * an ordered tree).  n >= 1. */
sig_status_t sig_multi_signature_combine(const float* sigs, int64_t n, int64_t B, int64_t C, int32_t depth,
                                         float* out, void* ws, size_t ws_bytes, sig_cuda_stream_t s);

/* ---------------------------------------------------------------- logsignature (K4/K5) */

/* Immutable per-(C, depth, mode) tables (Lyndon words, flat indices, exact integer inverse of
 * psi o phi for BRACKETS), uploaded to the current device at creation.  A plan may be shared by
 * threads; destroy it after the last call that uses it has completed on the device.
 * SIG_ERR_UNSUPPORTED when one row of the log does not fit one CTA's shared memory: of the
 * instantiated (C, depth), (3, 9), (3, 10), (4, 8), (5, 7), (6, 6) and (7, 6), in every mode. */
typedef struct sig_logsig_plan_s* sig_logsig_plan_t;

sig_status_t sig_logsig_plan_create(int64_t C, int32_t depth, sig_logsig_mode_t mode, sig_logsig_plan_t* plan);
sig_status_t sig_logsig_plan_destroy(sig_logsig_plan_t plan);

/* Workspace for sig_logsignature / _backward: the signature scan's own workspace, the scratch rows of
 * the log and its VJP, and the reversible backward's time-chunk workspace (so long paths and small
 * batches take the time-parallel backward, as sig_signature_backward_ex does with its workspace). */
size_t sig_logsignature_workspace_size(sig_logsig_plan_t plan, int64_t B, int64_t L, int32_t stream,
                                       sig_basepoint_t bp);

/* LogSig = log(Sig(path)) in the plan's basis.
 *   out        [B, w] (WORDS, BRACKETS) or [B, S] (EXPAND); stream: [B, M, w|S]
 *   sig_saved  [B, S] | [B, M, S]: receives the signature (needed by the backward); may be NULL
 *              only if ws is large enough to hold it (then it is written to the workspace) */
sig_status_t sig_logsignature(sig_logsig_plan_t plan, const float* path, int64_t B, int64_t L, int32_t stream,
                              sig_basepoint_t bp, const float* basepoint, float* out, float* sig_saved, void* ws,
                              size_t ws_bytes, sig_cuda_stream_t s);

/* Backward of sig_logsignature: grad_out [B, w|S] (| stream [B, M, w|S]); sig_saved from the
 * forward; grad_path [B, L, C] and grad_basepoint [B, C] (or NULL) overwritten. */
sig_status_t sig_logsignature_backward(sig_logsig_plan_t plan, const float* grad_out, const float* path,
                                       const float* sig_saved, int64_t B, int64_t L, int32_t stream,
                                       sig_basepoint_t bp, const float* basepoint, float* grad_path,
                                       float* grad_basepoint, void* ws, size_t ws_bytes, sig_cuda_stream_t s);

/* ---------------------------------------------------------------- logsignature of given signatures */

/* K4 / K5 on signature rows already computed (e.g. Path queries, "followed by a log"):
 *   sig  [rows, S] group-like signatures; out [rows, w] (words / brackets) or [rows, S] (expand)
 *   grad_sig [rows, S] overwritten; ws >= sig_logsignature_from_signature_workspace_size bytes.
 * Errors as sig_logsignature. */
size_t sig_logsignature_from_signature_workspace_size(sig_logsig_plan_t plan, int64_t rows);
sig_status_t sig_logsignature_from_signature(sig_logsig_plan_t plan, const float* sig, int64_t rows, float* out,
                                             sig_cuda_stream_t s);
sig_status_t sig_logsignature_from_signature_backward(sig_logsig_plan_t plan, const float* grad_out, const float* sig,
                                                      int64_t rows, float* grad_sig, void* ws, size_t ws_bytes,
                                                      sig_cuda_stream_t s);

/* ---------------------------------------------------------------- Path: O(1) interval queries */

/* P:L171-185 (algorithmic-path): with the prefix signatures and prefix inverse signatures of a
 * stream precomputed (sig_signature / sig_signature_ex with stream = 1, inverse = 0 / 1: row r is
 * Sig(x_0 .. x_{r+1}) resp. its inverse, M = number of points - 1), the signature of any interval
 *     Sig(x_s, .., x_{e-1}) = InvertSig(x_0 .. x_s) [x] Sig(x_0 .. x_{e-1})
 * is one [x] per query, independent of its length.
 *   prefix_sig, prefix_inv [B, M, S] (device); starts, ends: Q HOST int64 arrays, 0 <= s,
 *   s + 2 <= e <= M + 1 (half-open point ranges of >= 2 points; with a basepoint the indices count
 *   the augmented points); out [B, Q, S] (device).  ws: sig_path_query_workspace_size(M, Q) bytes
 *   (device copies of the indices; the host arrays may be freed when the call returns).
 * Backward: grad_prefix_sig / grad_prefix_inv [B, M, S] overwritten with the sums, in ascending
 * query order (deterministic, no atomics), of the [x]-VJPs of the queries reading each row.
 * SHAPE for a query outside the stream (checked before any launch).  The paper's caution applies:
 * numerically unstable for long prefixes. */
size_t sig_path_query_workspace_size(int64_t M, int64_t Q);
sig_status_t sig_path_query(const float* prefix_sig, const float* prefix_inv, int64_t B, int64_t M, int64_t C,
                            int32_t depth, const int64_t* starts, const int64_t* ends, int64_t Q, float* out, void* ws,
                            size_t ws_bytes, sig_cuda_stream_t s);
sig_status_t sig_path_query_backward(const float* grad_out, const float* prefix_sig, const float* prefix_inv,
                                     int64_t B, int64_t M, int64_t C, int32_t depth, const int64_t* starts,
                                     const int64_t* ends, int64_t Q, float* grad_prefix_sig, float* grad_prefix_inv,
                                     void* ws, size_t ws_bytes, sig_cuda_stream_t s);

#ifdef __cplusplus
}
#endif
#endif /* SIG_B200_H */
