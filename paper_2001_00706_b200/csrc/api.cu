// api.cu -- the C ABI of libsig.so (include/sig.h): validation, kernel selection, launch plans.
// No compute happens here: every step of the path runs in the sm_100a kernels of K1-K5.
#include <atomic>
#include <cstdio>
#include <cstdarg>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/sig.h"
#define SIG_DEFINE_COMBINE_KERNELS
#define SIG_DEFINE_LOGSIG_KERNELS
#include "combine.cuh"
#include "logsig.cuh"
#include "logsig_owned.cuh"
#include "logsig_rows.cuh"
#include "lyndon.h"
#include "sig_bwd.cuh"
#include "sig_table.h"

using namespace sigb200;

namespace {

thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

sig_status_t fail(sig_status_t st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return st;
}

sig_status_t ok() {
    g_last_error.clear();
    return SIG_OK;
}

sig_status_t cuda_status(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return ok();
    return fail(SIG_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

int64_t sig_channels_checked(int64_t C, int32_t depth) {
    if (C < 1 || depth < 1) return -1;
    __int128 s = 0, p = 1;
    for (int k = 1; k <= depth; ++k) {
        p *= C;
        s += p;
        if (s > (__int128)INT64_MAX) return -1;
    }
    return (int64_t)s;
}

// ---------------------------------------------------------------- forward launch plan
constexpr int64_t kTargetThreads = 148LL * 1024;  // ~2 resident waves of 512-thread CTAs
constexpr int64_t kOneWave = 148LL * 512;          // one resident wave
constexpr int64_t kMinChunk = 64;                 // increments per time chunk, at least
constexpr int64_t kLatencyBoundWork = 1LL << 20;  // threads x steps below which a scan is latency-bound
#ifndef SIG_LATENCY_CHUNK
#define SIG_LATENCY_CHUNK 16
#endif
constexpr int64_t kLatencyChunk = SIG_LATENCY_CHUNK;  // steps per chunk, at least, in the one-CTA-per-path plan

struct FwdPlan {
    const KernelSet* ks;
    int P;
    FwdLaunch launch;
    int64_t M, n_chunks, chunk_len;
    int G;                  // group size of the chunk fold
    int upc;                // chunks folded inside each scan CTA (0: none)
    int64_t n_parts;        // partial signatures per path left for the fold kernels
    int64_t fold_levels[40];
    int n_fold;             // number of fold launches (after the scan)
    size_t ws_bytes;
};

#ifndef SIG_FWD_GROUP_THREADS
#define SIG_FWD_GROUP_THREADS 256
#endif
#ifndef SIG_FOLD_G
#define SIG_FOLD_G 8
#endif
int group_size_for(int64_t S, bool compiled) {
    if (compiled) {
        // compiled fold (fold_group_t_kernel, one barrier per tree level): each CTA's fold is
        // latency-bound (c5, 740 partials, 512 threads: G = 4, 8, 16 measured 432, 435, 444 us for
        // the whole signature; 1480 partials: G = 8 with 1024 threads 390 us against 400 for G = 4
        // with 512)
        int G = SIG_FOLD_G;
        while (G > 2 && (size_t)(G + (G + 1) / 2) * S * sizeof(float) > 200 * 1024) G >>= 1;
        if ((size_t)(G + (G + 1) / 2) * S * sizeof(float) <= 200 * 1024) return G;
        return 0;
    }
    // small groups: many CTAs, few loads per thread (the fold is latency-bound, not FLOP-bound)
    int G = 8;
    while (G > 2 && (size_t)G * S * sizeof(float) > 200 * 1024) G >>= 1;
    if ((size_t)G * S * sizeof(float) > 200 * 1024) return 0;  // pairwise in global memory
    return G;
}

void plan_fold(int64_t n, int64_t S, int64_t B, int& G, int64_t* lv, int& nl, size_t& elems, bool compiled) {
    // n elements per path -> ... -> 1; intermediate results go to the workspace (the last to out)
    G = group_size_for(S, compiled);
    const int g = G > 0 ? G : 2;
    nl = 0;
    elems = 0;
    while (n > 1) {
        n = (n + g - 1) / g;
        lv[nl++] = n;
        if (n > 1) elems += (size_t)n * B * S;
    }
}

sig_status_t make_fwd_plan(int64_t B, int64_t L, int64_t C, int32_t depth, int32_t stream, sig_basepoint_t bp,
                           FwdPlan& pl) {
    if (C < 1 || depth < 1) return fail(SIG_ERR_INVALID_ARG, "C=%lld depth=%d must be >= 1", (long long)C, depth);
    if (B < 0) return fail(SIG_ERR_SHAPE, "B=%lld < 0", (long long)B);
    if (bp != SIG_BP_NONE && bp != SIG_BP_ZERO && bp != SIG_BP_GIVEN)
        return fail(SIG_ERR_INVALID_ARG, "bad basepoint mode %d", (int)bp);
    const int64_t S = sig_channels_checked(C, depth);
    if (S < 0) return fail(SIG_ERR_SHAPE, "signature size overflows int64");
    const int64_t M = L - 1 + (bp != SIG_BP_NONE ? 1 : 0);
    if (M < 1)
        return fail(SIG_ERR_SHAPE, "a stream needs >= 2 points (P:L69); got L=%lld%s", (long long)L,
                    bp != SIG_BP_NONE ? " with a basepoint (L >= 1 needed)" : "");
    const KernelSet* ks = (C <= 8) ? find_kernels((int)C, depth) : nullptr;
    if (!ks) return fail(SIG_ERR_UNSUPPORTED, "no sm_100a kernel instantiated for C=%lld depth=%d", (long long)C, depth);
    pl.ks = ks;
    pl.M = M;
    pl.P = ks->pf0;
    pl.launch = ks->fwd0;
    const int64_t cp0 = sigb200::ipow(C, ks->pf0);
    pl.n_chunks = 1;
    // split long paths into time chunks only when the batch cannot fill one wave of the GPU
    // (the fold costs a launch and a pass over the chunk signatures)
    if (!stream && B > 0 && B * cp0 < kOneWave && M >= 2 * kMinChunk) {
        int64_t want = (kTargetThreads + B * cp0 - 1) / (B * cp0);
        int64_t maxc = M / kMinChunk;
        pl.n_chunks = want < maxc ? want : maxc;
    }
    if (pl.n_chunks == 1 && B * cp0 < kOneWave && ks->fwd1 && !(ks->fwd2 && !stream && B >= kFwd2MinBatch)) {
        pl.P = ks->pf1;
        pl.launch = ks->fwd1;
    }
    pl.upc = 0;
    // Latency-bound problems (a few short paths, e.g. BASELINE config c1): one CTA per path holds
    // K consecutive time chunks of it (the wider prefix variant), scans them concurrently and folds
    // them in order in shared memory -- the path's signature in one launch, with a critical path of
    // M/K steps plus log2(K) fold levels instead of M steps.
    if (!stream && B > 0 && B <= 148 && ks->fwd1 && B * cp0 * M < kLatencyBoundWork && M >= 16) {
        const int cp1 = (int)sigb200::ipow(C, ks->pf1);
        int K = cp1 <= 512 ? 512 / cp1 : 0;
        if (K > 32) K = 32;
        if ((int64_t)K > M / kLatencyChunk) K = (int)(M / kLatencyChunk);
        while (K >= 2 && (size_t)(K + (K + 1) / 2) * S * sizeof(float) > 200 * 1024) --K;
        if (K >= 2) {
            pl.P = ks->pf1;
            pl.launch = ks->fwd1;
            pl.upc = K;
            pl.n_chunks = K;
            pl.chunk_len = (M + K - 1) / K;
            pl.n_parts = 1;
            pl.n_fold = 0;
            pl.G = 0;
            pl.ws_bytes = 0;
            return ok();
        }
    }
    if (pl.n_chunks > 1) {
        // group chunks so that each scan CTA folds upc consecutive chunks of one path itself
        const int cp = (int)sigb200::ipow(C, pl.P);
        // ~256-thread CTAs: two or more resident per SM, so one CTA's staging and fold phases
        // overlap another's scan (c5: 9 chunks of 27 threads, 506 -> 474 us vs 18 per CTA)
        int upc = cp <= SIG_FWD_GROUP_THREADS ? SIG_FWD_GROUP_THREADS / cp : 0;
        if (upc > 32) upc = 32;
        while (upc >= 2 && (size_t)(upc + (upc + 1) / 2) * S * sizeof(float) > 200 * 1024) --upc;
        if (upc >= 2) {
            pl.upc = upc;
            // one CTA per group of upc chunks: make the CTA count a whole number of waves
            int64_t groups = (B * pl.n_chunks + upc - 1) / upc;
            groups = (groups + 147) / 148 * 148;
            int64_t per_path = (groups + B - 1) / B;
            // a CTA stages its chunks' points and increments at once (2 x upc x chunk x C floats):
            // keep that within ~110 KB so that two CTAs stay resident per SM (c5: 630-step chunks,
            // 137 KB, one CTA per SM, 446 us -> 315-step chunks, 68 KB, two per SM, 409 us)
            while (per_path * upc * 2 <= M / kMinChunk &&
                   (size_t)2 * upc * ((M + per_path * upc - 1) / (per_path * upc)) * C * sizeof(float) > 110 * 1024)
                per_path *= 2;
            if (per_path * upc > M) per_path = M / upc > 0 ? M / upc : 1;
            pl.n_chunks = per_path * upc;
        }
    }
    pl.chunk_len = (M + pl.n_chunks - 1) / pl.n_chunks;
    if (pl.upc == 0) pl.n_chunks = (M + pl.chunk_len - 1) / pl.chunk_len;
    pl.n_parts = pl.upc > 0 ? pl.n_chunks / pl.upc : pl.n_chunks;
    size_t elems = 0;
    pl.n_fold = 0;
    pl.G = 0;
    if (pl.n_chunks > 1) {
        if (pl.n_parts > 1) plan_fold(pl.n_parts, S, B, pl.G, pl.fold_levels, pl.n_fold, elems, ks->fold != nullptr);
        elems += (size_t)pl.n_parts * B * S;  // the (partial) chunk signatures themselves
    }
    pl.ws_bytes = elems * sizeof(float);
    return ok();
}

// fold n elements per path (element (j, b) at in + j*sj + b*sb) into out[b] (row stride S)
cudaError_t launch_fold(const TensorDims& d, const float* in, int64_t sj, int64_t sb, int64_t n, int64_t B, float* out,
                        float* ws, cudaStream_t st, FoldLaunch tf = nullptr) {
    const int64_t S = d.S;
    if (n == 1) {
        return cudaMemcpy2DAsync(out, S * sizeof(float), in, sb * sizeof(float), S * sizeof(float), B,
                                 cudaMemcpyDeviceToDevice, st);
    }
    int G = group_size_for(S, tf != nullptr);
    const float* cur = in;
    int64_t csj = sj, csb = sb;
    float* buf = ws;
    while (n > 1) {
        const int g = G > 0 ? G : 2;
        const int64_t ng = (n + g - 1) / g;
        float* dst;
        int64_t dsj, dsb;
        if (ng == 1) {
            dst = out;
            dsj = 0;
            dsb = S;
        } else {
            dst = buf;
            dsj = B * S;  // [ng, B, S]
            dsb = S;
            buf += ng * B * S;
        }
        if (G > 0) {
            GroupParams gp;
            gp.d = d;
            gp.in = cur;
            gp.in_sj = csj;
            gp.in_sb = csb;
            gp.n = n;
            gp.G = G;
            gp.out = dst;
            gp.out_sj = dsj;
            gp.out_sb = dsb;
            gp.B = B;
            if (tf) {
                cudaError_t e = tf(gp, (unsigned)ng, (unsigned)B, st);
                if (e != cudaSuccess) return e;
                count_launch();
                cur = dst;
                csj = dsj;
                csb = dsb;
                n = ng;
                continue;
            }
            const size_t smem = (size_t)G * S * sizeof(float);
            if (smem > 48 * 1024) {
                cudaError_t e = cudaFuncSetAttribute(combine_group_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)smem);
                if (e != cudaSuccess) return e;
            }
            dim3 grid((unsigned)ng, (unsigned)(B < 65535 ? B : 65535));
            combine_group_kernel<<<grid, 512, smem, st>>>(gp);
            count_launch();
        } else {
            // pairwise in global memory: dst(g) = cur(2g) [x] cur(2g+1)
            for (int64_t q = 0; q < ng; ++q) {
                const float* a = cur + 2 * q * csj;
                float* o = dst + q * dsj;
                if (2 * q + 1 < n) {
                    dim3 grid((unsigned)((S + 255) / 256), (unsigned)(B < 65535 ? B : 65535));
                    combine_pair_kernel<<<grid, 256, 0, st>>>(d, a, csb, a + csj, csb, o, dsb, B);
                    count_launch();
                } else {
                    cudaError_t e = cudaMemcpy2DAsync(o, dsb * sizeof(float), a, csb * sizeof(float),
                                                      S * sizeof(float), B, cudaMemcpyDeviceToDevice, st);
                    if (e != cudaSuccess) return e;
                }
            }
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        cur = dst;
        csj = dsj;
        csb = dsb;
        n = ng;
    }
    return cudaSuccess;
}

cudaError_t launch_word_reverse(const TensorDims& d, const float* in, int64_t si, float* out, int64_t so,
                                int64_t rows, cudaStream_t s) {
    const int64_t n = rows * d.S;
    if (n == 0) return cudaSuccess;
    word_reverse_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(d, in, si, out, so, rows);
    count_launch();
    return cudaGetLastError();
}

inline size_t align256(size_t n) { return (n + 255) / 256 * 256; }

sig_status_t run_signature(const float* path, int64_t B, int64_t L, int64_t C, int32_t depth, int32_t stream,
                           sig_basepoint_t bp, const float* basepoint, float* out, void* ws, size_t ws_bytes,
                           cudaStream_t s, float zsign = 1.0f, const float* initial = nullptr) {
    FwdPlan pl;
    sig_status_t st = make_fwd_plan(B, L, C, depth, stream, bp, pl);
    if (st != SIG_OK) return st;
    if (B == 0) return ok();  // empty batch: nothing to do (empty tensors may carry null pointers)
    if (!path || !out) return fail(SIG_ERR_INVALID_ARG, "path and out must be non-null");
    if (bp == SIG_BP_GIVEN && !basepoint) return fail(SIG_ERR_INVALID_ARG, "basepoint is NULL with SIG_BP_GIVEN");
    if (ws_bytes < pl.ws_bytes || (pl.ws_bytes > 0 && !ws))
        return fail(SIG_ERR_WORKSPACE, "workspace of %zu bytes needed, %zu given", pl.ws_bytes, ws_bytes);
    const TensorDims d = make_dims((int)C, depth);
    FwdParams prm{};
    prm.path = path;
    prm.basepoint = basepoint;
    prm.bp_mode = (int)bp;
    prm.stream = stream ? 1 : 0;
    prm.B = B;
    prm.L = L;
    prm.M = pl.M;
    prm.chunk_len = pl.chunk_len;
    prm.n_chunks = pl.n_chunks;
    prm.n_units = B * pl.n_chunks;
    prm.upc = pl.upc;
    prm.dims = d;
    prm.zsign = zsign;
    prm.initial = initial;
    float* units = (pl.n_chunks > 1 && pl.n_parts > 1) ? static_cast<float*>(ws) : out;
    prm.out = units;
    cudaError_t e = pl.launch(prm, s);
    if (e == cudaErrorInvalidConfiguration)
        return fail(SIG_ERR_UNSUPPORTED, "scan configuration exceeds the shared memory of one CTA");
    if (e != cudaSuccess) return cuda_status(e, "signature scan launch");
    count_launch();
    if (pl.n_chunks > 1 && pl.n_parts > 1) {
        // part (b, j) at units + (b*n_parts + j)*S  ->  element (j, b): sj = S, sb = n_parts*S
        float* fold_ws = units + (size_t)pl.n_parts * B * d.S;
        e = launch_fold(d, units, d.S, pl.n_parts * d.S, pl.n_parts, B, out, fold_ws, s, pl.ks->fold);
        if (e != cudaSuccess) return cuda_status(e, "chunk fold launch");
    }
    return ok();
}

// ---------------------------------------------------------------- logsig plans
struct DeviceTables {
    int64_t* lyn_idx = nullptr;
    int *rowptr = nullptr, *col = nullptr, *rowptrT = nullptr, *colT = nullptr;
    float *val = nullptr, *valT = nullptr;
    int device = 0;
};

}  // namespace

struct sig_logsig_plan_s {
    int C, N;
    sig_logsig_mode_t mode;
    int64_t S, w;
    DeviceTables dt;
};

namespace {

template <class T>
cudaError_t upload(T** dst, const std::vector<T>& v) {
    *dst = nullptr;
    if (v.empty()) return cudaSuccess;
    cudaError_t e = cudaMalloc(dst, v.size() * sizeof(T));
    if (e != cudaSuccess) return e;
    return cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
}

LogsigTables device_view(const sig_logsig_plan_s* pl) {
    LogsigTables tb{};
    tb.w = (int)pl->w;
    tb.lyn_idx = pl->dt.lyn_idx;
    tb.minv_rowptr = pl->dt.rowptr;
    tb.minv_col = pl->dt.col;
    tb.minv_val = pl->dt.val;
    tb.minvT_rowptr = pl->dt.rowptrT;
    tb.minvT_col = pl->dt.colT;
    tb.minvT_val = pl->dt.valT;
    return tb;
}

constexpr size_t kMaxSmem = 227 * 1024 - 512;  // dynamic shared memory per CTA (static arrays need the rest)

// K4's shared memory for one row: the compiled kernel where (C, N) has one (it keeps x only on
// levels < N, so e.g. brackets at C = 8, N = 5 fit), else the generic one.
size_t logsig_fwd_smem_any(const LDims& d, int64_t w, bool brackets) {
    if (find_logsig_fwd_t(d.C, d.N)) return logsig_fwd_t_smem(d.C, d.N, (int)w, brackets);
    return logsig_fwd_smem(d, (int)w, brackets);
}

sig_status_t check_logsig_smem(const LDims& d, int64_t w, bool brackets) {
    const bool bwd_ok = find_logsig_bwd_owned(d.C, d.N) != nullptr || logsig_bwd_smem(d, false) <= kMaxSmem;
    if (logsig_fwd_smem_any(d, w, brackets) > 227 * 1024 || !bwd_ok)
        return fail(SIG_ERR_UNSUPPORTED, "logsignature of C=%d depth=%d exceeds one CTA's shared memory", d.C, d.N);
    return SIG_OK;
}

// ---------------------------------------------------------------- backward time chunks (8(f)1)
struct BwdChunking {
    int64_t m = 1, chunk_len = 0;
};

// Time chunks of the reversible backward.  K2 stages increments per tile, so any
// path fits one CTA; chunks only add parallelism.  They are used -- when the caller gave the
// workspace -- if the batch alone cannot fill one resident wave of the backward (bwd_slots() CTAs
// per SM, register-limited): then ~one wave of CTAs in total, chunks of >= 64 steps.  Stream mode
// is never chunked (every output row feeds the gradient of all earlier steps).
void bwd_chunking(const FwdPlan& pl, int64_t B, int32_t stream, bool may_chunk, BwdChunking& ch) {
    ch.m = 1;
    ch.chunk_len = pl.M;
    if (stream || !may_chunk || B <= 0) return;
    const int64_t slots = pl.ks->bwd_slots ? pl.ks->bwd_slots() : 0;
    const int64_t wave = 148 * (slots > 0 ? slots : 8);
    if (B >= wave || B >= 148 * 4) return;
    int64_t m = (wave + B - 1) / B;
    const int64_t cap = pl.M / 64 > 1 ? pl.M / 64 : 1;
    if (m > cap) m = cap;
    ch.chunk_len = (pl.M + m - 1) / m;
    ch.m = (pl.M + ch.chunk_len - 1) / ch.chunk_len;
}

size_t bwd_chunk_ws_bytes(const BwdChunking& ch, int64_t B, int64_t S, int64_t C) {
    if (ch.m <= 1) return 0;
    const size_t rows = (size_t)B * ch.m;
    return align256(5 * rows * (size_t)S * sizeof(float)) + align256(rows * (size_t)C * sizeof(float));
}

// group size of the blocked chunk scan: the largest power of two <= 16 whose group, outputs and
// carry fit 200 KB of shared memory; 0 when fewer than 4 fit (large S: Hillis-Steele steps in
// global memory instead)
int block_scan_group(int64_t S) {
    int g = 16;
    while (g >= 4 && (size_t)(2 * g + 1) * S * sizeof(float) > 200 * 1024) g >>= 1;
    return g >= 4 ? g : 0;
}

// inclusive ordered product along the chunk axis of in[b*m + j] into out (suffix = 1: from the
// end).  Blocked (scan_group_t_kernel, compiled per shape): group totals, the scan of the totals
// (recursively), then every group's inclusive products started from its carry.  For signatures too
// large for it: Hillis-Steele steps (ceil(log2 m) launches, the last one writing `out`, the others
// alternating with tmp).  tmp holds rows * S floats (the blocked scan needs < 2/3 of that).
cudaError_t chunk_scan(const TensorDims& d, ScanLaunch sc, const float* in, float* out, float* tmp, int64_t B, int64_t m,
                       int suffix, cudaStream_t s) {
    const int g = block_scan_group(d.S);
    if (sc != nullptr && g > 0 && m > 1) {
        const int64_t ng = (m + g - 1) / g;
        ScanParams p{};
        p.in = in;
        p.B = B;
        p.m = m;
        p.g = g;
        p.suffix = suffix;
        if (ng > 1) {
            float* T = tmp;                        // [B, ng] group totals
            float* Ts = T + (size_t)B * ng * d.S;  // [B, ng] their inclusive scan
            p.tot = T;
            cudaError_t e = sc(p, s);
            count_launch();
            if (e == cudaSuccess) e = chunk_scan(d, sc, T, Ts, Ts + (size_t)B * ng * d.S, B, ng, suffix, s);
            if (e != cudaSuccess) return e;
            p.tot = nullptr;
            p.carry = Ts;
        }
        p.out = out;
        cudaError_t e = sc(p, s);
        count_launch();
        return e;
    }
    int steps = 0;
    for (int64_t o = 1; o < m; o <<= 1) ++steps;
    if (steps == 0) return cudaMemcpyAsync(out, in, (size_t)B * m * d.S * sizeof(float), cudaMemcpyDeviceToDevice, s);
    const int64_t n = B * m * d.S;
    const float* cur = in;
    int i = 0;
    for (int64_t o = 1; o < m; o <<= 1, ++i) {
        float* dst = ((steps - 1 - i) % 2 == 0) ? out : tmp;
        chunk_scan_step_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(d, cur, dst, B, m, o, suffix);
        count_launch();
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        cur = dst;
    }
    return cudaSuccess;
}

// The time-parallel reversible backward: recompute the chunk signatures (K1), their inclusive
// prefix and suffix products (K3 steps), the gradient at the end of every chunk, then reverse all
// chunks at once (K2, one CTA per chunk, each starting from its prefix product) and add the shares
// of the points two chunks have in common.
// Chunk signatures S_j of every path ([B, m, S], unit u = chunk u mod m of path u / m) by one K1
// launch over all chunks (the same launch for the forward's saved state and the backward's
// recomputation, so both produce the same bits).
cudaError_t launch_chunk_sigs(const FwdPlan& pl, const BwdChunking& ch, const BwdParams& prm, const TensorDims& d,
                              float* units, cudaStream_t s) {
    FwdParams f{};
    f.path = prm.path;
    f.basepoint = prm.basepoint;
    f.bp_mode = prm.bp_mode;
    f.stream = 0;
    f.B = prm.B;
    f.L = prm.L;
    f.M = pl.M;
    f.chunk_len = ch.chunk_len;
    f.n_chunks = ch.m;
    f.n_units = prm.B * ch.m;
    f.upc = 0;
    f.dims = d;
    f.out = units;
    f.zsign = prm.zsign;
    f.initial = prm.initial;
    cudaError_t e = pl.ks->fwd0(f, s);
    if (e == cudaSuccess) count_launch();
    return e;
}

// saved: the forward's chunk signatures and their inclusive prefix products ([2][B, m, S], from
// sig_signature_save), or nullptr to recompute them here.
sig_status_t run_bwd_chunked(const FwdPlan& pl, const BwdChunking& ch, BwdParams prm, const TensorDims& d, void* ws,
                             cudaStream_t s, const float* saved = nullptr) {
    const int64_t B = prm.B, m = ch.m, S = d.S, C = d.C;
    const size_t rows = (size_t)B * m;
    float* w = static_cast<float*>(ws);
    const float* units;
    const float* pin;
    cudaError_t e = cudaSuccess;
    if (saved) {
        units = saved;
        pin = saved + rows * S;
    } else {
        float* u = w;
        float* pn = u + rows * S;
        w = pn + rows * S;
        e = launch_chunk_sigs(pl, ch, prm, d, u, s);
        if (e != cudaSuccess) return cuda_status(e, "chunk signature launch");
        e = chunk_scan(d, pl.ks->scan, u, pn, w + rows * S, B, m, 0, s);
        if (e != cudaSuccess) return cuda_status(e, "chunk scan launch");
        units = u;
        pin = pn;
    }
    float* sfx = w;
    float* tmp = sfx + rows * S;
    float* gend = tmp + rows * S;
    float* edge = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) +
                                           align256((saved ? 3 : 5) * rows * (size_t)S * sizeof(float)));
    e = chunk_scan(d, pl.ks->scan, units, sfx, tmp, B, m, 1, s);
    if (e != cudaSuccess) return cuda_status(e, "chunk scan launch");
    const int64_t n = (int64_t)rows * S;
    chunk_gend_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(d, prm.grad_out, sfx, B, m, gend);
    count_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_status(e, "chunk gradient launch");
    prm.n_chunks = m;
    prm.chunk_len = ch.chunk_len;
    prm.sig_final = pin;
    prm.sf_stride = S;
    prm.grad_out = gend;
    prm.go_stride = S;
    prm.chunk_init = pin;
    prm.edge = edge;
    e = pl.ks->bwd(prm, s);
    if (e == cudaErrorInvalidConfiguration)
        return fail(SIG_ERR_UNSUPPORTED, "backward chunk of %lld increments does not fit", (long long)ch.chunk_len);
    if (e != cudaSuccess) return cuda_status(e, "signature backward launch");
    count_launch();
    const int64_t nf = B * (m - 1) * C;
    chunk_edge_fixup_kernel<<<(unsigned)((nf + 255) / 256), 256, 0, s>>>(prm.grad_path, edge, B, m, ch.chunk_len, prm.L,
                                                                          prm.bp_mode != 0, (int)C);
    count_launch();
    return cuda_status(cudaGetLastError(), "chunk edge launch");
}

// K4 on `rows` signature rows -> out
sig_status_t launch_logsig_fwd(const sig_logsig_plan_s* plan, const float* sig, int64_t rows, float* out,
                               cudaStream_t s) {
    LogsigParams p{};
    p.d = make_ldims(plan->C, plan->N);
    p.mode = (plan->mode == SIG_LOGSIG_EXPAND) ? 0 : (plan->mode == SIG_LOGSIG_BRACKETS ? 1 : 2);
    p.tb = device_view(plan);
    p.rows = rows;
    p.sig = sig;
    p.out = out;
    if (rows == 0) return ok();
    // many small rows (stream mode): one warp per row (logsig_rows.cuh) when its slice of shared
    // memory is small; big rows keep a CTA each
    LogsigRowsLaunch rl = find_logsig_rows_t(plan->C, plan->N);
    if (rows >= 8 * 148 &&
        (rl != nullptr || logsig_rows_warp_floats(p.d, (int)plan->w, p.mode == 1) * sizeof(float) <= 24 * 1024)) {
        cudaError_t e = rl ? rl(p, s) : launch_logsig_rows(p, s);
        if (e == cudaSuccess) {
            count_launch();
            return ok();
        }
        if (e != cudaErrorInvalidConfiguration) return cuda_status(e, "logsig rows launch");
        (void)cudaGetLastError();
    }
#if !defined(SIG_LOGSIG_FWD_GENERIC)
    if (LogsigFwdLaunch fn = find_logsig_fwd_t(plan->C, plan->N)) {
        cudaError_t e = fn(p, s);
        if (e == cudaSuccess) {
            count_launch();
            return ok();
        }
        if (e != cudaErrorInvalidConfiguration) return cuda_status(e, "logsig launch");
        (void)cudaGetLastError();  // shape too large for the compiled form: the generic kernel below
    }
#endif
    const size_t smem = logsig_fwd_smem(p.d, (int)plan->w, p.mode == 1);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(logsig_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return cuda_status(e, "logsig smem attribute");
    }
    logsig_fwd_kernel<<<(unsigned)rows, LOGSIG_THREADS, smem, s>>>(p);
    count_launch();
    return cuda_status(cudaGetLastError(), "logsig launch");
}

// K5 on `rows` rows: dL/dlog -> dL/dSig (gsig), glog = [rows, S] scratch of the fallback kernel
sig_status_t launch_logsig_bwd(const sig_logsig_plan_s* plan, const float* grad_out, const float* sig, int64_t rows,
                               float* glog, float* gsig, cudaStream_t s) {
    LogsigParams p{};
    p.d = make_ldims(plan->C, plan->N);
    p.mode = (plan->mode == SIG_LOGSIG_EXPAND) ? 0 : (plan->mode == SIG_LOGSIG_BRACKETS ? 1 : 2);
    p.tb = device_view(plan);
    p.rows = rows;
    p.sig = sig;
    p.gout = grad_out;
    p.gsig = gsig;
    p.glog_ws = glog;
    const size_t smem_owned = logsig_bwd_owned_smem(p.d);
    if (LogsigBwdLaunch fn = find_logsig_bwd_owned(plan->C, plan->N)) {
        cudaError_t e = fn(p, s);
        if (e != cudaSuccess) return cuda_status(e, "logsig backward launch");
    } else if (smem_owned <= kMaxSmem) {
        if (smem_owned > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(logsig_bwd_owned_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem_owned);
            if (e != cudaSuccess) return cuda_status(e, "logsig bwd smem attribute");
        }
        logsig_bwd_owned_kernel<<<(unsigned)rows, LOGSIG_THREADS, smem_owned, s>>>(p);
    } else {
        p.gl_smem = logsig_bwd_smem(p.d, true) <= kMaxSmem;
        const size_t smem = logsig_bwd_smem(p.d, p.gl_smem);
        if (smem > 48 * 1024) {
            cudaError_t e =
                cudaFuncSetAttribute(logsig_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return cuda_status(e, "logsig bwd smem attribute");
        }
        logsig_bwd_kernel<<<(unsigned)rows, LOGSIG_THREADS, smem, s>>>(p);
    }
    count_launch();
    return cuda_status(cudaGetLastError(), "logsig backward launch");
}

// host index arrays -> device copies in the workspace (pageable source: the copy is staged before
// cudaMemcpyAsync returns, so the host arrays may go away afterwards)
cudaError_t upload(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes == 0) return cudaSuccess;
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
}

}  // namespace

// ================================================================ extern "C"
extern "C" {

int64_t sig_signature_channels(int64_t C, int32_t depth) { return sig_channels_checked(C, depth); }

int64_t sig_logsignature_channels(int64_t C, int32_t depth, sig_logsig_mode_t mode) {
    if (C < 1 || depth < 1) return -1;
    if (mode == SIG_LOGSIG_EXPAND) return sig_channels_checked(C, depth);
    if (mode == SIG_LOGSIG_WORDS || mode == SIG_LOGSIG_BRACKETS) return witt_dimension(C, depth);
    return -1;
}

int32_t sig_is_supported(int64_t C, int32_t depth, int32_t backward) {
    if (C < 1 || C > 8 || depth < 1) return 0;
    const KernelSet* ks = find_kernels((int)C, depth);
    if (!ks) return 0;
    return backward ? (ks->bwd != nullptr) : 1;
}

uint64_t sig_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

const char* sig_status_string(sig_status_t st) {
    switch (st) {
        case SIG_OK: return "SIG_OK";
        case SIG_ERR_INVALID_ARG: return "SIG_ERR_INVALID_ARG";
        case SIG_ERR_SHAPE: return "SIG_ERR_SHAPE";
        case SIG_ERR_UNSUPPORTED: return "SIG_ERR_UNSUPPORTED";
        case SIG_ERR_CUDA: return "SIG_ERR_CUDA";
        case SIG_ERR_WORKSPACE: return "SIG_ERR_WORKSPACE";
    }
    return "SIG_ERR_UNKNOWN";
}

const char* sig_last_error(void) { return g_last_error.c_str(); }

size_t sig_signature_workspace_size(int64_t B, int64_t L, int64_t C, int32_t depth, int32_t stream,
                                    sig_basepoint_t bp) {
    FwdPlan pl;
    if (make_fwd_plan(B, L, C, depth, stream, bp, pl) != SIG_OK) return 0;
    return pl.ws_bytes;
}

sig_status_t sig_signature(const float* path, int64_t B, int64_t L, int64_t C, int32_t depth, int32_t stream,
                           sig_basepoint_t bp, const float* basepoint, float* out, void* ws, size_t ws_bytes,
                           sig_cuda_stream_t s) {
    return run_signature(path, B, L, C, depth, stream, bp, basepoint, out, ws, ws_bytes, (cudaStream_t)s);
}

size_t sig_signature_ex_workspace_size(int64_t B, int64_t L, int64_t C, int32_t depth, int32_t stream,
                                       sig_basepoint_t bp, int32_t inverse, int32_t has_initial) {
    FwdPlan pl;
    if (make_fwd_plan(B, L, C, depth, stream, bp, pl) != SIG_OK) return 0;
    if (!inverse || !has_initial) return pl.ws_bytes;
    return align256(pl.ws_bytes) + (size_t)B * (size_t)sig_channels_checked(C, depth) * sizeof(float);
}

sig_status_t sig_signature_ex(const float* path, int64_t B, int64_t L, int64_t C, int32_t depth, int32_t stream,
                              sig_basepoint_t bp, const float* basepoint, int32_t inverse, const float* initial,
                              float* out, void* ws, size_t ws_bytes, sig_cuda_stream_t s) {
    if (!inverse)
        return run_signature(path, B, L, C, depth, stream, bp, basepoint, out, ws, ws_bytes, (cudaStream_t)s, 1.0f,
                             initial);
    // inverse (reading R18): scan the negated path from alpha(initial), then reverse the
    // words -- alpha(Sig(x)^-1 [x] I) = alpha(I) [x] exp(-z_0) [x] ... [x] exp(-z_{M-1})
    FwdPlan pl;
    sig_status_t st = make_fwd_plan(B, L, C, depth, stream, bp, pl);
    if (st != SIG_OK) return st;
    if (B == 0) return ok();
    const size_t need = sig_signature_ex_workspace_size(B, L, C, depth, stream, bp, inverse, initial != nullptr);
    if (ws_bytes < need || (need > 0 && !ws))
        return fail(SIG_ERR_WORKSPACE, "workspace of %zu bytes needed, %zu given", need, ws_bytes);
    if (!out) return fail(SIG_ERR_INVALID_ARG, "out must be non-null");
    const TensorDims d = make_dims((int)C, depth);
    const float* ia = nullptr;
    if (initial) {
        float* t = reinterpret_cast<float*>(static_cast<char*>(ws) + align256(pl.ws_bytes));
        cudaError_t e = launch_word_reverse(d, initial, d.S, t, d.S, B, (cudaStream_t)s);
        if (e != cudaSuccess) return cuda_status(e, "word reversal launch");
        ia = t;
    }
    st = run_signature(path, B, L, C, depth, stream, bp, basepoint, out, ws, pl.ws_bytes, (cudaStream_t)s, -1.0f, ia);
    if (st != SIG_OK) return st;
    const int64_t rows = stream ? B * pl.M : B;
    cudaError_t e = launch_word_reverse(d, out, d.S, out, d.S, rows, (cudaStream_t)s);
    return cuda_status(e, "word reversal launch");
}

size_t sig_signature_backward_ex_workspace_size(int64_t B, int64_t L, int64_t C, int32_t depth, int32_t stream,
                                                sig_basepoint_t bp, int32_t inverse, int32_t has_initial,
                                                int32_t want_grad_initial) {
    FwdPlan pl;
    if (make_fwd_plan(B, L, C, depth, stream, bp, pl) != SIG_OK || !pl.ks->bwd) return 0;
    const size_t S = (size_t)sig_channels_checked(C, depth);
    size_t inv = 0;
    if (inverse) {
        const int64_t rows = stream ? B * pl.M : B;
        inv = align256(((size_t)rows * S + (size_t)B * S * (1 + (has_initial ? 1 : 0) + (want_grad_initial ? 1 : 0))) *
                       sizeof(float));
    }
    BwdChunking ch;
    bwd_chunking(pl, B, stream, true, ch);
    return inv + bwd_chunk_ws_bytes(ch, B, (int64_t)S, C);
}

sig_status_t sig_signature_backward_ex(const float* grad_out, const float* path, const float* out_saved, int64_t B,
                                       int64_t L, int64_t C, int32_t depth, int32_t stream, sig_basepoint_t bp,
                                       const float* basepoint, int32_t inverse, const float* initial,
                                       float* grad_path, float* grad_basepoint, float* grad_initial, void* ws,
                                       size_t ws_bytes, sig_cuda_stream_t s) {
    FwdPlan pl;
    sig_status_t st = make_fwd_plan(B, L, C, depth, stream, bp, pl);
    if (st != SIG_OK) return st;
    if (!pl.ks->bwd)
        return fail(SIG_ERR_UNSUPPORTED, "no sm_100a backward kernel for C=%lld depth=%d", (long long)C, depth);
    if (B == 0) return ok();
    if (!grad_out || !path || !out_saved || !grad_path)
        return fail(SIG_ERR_INVALID_ARG, "grad_out, path, out_saved and grad_path must be non-null");
    if (bp == SIG_BP_GIVEN && !basepoint) return fail(SIG_ERR_INVALID_ARG, "basepoint is NULL with SIG_BP_GIVEN");
    const TensorDims d = make_dims((int)C, depth);
    const int64_t S = d.S;
    // workspace: the alpha images (inverse) first, then the backward's time chunks.  Chunks that
    // only improve occupancy are used when the caller gave room for them.
    const size_t inv_bytes =
        inverse ? align256((((size_t)(stream ? B * pl.M : B)) * S +
                            (size_t)B * S * (1 + (initial ? 1 : 0) + (grad_initial ? 1 : 0))) * sizeof(float))
                : 0;
    BwdChunking ch;
    const size_t full = sig_signature_backward_ex_workspace_size(B, L, C, depth, stream, bp, inverse,
                                                                 initial != nullptr, grad_initial != nullptr);
    const bool roomy = ws != nullptr && ws_bytes >= full;
    bwd_chunking(pl, B, stream, roomy, ch);
    const size_t need = inv_bytes + bwd_chunk_ws_bytes(ch, B, S, C);
    if (ws_bytes < need || (need > 0 && !ws))
        return fail(SIG_ERR_WORKSPACE, "workspace of %zu bytes needed, %zu given", need, ws_bytes);
    const int64_t rows = stream ? B * pl.M : B;
    // the forward's final state of each path: its last output row
    const float* fin = stream ? out_saved + (size_t)(pl.M - 1) * S : out_saved;
    const int64_t fin_stride = stream ? pl.M * S : S;
    BwdParams prm{};
    prm.grad_out = grad_out;
    prm.path = path;
    prm.basepoint = basepoint;
    prm.sig_final = fin;
    prm.sf_stride = fin_stride;
    prm.bp_mode = (int)bp;
    prm.stream = stream ? 1 : 0;
    prm.B = B;
    prm.L = L;
    prm.M = pl.M;
    prm.grad_path = grad_path;
    prm.grad_bp = (bp == SIG_BP_GIVEN) ? grad_basepoint : nullptr;
    prm.zsign = 1.0f;
    prm.initial = initial;
    prm.grad_initial = grad_initial;
    float* gi_alpha = nullptr;
    cudaStream_t cs = (cudaStream_t)s;
    if (inverse) {
        // the forward scanned the negated path from alpha(initial) and reversed the words of its
        // output (reading R18): pull every tensor back through alpha, run the scan's VJP, push the
        // initial's gradient forward through alpha again
        float* w = static_cast<float*>(ws);
        float* ga = w;
        float* sa = ga + (size_t)rows * S;
        float* ia = sa + (size_t)B * S;
        float* gia = ia + (initial ? (size_t)B * S : 0);
        cudaError_t e = launch_word_reverse(d, grad_out, S, ga, S, rows, cs);
        if (e == cudaSuccess) e = launch_word_reverse(d, fin, fin_stride, sa, S, B, cs);
        if (e == cudaSuccess && initial) e = launch_word_reverse(d, initial, S, ia, S, B, cs);
        if (e != cudaSuccess) return cuda_status(e, "word reversal launch");
        prm.grad_out = ga;
        prm.sig_final = sa;
        prm.sf_stride = S;
        prm.zsign = -1.0f;
        prm.initial = initial ? ia : nullptr;
        if (grad_initial) {
            gi_alpha = gia;
            prm.grad_initial = gia;
        }
    }
    prm.n_chunks = 1;
    prm.chunk_len = pl.M;
    prm.go_stride = S;
    if (ch.m > 1) {
        st = run_bwd_chunked(pl, ch, prm, d, static_cast<char*>(ws) + inv_bytes, cs);
        if (st != SIG_OK) return st;
    } else {
        cudaError_t e = pl.ks->bwd(prm, cs);
        if (e == cudaSuccess) count_launch();
        if (e == cudaErrorInvalidConfiguration)
            return fail(SIG_ERR_UNSUPPORTED, "path of %lld increments does not fit the backward's shared memory",
                        (long long)pl.M);
        if (e != cudaSuccess) return cuda_status(e, "signature backward launch");
    }
    if (gi_alpha) {
        cudaError_t e;
        e = launch_word_reverse(d, gi_alpha, S, grad_initial, S, B, cs);
        if (e != cudaSuccess) return cuda_status(e, "word reversal launch");
    }
    return ok();
}

// ---------------------------------------------------------------- saved chunk states
// (sig.h "forward with saved chunk states"): the time-parallel backward starts every chunk from the
// product of the earlier chunks; the forward can leave those states behind instead of the backward
// recomputing them (one K1 pass over the whole path plus a prefix scan).
// chunking of the backward for a plain call (no stream / inverse / initial); m <= 1: none
static bool saved_plan(int64_t B, int64_t L, int64_t C, int32_t depth, sig_basepoint_t bp, FwdPlan& pl, BwdChunking& ch) {
    if (make_fwd_plan(B, L, C, depth, 0, bp, pl) != SIG_OK || !pl.ks->bwd || B <= 0) return false;
    bwd_chunking(pl, B, 0, true, ch);
    return ch.m > 1;
}

size_t sig_signature_saved_bytes(int64_t B, int64_t L, int64_t C, int32_t depth, sig_basepoint_t bp) {
    FwdPlan pl;
    BwdChunking ch;
    if (!saved_plan(B, L, C, depth, bp, pl, ch)) return 0;
    return align256(2 * (size_t)B * ch.m * (size_t)sig_channels_checked(C, depth) * sizeof(float));
}

size_t sig_signature_save_workspace_size(int64_t B, int64_t L, int64_t C, int32_t depth, sig_basepoint_t bp) {
    FwdPlan pl;
    BwdChunking ch;
    if (!saved_plan(B, L, C, depth, bp, pl, ch)) return sig_signature_workspace_size(B, L, C, depth, 0, bp);
    return align256((size_t)B * ch.m * (size_t)sig_channels_checked(C, depth) * sizeof(float));
}

sig_status_t sig_signature_save(const float* path, int64_t B, int64_t L, int64_t C, int32_t depth, sig_basepoint_t bp,
                                const float* basepoint, float* out, float* saved, size_t saved_bytes, void* ws,
                                size_t ws_bytes, sig_cuda_stream_t s) {
    FwdPlan pl;
    BwdChunking ch;
    if (!saved_plan(B, L, C, depth, bp, pl, ch))  // no chunks: the plain forward (argument checks there)
        return run_signature(path, B, L, C, depth, 0, bp, basepoint, out, ws, ws_bytes, (cudaStream_t)s);
    if (!path || !out || !saved) return fail(SIG_ERR_INVALID_ARG, "path, out and saved must be non-null");
    if (bp == SIG_BP_GIVEN && !basepoint) return fail(SIG_ERR_INVALID_ARG, "basepoint is NULL with SIG_BP_GIVEN");
    const size_t need_saved = sig_signature_saved_bytes(B, L, C, depth, bp);
    const size_t need_ws = sig_signature_save_workspace_size(B, L, C, depth, bp);
    if (saved_bytes < need_saved)
        return fail(SIG_ERR_WORKSPACE, "saved buffer of %zu bytes needed, %zu given", need_saved, saved_bytes);
    if (ws_bytes < need_ws || !ws) return fail(SIG_ERR_WORKSPACE, "workspace of %zu bytes needed, %zu given", need_ws, ws_bytes);
    const TensorDims d = make_dims((int)C, depth);
    const int64_t S = d.S, m = ch.m;
    const size_t rows = (size_t)B * m;
    BwdParams prm{};
    prm.path = path;
    prm.basepoint = basepoint;
    prm.bp_mode = (int)bp;
    prm.B = B;
    prm.L = L;
    prm.M = pl.M;
    prm.zsign = 1.0f;
    cudaStream_t cs = (cudaStream_t)s;
    cudaError_t e = launch_chunk_sigs(pl, ch, prm, d, saved, cs);
    if (e != cudaSuccess) return cuda_status(e, "chunk signature launch");
    float* pin = saved + rows * S;  // inclusive prefix products: the last one of a path is its signature
    e = chunk_scan(d, pl.ks->scan, saved, pin, static_cast<float*>(ws), B, m, 0, cs);
    if (e != cudaSuccess) return cuda_status(e, "chunk scan launch");
    e = cudaMemcpy2DAsync(out, (size_t)S * sizeof(float), pin + (size_t)(m - 1) * S, (size_t)m * S * sizeof(float),
                          (size_t)S * sizeof(float), (size_t)B, cudaMemcpyDeviceToDevice, cs);
    return cuda_status(e, "signature copy");
}

size_t sig_signature_backward_saved_workspace_size(int64_t B, int64_t L, int64_t C, int32_t depth, sig_basepoint_t bp) {
    FwdPlan pl;
    BwdChunking ch;
    if (!saved_plan(B, L, C, depth, bp, pl, ch)) return 0;
    const size_t S = (size_t)sig_channels_checked(C, depth), rows = (size_t)B * ch.m;
    return align256(3 * rows * S * sizeof(float)) + align256(rows * (size_t)C * sizeof(float));
}

sig_status_t sig_signature_backward_saved(const float* grad_out, const float* path, const float* out_saved,
                                          const float* saved, size_t saved_bytes, int64_t B, int64_t L, int64_t C,
                                          int32_t depth, sig_basepoint_t bp, const float* basepoint, float* grad_path,
                                          float* grad_basepoint, void* ws, size_t ws_bytes, sig_cuda_stream_t s) {
    FwdPlan pl;
    BwdChunking ch;
    if (!saved_plan(B, L, C, depth, bp, pl, ch))  // no chunks: the plain reversal from out_saved
        return sig_signature_backward_ex(grad_out, path, out_saved, B, L, C, depth, 0, bp, basepoint, 0, nullptr,
                                         grad_path, grad_basepoint, nullptr, nullptr, 0, s);
    if (!grad_out || !path || !saved || !grad_path)
        return fail(SIG_ERR_INVALID_ARG, "grad_out, path, saved and grad_path must be non-null");
    if (bp == SIG_BP_GIVEN && !basepoint) return fail(SIG_ERR_INVALID_ARG, "basepoint is NULL with SIG_BP_GIVEN");
    const size_t need_saved = sig_signature_saved_bytes(B, L, C, depth, bp);
    const size_t need_ws = sig_signature_backward_saved_workspace_size(B, L, C, depth, bp);
    if (saved_bytes < need_saved)
        return fail(SIG_ERR_WORKSPACE, "saved buffer of %zu bytes needed, %zu given", need_saved, saved_bytes);
    if (ws_bytes < need_ws || !ws) return fail(SIG_ERR_WORKSPACE, "workspace of %zu bytes needed, %zu given", need_ws, ws_bytes);
    const TensorDims d = make_dims((int)C, depth);
    BwdParams prm{};
    prm.grad_out = grad_out;
    prm.path = path;
    prm.basepoint = basepoint;
    prm.bp_mode = (int)bp;
    prm.stream = 0;
    prm.B = B;
    prm.L = L;
    prm.M = pl.M;
    prm.grad_path = grad_path;
    prm.grad_bp = (bp == SIG_BP_GIVEN) ? grad_basepoint : nullptr;
    prm.zsign = 1.0f;
    prm.go_stride = d.S;
    return run_bwd_chunked(pl, ch, prm, d, ws, (cudaStream_t)s, saved);
}

sig_status_t sig_signature_backward(const float* grad_out, const float* path, const float* out_saved, int64_t B,
                                    int64_t L, int64_t C, int32_t depth, int32_t stream, sig_basepoint_t bp,
                                    const float* basepoint, float* grad_path, float* grad_basepoint,
                                    sig_cuda_stream_t s) {
    return sig_signature_backward_ex(grad_out, path, out_saved, B, L, C, depth, stream, bp, basepoint, 0, nullptr,
                                     grad_path, grad_basepoint, nullptr, nullptr, 0, s);
}

// ---------------------------------------------------------------- host-resident batches
// Workspace layout: [path B*L*C][grad_out B*S][sig B*S][grad_path B*L*C][forward workspace of one
// slice], each region 256-byte aligned.
static size_t host_fb_layout(int64_t B, int64_t L, int64_t C, int32_t depth, int32_t chunks, size_t off[5]) {
    const int64_t S = sig_channels_checked(C, depth);
    if (S < 0 || B < 1 || L < 2 || C < 1 || chunks < 1) return 0;
    const int64_t bc = (B + chunks - 1) / chunks;
    size_t o = 0;
    off[0] = o; o = align256(o + (size_t)B * L * C * sizeof(float));
    off[1] = o; o = align256(o + (size_t)B * S * sizeof(float));
    off[2] = o; o = align256(o + (size_t)B * S * sizeof(float));
    off[3] = o; o = align256(o + (size_t)B * L * C * sizeof(float));
    off[4] = o;
    // the slices are bc paths each except a shorter last one, whose plan may differ (time chunks)
    FwdPlan pl, pll;
    const int64_t last = B - (B - 1) / bc * bc;
    if (make_fwd_plan(bc, L, C, depth, 0, SIG_BP_NONE, pl) != SIG_OK) return 0;
    if (make_fwd_plan(last, L, C, depth, 0, SIG_BP_NONE, pll) != SIG_OK) return 0;
    return o + align256(pl.ws_bytes > pll.ws_bytes ? pl.ws_bytes : pll.ws_bytes);
}

// Copy streams and events of the host pipeline, per device and per host thread (a stream belongs to
// the device that was current when it was created).  Events are reused call after call: every wait
// on them is enqueued before the call returns.
struct HostPipeRes {
    cudaStream_t h2d = nullptr, d2h = nullptr;
    std::vector<cudaEvent_t> ev;
};

static sig_status_t host_pipe_res(int n_events, HostPipeRes*& out) {
    thread_local std::vector<std::pair<int, HostPipeRes>> per_dev;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
    HostPipeRes* r = nullptr;
    for (auto& pr : per_dev)
        if (pr.first == dev) r = &pr.second;
    if (!r) {
        per_dev.emplace_back(dev, HostPipeRes{});
        r = &per_dev.back().second;
    }
    if (!r->h2d && (e = cudaStreamCreateWithFlags(&r->h2d, cudaStreamNonBlocking)) != cudaSuccess)
        return cuda_status(e, "stream");
    if (!r->d2h && (e = cudaStreamCreateWithFlags(&r->d2h, cudaStreamNonBlocking)) != cudaSuccess)
        return cuda_status(e, "stream");
    while ((int)r->ev.size() < n_events) {
        cudaEvent_t ev;
        if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return cuda_status(e, "event");
        r->ev.push_back(ev);
    }
    out = r;
    return SIG_OK;
}

size_t sig_signature_fwd_bwd_host_workspace_size(int64_t B, int64_t L, int64_t C, int32_t depth, int32_t chunks) {
    size_t off[5];
    return host_fb_layout(B, L, C, depth, chunks, off);
}

sig_status_t sig_signature_fwd_bwd_host(const float* path_h, const float* grad_out_h, int64_t B, int64_t L, int64_t C,
                                        int32_t depth, float* grad_path_h, int32_t chunks, void* ws, size_t ws_bytes,
                                        sig_cuda_stream_t s) {
    if (!path_h || !grad_out_h || !grad_path_h) return fail(SIG_ERR_INVALID_ARG, "host buffers must be non-null");
    if (B == 0) return ok();
    size_t off[5];
    const size_t need = host_fb_layout(B, L, C, depth, chunks, off);
    if (need == 0) return fail(SIG_ERR_SHAPE, "bad shape B=%lld L=%lld C=%lld depth=%d chunks=%d", (long long)B,
                               (long long)L, (long long)C, depth, chunks);
    if (!ws || ws_bytes < need) return fail(SIG_ERR_WORKSPACE, "workspace of %zu bytes needed, %zu given", need, ws_bytes);
    const int64_t S = sig_channels_checked(C, depth);
    char* w = static_cast<char*>(ws);
    float* d_path = reinterpret_cast<float*>(w + off[0]);
    float* d_go = reinterpret_cast<float*>(w + off[1]);
    float* d_sig = reinterpret_cast<float*>(w + off[2]);
    float* d_gp = reinterpret_cast<float*>(w + off[3]);
    void* d_fws = w + off[4];
    const size_t fws_bytes = need - off[4];
    const cudaStream_t cs = (cudaStream_t)s;
    const int64_t bc = (B + chunks - 1) / chunks;
    const int n = (int)((B + bc - 1) / bc);
    HostPipeRes* res = nullptr;
    sig_status_t rs = host_pipe_res(2 * n + 3, res);
    if (rs != SIG_OK) return rs;
    const cudaStream_t h2d = res->h2d, d2h = res->d2h;
    cudaEvent_t* ev = res->ev.data();
    // the caller's stream resumes only after every copy issued so far (also on an early error
    // return, so that no copy into the caller's buffers outlives the call's stream order)
    auto join = [&] {
        cudaEventRecord(ev[2 * n + 1], d2h);
        cudaStreamWaitEvent(cs, ev[2 * n + 1], 0);
        cudaEventRecord(ev[2 * n + 2], h2d);
        cudaStreamWaitEvent(cs, ev[2 * n + 2], 0);
    };
    // the copies start after everything already queued on the caller's stream
    cudaEventRecord(ev[2 * n], cs);
    cudaStreamWaitEvent(h2d, ev[2 * n], 0);
    cudaStreamWaitEvent(d2h, ev[2 * n], 0);
    for (int k = 0; k < n; ++k) {
        const int64_t a = k * bc, b = (a + bc < B) ? a + bc : B;
        cudaMemcpyAsync(d_path + a * L * C, path_h + a * L * C, (size_t)(b - a) * L * C * sizeof(float),
                        cudaMemcpyHostToDevice, h2d);
        cudaMemcpyAsync(d_go + a * S, grad_out_h + a * S, (size_t)(b - a) * S * sizeof(float), cudaMemcpyHostToDevice,
                        h2d);
        cudaEventRecord(ev[k], h2d);
    }
    for (int k = 0; k < n; ++k) {
        const int64_t a = k * bc, b = (a + bc < B) ? a + bc : B;
        cudaStreamWaitEvent(cs, ev[k], 0);
        sig_status_t st = run_signature(d_path + a * L * C, b - a, L, C, depth, 0, SIG_BP_NONE, nullptr, d_sig + a * S,
                                        d_fws, fws_bytes, cs);
        if (st == SIG_OK)
            st = sig_signature_backward(d_go + a * S, d_path + a * L * C, d_sig + a * S, b - a, L, C, depth, 0,
                                        SIG_BP_NONE, nullptr, d_gp + a * L * C, nullptr, s);
        if (st != SIG_OK) {
            const std::string msg = g_last_error;
            join();
            g_last_error = msg;
            return st;
        }
        cudaEventRecord(ev[n + k], cs);
        cudaStreamWaitEvent(d2h, ev[n + k], 0);
        cudaMemcpyAsync(grad_path_h + a * L * C, d_gp + a * L * C, (size_t)(b - a) * L * C * sizeof(float),
                        cudaMemcpyDeviceToHost, d2h);
    }
    join();
    return cuda_status(cudaGetLastError(), "host pipeline");
}

sig_status_t sig_signature_combine(const float* a, const float* b, int64_t B, int64_t C, int32_t depth, float* out,
                                   sig_cuda_stream_t s) {
    const int64_t S = sig_channels_checked(C, depth);
    if (S < 0 || depth > 15) return fail(SIG_ERR_INVALID_ARG, "bad C=%lld depth=%d", (long long)C, depth);
    if (S >= (1LL << 28)) return fail(SIG_ERR_UNSUPPORTED, "signature of %lld floats too large", (long long)S);
    if (!a || !b || !out) return fail(SIG_ERR_INVALID_ARG, "a, b and out must be non-null");
    if (B < 0) return fail(SIG_ERR_SHAPE, "B < 0");
    if (B == 0) return ok();
    const TensorDims d = make_dims((int)C, depth);
    dim3 grid((unsigned)((S + 255) / 256), (unsigned)(B < 65535 ? B : 65535));
    combine_pair_kernel<<<grid, 256, 0, (cudaStream_t)s>>>(d, a, S, b, S, out, S, B);
    count_launch();
    return cuda_status(cudaGetLastError(), "combine launch");
}

sig_status_t sig_signature_combine_backward(const float* grad_out, const float* a, const float* b, int64_t B,
                                            int64_t C, int32_t depth, float* grad_a, float* grad_b,
                                            sig_cuda_stream_t s) {
    const int64_t S = sig_channels_checked(C, depth);
    if (S < 0 || depth > 15) return fail(SIG_ERR_INVALID_ARG, "bad C=%lld depth=%d", (long long)C, depth);
    if (S >= (1LL << 28)) return fail(SIG_ERR_UNSUPPORTED, "signature of %lld floats too large", (long long)S);
    if (!grad_out || !a || !b) return fail(SIG_ERR_INVALID_ARG, "grad_out, a and b must be non-null");
    if (B < 0) return fail(SIG_ERR_SHAPE, "B < 0");
    if (B == 0 || (!grad_a && !grad_b)) return ok();
    const TensorDims d = make_dims((int)C, depth);
    dim3 grid((unsigned)((S + 255) / 256), (unsigned)(B < 65535 ? B : 65535));
    combine_pair_bwd_kernel<<<grid, 256, 0, (cudaStream_t)s>>>(d, grad_out, a, b, grad_a, grad_b, B);
    count_launch();
    return cuda_status(cudaGetLastError(), "combine backward launch");
}

size_t sig_multi_signature_combine_workspace_size(int64_t n, int64_t B, int64_t C, int32_t depth) {
    const int64_t S = sig_channels_checked(C, depth);
    if (S < 0 || n < 1 || B < 0) return 0;
    int G;
    int64_t lv[64];
    int nl;
    size_t elems;
    const KernelSet* ks = (C <= 8) ? find_kernels((int)C, depth) : nullptr;
    plan_fold(n, S, B, G, lv, nl, elems, ks && ks->fold);
    return elems * sizeof(float);
}

sig_status_t sig_multi_signature_combine(const float* sigs, int64_t n, int64_t B, int64_t C, int32_t depth,
                                         float* out, void* ws, size_t ws_bytes, sig_cuda_stream_t s) {
    const int64_t S = sig_channels_checked(C, depth);
    if (S < 0 || depth > 15) return fail(SIG_ERR_INVALID_ARG, "bad C=%lld depth=%d", (long long)C, depth);
    if (S >= (1LL << 28)) return fail(SIG_ERR_UNSUPPORTED, "signature of %lld floats too large", (long long)S);
    if (!sigs || !out) return fail(SIG_ERR_INVALID_ARG, "sigs and out must be non-null");
    if (n < 1 || B < 0) return fail(SIG_ERR_SHAPE, "n=%lld must be >= 1", (long long)n);
    const size_t need = sig_multi_signature_combine_workspace_size(n, B, C, depth);
    if (ws_bytes < need || (need > 0 && !ws))
        return fail(SIG_ERR_WORKSPACE, "workspace of %zu bytes needed, %zu given", need, ws_bytes);
    if (B == 0) return ok();
    const TensorDims d = make_dims((int)C, depth);
    const KernelSet* ks = (C <= 8) ? find_kernels((int)C, depth) : nullptr;
    cudaError_t e = launch_fold(d, sigs, B * S, S, n, B, out, static_cast<float*>(ws), (cudaStream_t)s,
                                ks ? ks->fold : nullptr);
    return cuda_status(e, "multi combine launch");
}

sig_status_t sig_logsig_plan_create(int64_t C, int32_t depth, sig_logsig_mode_t mode, sig_logsig_plan_t* plan) {
    if (!plan) return fail(SIG_ERR_INVALID_ARG, "plan is NULL");
    *plan = nullptr;
    if (C < 1 || C > 8 || depth < 1 || depth > 15)
        return fail(SIG_ERR_INVALID_ARG, "bad C=%lld depth=%d", (long long)C, depth);
    if (mode != SIG_LOGSIG_EXPAND && mode != SIG_LOGSIG_BRACKETS && mode != SIG_LOGSIG_WORDS)
        return fail(SIG_ERR_INVALID_ARG, "bad logsignature mode %d", (int)mode);
    if (!find_kernels((int)C, depth))
        return fail(SIG_ERR_UNSUPPORTED, "no sm_100a kernel instantiated for C=%lld depth=%d", (long long)C, depth);
    const LDims d = make_ldims((int)C, depth);
    auto pl = std::make_unique<sig_logsig_plan_s>();
    pl->C = (int)C;
    pl->N = depth;
    pl->mode = mode;
    pl->S = d.S;
    pl->w = (mode == SIG_LOGSIG_EXPAND) ? d.S : witt_dimension(C, depth);
    sig_status_t st = check_logsig_smem(d, pl->w, mode == SIG_LOGSIG_BRACKETS);
    if (st != SIG_OK) return st;
    cudaGetDevice(&pl->dt.device);
    if (mode != SIG_LOGSIG_EXPAND) {
        LyndonTables T;
        try {
            T = build_lyndon_tables((int)C, depth, mode == SIG_LOGSIG_BRACKETS);
        } catch (const std::exception& ex) {
            return fail(SIG_ERR_INVALID_ARG, "Lyndon tables: %s", ex.what());
        }
        if ((int64_t)T.flat_index.size() != pl->w)
            return fail(SIG_ERR_INVALID_ARG, "Lyndon word count %zu != Witt %lld", T.flat_index.size(),
                        (long long)pl->w);
        std::vector<float> v(T.minv_val.begin(), T.minv_val.end()), vT(T.minvT_val.begin(), T.minvT_val.end());
        cudaError_t e = upload(&pl->dt.lyn_idx, T.flat_index);
        if (e == cudaSuccess) e = upload(&pl->dt.rowptr, T.minv_rowptr);
        if (e == cudaSuccess) e = upload(&pl->dt.col, T.minv_col);
        if (e == cudaSuccess) e = upload(&pl->dt.val, v);
        if (e == cudaSuccess) e = upload(&pl->dt.rowptrT, T.minvT_rowptr);
        if (e == cudaSuccess) e = upload(&pl->dt.colT, T.minvT_col);
        if (e == cudaSuccess) e = upload(&pl->dt.valT, vT);
        if (e != cudaSuccess) {
            sig_logsig_plan_destroy(pl.release());
            return cuda_status(e, "logsig plan upload");
        }
    }
    *plan = pl.release();
    return ok();
}

sig_status_t sig_logsig_plan_destroy(sig_logsig_plan_t plan) {
    if (!plan) return ok();
    cudaFree(plan->dt.lyn_idx);
    cudaFree(plan->dt.rowptr);
    cudaFree(plan->dt.col);
    cudaFree(plan->dt.val);
    cudaFree(plan->dt.rowptrT);
    cudaFree(plan->dt.colT);
    cudaFree(plan->dt.valT);
    delete plan;
    return ok();
}

size_t sig_logsignature_workspace_size(sig_logsig_plan_t plan, int64_t B, int64_t L, int32_t stream,
                                       sig_basepoint_t bp) {
    if (!plan) return 0;
    FwdPlan pl;
    if (make_fwd_plan(B, L, plan->C, plan->N, stream, bp, pl) != SIG_OK) return 0;
    const int64_t rows = stream ? B * pl.M : B;
    // scan workspace | signature (if the caller gives no sig_saved) | dense dL/dlog and dL/dSig |
    // the reversible backward's own workspace (time chunks of long or few paths)
    size_t a = pl.ws_bytes;
    size_t b = (size_t)rows * plan->S * sizeof(float) * 3;
    size_t c = sig_signature_backward_ex_workspace_size(B, L, plan->C, plan->N, stream, bp, 0, 0, 0);
    return align256(a + b) + c;
}

sig_status_t sig_logsignature(sig_logsig_plan_t plan, const float* path, int64_t B, int64_t L, int32_t stream,
                              sig_basepoint_t bp, const float* basepoint, float* out, float* sig_saved, void* ws,
                              size_t ws_bytes, sig_cuda_stream_t s) {
    if (!plan) return fail(SIG_ERR_INVALID_ARG, "plan is NULL");
    if (!out) return fail(SIG_ERR_INVALID_ARG, "out is NULL");
    FwdPlan pl;
    sig_status_t st = make_fwd_plan(B, L, plan->C, plan->N, stream, bp, pl);
    if (st != SIG_OK) return st;
    const size_t need = sig_logsignature_workspace_size(plan, B, L, stream, bp);
    if (ws_bytes < need || (need > 0 && !ws))
        return fail(SIG_ERR_WORKSPACE, "workspace of %zu bytes needed, %zu given", need, ws_bytes);
    if (B == 0) return ok();
    const int64_t rows = stream ? B * pl.M : B;
    char* wsb = static_cast<char*>(ws);
    float* sig = sig_saved ? sig_saved : reinterpret_cast<float*>(wsb + pl.ws_bytes);
    st = run_signature(path, B, L, plan->C, plan->N, stream, bp, basepoint, sig, ws, pl.ws_bytes, (cudaStream_t)s);
    if (st != SIG_OK) return st;
    return launch_logsig_fwd(plan, sig, rows, out, (cudaStream_t)s);
}

sig_status_t sig_logsignature_backward(sig_logsig_plan_t plan, const float* grad_out, const float* path,
                                       const float* sig_saved, int64_t B, int64_t L, int32_t stream,
                                       sig_basepoint_t bp, const float* basepoint, float* grad_path,
                                       float* grad_basepoint, void* ws, size_t ws_bytes, sig_cuda_stream_t s) {
    if (!plan) return fail(SIG_ERR_INVALID_ARG, "plan is NULL");
    if (!grad_out || !path || !sig_saved || !grad_path)
        return fail(SIG_ERR_INVALID_ARG, "grad_out, path, sig_saved and grad_path must be non-null");
    FwdPlan pl;
    sig_status_t st = make_fwd_plan(B, L, plan->C, plan->N, stream, bp, pl);
    if (st != SIG_OK) return st;
    if (!pl.ks->bwd)
        return fail(SIG_ERR_UNSUPPORTED, "no sm_100a backward kernel for C=%d depth=%d", plan->C, plan->N);
    const size_t need = sig_logsignature_workspace_size(plan, B, L, stream, bp);
    if (ws_bytes < need || (need > 0 && !ws))
        return fail(SIG_ERR_WORKSPACE, "workspace of %zu bytes needed, %zu given", need, ws_bytes);
    if (B == 0) return ok();
    const int64_t rows = stream ? B * pl.M : B;
    char* wsb = static_cast<char*>(ws) + pl.ws_bytes;
    float* glog = reinterpret_cast<float*>(wsb) + (size_t)rows * plan->S;
    float* gsig = glog + (size_t)rows * plan->S;
    st = launch_logsig_bwd(plan, grad_out, sig_saved, rows, glog, gsig, (cudaStream_t)s);
    if (st != SIG_OK) return st;
    const size_t off = align256(pl.ws_bytes + (size_t)rows * plan->S * sizeof(float) * 3);
    return sig_signature_backward_ex(gsig, path, sig_saved, B, L, plan->C, plan->N, stream, bp, basepoint, 0, nullptr,
                                     grad_path, grad_basepoint, nullptr, static_cast<char*>(ws) + off, ws_bytes - off,
                                     s);
}

size_t sig_logsignature_from_signature_workspace_size(sig_logsig_plan_t plan, int64_t rows) {
    if (!plan || rows < 0) return 0;
    return (size_t)rows * plan->S * sizeof(float);
}

sig_status_t sig_logsignature_from_signature(sig_logsig_plan_t plan, const float* sig, int64_t rows, float* out,
                                             sig_cuda_stream_t s) {
    if (!plan) return fail(SIG_ERR_INVALID_ARG, "plan is NULL");
    if (rows < 0) return fail(SIG_ERR_SHAPE, "rows < 0");
    if (rows == 0) return ok();
    if (!sig || !out) return fail(SIG_ERR_INVALID_ARG, "sig and out must be non-null");
    return launch_logsig_fwd(plan, sig, rows, out, (cudaStream_t)s);
}

sig_status_t sig_logsignature_from_signature_backward(sig_logsig_plan_t plan, const float* grad_out, const float* sig,
                                                      int64_t rows, float* grad_sig, void* ws, size_t ws_bytes,
                                                      sig_cuda_stream_t s) {
    if (!plan) return fail(SIG_ERR_INVALID_ARG, "plan is NULL");
    if (rows < 0) return fail(SIG_ERR_SHAPE, "rows < 0");
    if (rows == 0) return ok();
    if (!grad_out || !sig || !grad_sig) return fail(SIG_ERR_INVALID_ARG, "grad_out, sig and grad_sig must be non-null");
    const size_t need = sig_logsignature_from_signature_workspace_size(plan, rows);
    if (ws_bytes < need || !ws) return fail(SIG_ERR_WORKSPACE, "workspace of %zu bytes needed, %zu given", need, ws_bytes);
    return launch_logsig_bwd(plan, grad_out, sig, rows, static_cast<float*>(ws), grad_sig, (cudaStream_t)s);
}

size_t sig_path_query_workspace_size(int64_t M, int64_t Q) {
    if (M < 0 || Q < 0) return 0;
    // starts, ends (int64) + two CSRs (int32: M+1 pointers, Q indices), 256-byte aligned pieces
    return align256(2 * (size_t)Q * sizeof(int64_t)) + 2 * align256(((size_t)M + 1 + (size_t)Q) * sizeof(int));
}

static sig_status_t check_queries(int64_t M, const int64_t* starts, const int64_t* ends, int64_t Q) {
    for (int64_t q = 0; q < Q; ++q) {
        if (starts[q] < 0 || ends[q] < starts[q] + 2 || ends[q] > M + 1)
            return fail(SIG_ERR_SHAPE, "query %lld = [%lld, %lld) is not an interval of >= 2 of the %lld points",
                        (long long)q, (long long)starts[q], (long long)ends[q], (long long)(M + 1));
    }
    return SIG_OK;
}

sig_status_t sig_path_query(const float* prefix_sig, const float* prefix_inv, int64_t B, int64_t M, int64_t C,
                            int32_t depth, const int64_t* starts, const int64_t* ends, int64_t Q, float* out, void* ws,
                            size_t ws_bytes, sig_cuda_stream_t s) {
    const int64_t S = sig_channels_checked(C, depth);
    if (S < 0 || C > 8) return fail(SIG_ERR_INVALID_ARG, "bad C=%lld depth=%d", (long long)C, depth);
    if (B < 0 || M < 1 || Q < 0) return fail(SIG_ERR_SHAPE, "B=%lld M=%lld Q=%lld", (long long)B, (long long)M, (long long)Q);
    if (Q > 0 && (!starts || !ends)) return fail(SIG_ERR_INVALID_ARG, "starts and ends must be non-null");
    sig_status_t st = check_queries(M, starts, ends, Q);
    if (st != SIG_OK) return st;
    if (B == 0 || Q == 0) return ok();
    if (!prefix_sig || !prefix_inv || !out) return fail(SIG_ERR_INVALID_ARG, "prefix_sig, prefix_inv and out must be non-null");
    const size_t need = sig_path_query_workspace_size(M, Q);
    if (ws_bytes < need || !ws) return fail(SIG_ERR_WORKSPACE, "workspace of %zu bytes needed, %zu given", need, ws_bytes);
    cudaStream_t cs = (cudaStream_t)s;
    int64_t* qs = static_cast<int64_t*>(ws);
    int64_t* qe = qs + Q;
    cudaError_t e = upload(qs, starts, Q * sizeof(int64_t), cs);
    if (e == cudaSuccess) e = upload(qe, ends, Q * sizeof(int64_t), cs);
    if (e != cudaSuccess) return cuda_status(e, "query upload");
    PathQueryParams p{};
    p.d = make_dims((int)C, depth);
    p.sig = prefix_sig;
    p.inv = prefix_inv;
    p.B = B;
    p.M = M;
    p.Q = Q;
    p.qs = qs;
    p.qe = qe;
    p.out = out;
    const int64_t n = B * Q * S;
    path_query_kernel<<<(unsigned)((n + 255) / 256), 256, 0, cs>>>(p);
    count_launch();
    return cuda_status(cudaGetLastError(), "path query launch");
}

sig_status_t sig_path_query_backward(const float* grad_out, const float* prefix_sig, const float* prefix_inv,
                                     int64_t B, int64_t M, int64_t C, int32_t depth, const int64_t* starts,
                                     const int64_t* ends, int64_t Q, float* grad_prefix_sig, float* grad_prefix_inv,
                                     void* ws, size_t ws_bytes, sig_cuda_stream_t s) {
    const int64_t S = sig_channels_checked(C, depth);
    if (S < 0 || C > 8) return fail(SIG_ERR_INVALID_ARG, "bad C=%lld depth=%d", (long long)C, depth);
    if (B < 0 || M < 1 || Q < 0) return fail(SIG_ERR_SHAPE, "B=%lld M=%lld Q=%lld", (long long)B, (long long)M, (long long)Q);
    if (Q > 0 && (!starts || !ends)) return fail(SIG_ERR_INVALID_ARG, "starts and ends must be non-null");
    sig_status_t st = check_queries(M, starts, ends, Q);
    if (st != SIG_OK) return st;
    if (B == 0) return ok();
    if (!prefix_sig || !prefix_inv || !grad_prefix_sig || !grad_prefix_inv || (Q > 0 && !grad_out))
        return fail(SIG_ERR_INVALID_ARG, "tensor pointers must be non-null");
    const size_t need = sig_path_query_workspace_size(M, Q);
    if (ws_bytes < need || !ws) return fail(SIG_ERR_WORKSPACE, "workspace of %zu bytes needed, %zu given", need, ws_bytes);
    // CSRs row -> queries (ascending), built on the host: the sums over queries then have a fixed order
    std::vector<int> sp(M + 1, 0), ip(M + 1, 0), sq(Q), iq(Q);
    int64_t ni = 0;
    for (int64_t q = 0; q < Q; ++q) {
        ++sp[ends[q] - 2 + 1];
        if (starts[q] > 0) ++ip[starts[q] - 1 + 1], ++ni;
    }
    for (int64_t r = 0; r < M; ++r) sp[r + 1] += sp[r], ip[r + 1] += ip[r];
    {
        std::vector<int> fs(sp.begin(), sp.end() - 1), fi(ip.begin(), ip.end() - 1);
        for (int64_t q = 0; q < Q; ++q) {
            sq[fs[ends[q] - 2]++] = (int)q;
            if (starts[q] > 0) iq[fi[starts[q] - 1]++] = (int)q;
        }
    }
    cudaStream_t cs = (cudaStream_t)s;
    char* w = static_cast<char*>(ws);
    int64_t* qs = reinterpret_cast<int64_t*>(w);
    int64_t* qe = qs + Q;
    int* csr_s = reinterpret_cast<int*>(w + align256(2 * (size_t)Q * sizeof(int64_t)));
    int* csr_i = reinterpret_cast<int*>(reinterpret_cast<char*>(csr_s) + align256(((size_t)M + 1 + Q) * sizeof(int)));
    cudaError_t e = upload(qs, starts, Q * sizeof(int64_t), cs);
    if (e == cudaSuccess) e = upload(qe, ends, Q * sizeof(int64_t), cs);
    if (e == cudaSuccess) e = upload(csr_s, sp.data(), (M + 1) * sizeof(int), cs);
    if (e == cudaSuccess) e = upload(csr_s + M + 1, sq.data(), Q * sizeof(int), cs);
    if (e == cudaSuccess) e = upload(csr_i, ip.data(), (M + 1) * sizeof(int), cs);
    if (e == cudaSuccess) e = upload(csr_i + M + 1, iq.data(), ni * sizeof(int), cs);
    if (e != cudaSuccess) return cuda_status(e, "query upload");
    PathQueryParams p{};
    p.d = make_dims((int)C, depth);
    p.sig = prefix_sig;
    p.inv = prefix_inv;
    p.B = B;
    p.M = M;
    p.Q = Q;
    p.qs = qs;
    p.qe = qe;
    p.gout = grad_out;
    p.sig_ptr = csr_s;
    p.sig_q = csr_s + M + 1;
    p.inv_ptr = csr_i;
    p.inv_q = csr_i + M + 1;
    p.gsig = grad_prefix_sig;
    p.ginv = grad_prefix_inv;
    const int64_t n = B * M * S;
    path_query_bwd_kernel<<<(unsigned)((n + 255) / 256), 256, 0, cs>>>(p);
    count_launch();
    return cuda_status(cudaGetLastError(), "path query backward launch");
}

}  // extern "C"
