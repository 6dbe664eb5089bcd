// sig_bwd.cuh -- K2: reversible backward of the signature, sm_100a.
//
// Method: Appendix C.  Walking t = M-1 .. 0 with the state A' = Sig after step t:
//   (1) reversibility (eq-reverse): A = A' [x] exp(-z_t), the same fused Horner update
//       with the increment negated.  Only levels < N are rebuilt: the VJP never reads A_N.
//   (2) recompute the Horner chains of eq-fusedterm from A:
//       B^(k)_0 = 1,  B^(k)_i = B^(k)_{i-1} (x) z/(k-i+1) + A_i.
//   (3) VJP of the chains, k = 1..N bottom-up so the incoming gradient G'_k is read before any
//       chain k' > k adds into it:  beta <- G'_k;  for i = k..1 (s = k-i+1):
//         gz[c] += (1/s) sum_w B_{i-1}[w] beta[w c];   beta <- (1/s) sum_c beta[. c] z_c;
//         G_{i-1} += beta  (i >= 2)
//   (4) grad x_{t+1} += gz, grad x_t -= gz.
// The top-level gradient G_N is never modified (it is constant over all steps).
//
// B200 design: one CTA per path, one thread per word prefix p of length P.
// * Levels >= P: the thread holds G and A for the words starting with p in registers and runs
//   (1)-(3) on them depth-first with no communication (as in the forward).
// * Levels < P: every operation there is LINEAR in the gradient.  So instead of reducing the
//   chain values beta_P[p] over threads every step, thread p keeps its own partial of the
//   low-level gradient, Ghat_i(p) with G_i[u] = sum_{p : p[:i] = u} Ghat_i(p), and runs the low
//   tails of all chains along its own prefix (it already holds the prefix chain values B_i[p[:i]]).
//   Its contributions to gz at level i land in channel p_{i-1}.  Grad-out coefficients of the low
//   levels are owned by the thread whose trailing prefix digits are zero.
// * The only collective per step is the C-vector gz: one warp reduce-scatter (channel = lane mod
//   C when C divides 32, which also absorbs the per-level scalars), then one float per warp and
//   channel into a shared-memory tile; every T steps the CTA sums the tile in a fixed order and
//   writes the gradient rows.  No cross-warp synchronisation inside a tile.
// All reductions have a fixed order, so results are bitwise reproducible.
// sig_bwd2_kernel (below) is the same algorithm with two sibling prefixes per thread, chosen for
// plain calls of shapes whose doubled state fits the register file.
#pragma once
#include "sig_fwd.cuh"

namespace sigb200 {

struct BwdParams {
    const float* grad_out;   // [B, S] | stream: [B, M, S]
    const float* path;       // [B, L, C]
    const float* basepoint;  // [B, C] (bp_mode == 2)
    const float* sig_final;  // forward output: [B, S] | stream: [B, M, S]
    int bp_mode, stream;
    int64_t B, L, M;
    float* grad_path;        // [B, L, C]
    float* grad_bp;          // [B, C] or nullptr
    int64_t sf_stride;       // floats between consecutive paths' final states in sig_final
    float zsign;             // +1, or -1: the forward scanned the negated path (inverse option)
    const float* initial;    // [B, S] start state of the forward scan, or nullptr (identity)
    float* grad_initial;     // [B, S] gradient w.r.t. initial, or nullptr
    // time-parallel backward: CTA u reverses chunk j = u % n_chunks of path
    // b = u / n_chunks, increments [j * chunk_len, min((j+1) * chunk_len, M)).  n_chunks = 1 is the
    // plain per-path backward.
    int64_t n_chunks, chunk_len;
    int64_t go_stride;       // floats between consecutive units' grad_out rows (non-stream)
    const float* chunk_init; // [B * n_chunks, S]: start state of chunk j >= 1 is row b * n_chunks + j - 1
    float* edge;             // [B * n_chunks, C]: chunk j >= 1 writes its first point's share here
    int tile;                // sig_bwd_kernel: steps per tile (set by launch_bwd from the occupancy)
    int64_t raw_off;         // > 0 (two-prefix kernels): the path's points are bulk-copied by TMA into
                             // shared memory at this float offset and the increments formed there
};

// Increments of one whole path into zbuf[M][C] (the two-prefix K2 kernels).  raw_off > 0: the
// 16-byte-aligned cover of the path's L points arrives by TMA bulk copies (cp.async.bulk, one
// mbarrier) and the increments are formed from shared memory; else coalesced loads from global.
// The caller synchronises the CTA afterwards.
template <int C>
__device__ __forceinline__ void stage_path_increments(const BwdParams& prm, int64_t bidx, int64_t M, float* zbuf,
                                                      float* smem_base, uint64_t* bar) {
    const int tid = threadIdx.x;
    const int has_bp = prm.bp_mode != 0;
    const float* xr = prm.path + bidx * prm.L * C;
    const float* base = xr;
    if (prm.raw_off > 0) {
        float* raw = smem_base + prm.raw_off;
        const uintptr_t a = reinterpret_cast<uintptr_t>(xr) & ~(uintptr_t)15;
        const uintptr_t e = (reinterpret_cast<uintptr_t>(xr + prm.L * C) + 15) & ~(uintptr_t)15;
        if (tid == 0) {
            mbar_init(bar, 1);
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(bar, (unsigned)(e - a));
            bulk_g2s_big(raw, reinterpret_cast<const void*>(a), e - a, bar);
        }
        __syncthreads();  // the barrier is initialised before anyone waits on it
        mbar_wait(bar, 0);
        base = raw + ((reinterpret_cast<uintptr_t>(xr) & 15) >> 2);
    }
    for (int64_t e = tid; e < M * C; e += blockDim.x) {
        const int64_t s = e / C;
        const int c = (int)(e % C);
        const int64_t r1 = s + 1 - has_bp, r0 = s - has_bp;
        const float x1 = base[r1 * C + c];
        const float x0 = (r0 >= 0) ? base[r0 * C + c] : ((prm.bp_mode == 2) ? prm.basepoint[bidx * C + c] : 0.0f);
        zbuf[e] = prm.zsign * (x1 - x0);
    }
}

// Per-step gz records are flushed every T steps (a CTA barrier each time).  With up to 256 steps
// per tile a c2/c4 path has a single flush, so the warps run the whole reversal without a barrier
// (c4's 255 steps: 128-step tiles 679 us, one 256-step tile 677 us).
#ifndef SIG_BWD_TMAX
#define SIG_BWD_TMAX 256
#endif
#ifndef SIG_BWD_TILE_KB
#define SIG_BWD_TILE_KB 160
#endif
// With two warps per SM sub-partition (the 8-warp CTAs of e.g. C=4, N=7), delaying one of them by
// about half a step at the start keeps their FMA-dense and latency-bound phases interleaved
// (measured: c4 backward -5%; with four warps per sub-partition it costs 7%, so it is off there).
#ifndef SIG_BWD_STAGGER
#define SIG_BWD_STAGGER 400
#endif

#ifndef SIG_BWD_GNS
#define SIG_BWD_GNS 0
#endif
// one-warp backward CTAs (small states, e.g. C=3, N=6) resident per SM (registers <= 64K / (32 n))
#ifndef SIG_BWD_WARP_CTAS
#define SIG_BWD_WARP_CTAS 16
#endif
#ifndef SIG_BWD_GNS_MAXKB
#define SIG_BWD_GNS_MAXKB 96
#endif
#ifndef SIG_BWD_GNS_MINB
#define SIG_BWD_GNS_MINB 2
#endif
// Dot products over channels in vjp_visit as scalar FFMA chains (no horizontal add per node; the
// default) or as FFMA2 on channel pairs plus one FADD.  Measured (same-run A/B): c5's time-chunked
// backward (C = 3, odd: pairs + a scalar + the add) 1762 -> 1661 us, c4's backward 683 -> 680 us.
#ifndef SIG_BWD_SDOT
#define SIG_BWD_SDOT 1
#endif
template <class SH>
struct BwdLayout {
    static constexpr int C = SH::C, N = SH::N, P = SH::P;
    static constexpr int HW = (SH::CP + 31) / 32;  // warps
    static constexpr int NT = HW * 32;
    // warp-shuffle reduction applies when C is a power of two dividing 32 and the warps are full
    static constexpr bool FAST = (32 % C == 0) && ((C & (C - 1)) == 0) && (SH::CP % 32 == 0);
    static constexpr int PL = P > 0 ? P : 1;
    // floats per record: FAST, one per warp and channel; else one C-vector per thread (the thread
    // folds its low-level channel partials into their channels before writing)
    static constexpr int REC = C;
    // one-warp CTAs (e.g. C=3, N=6 with 27 prefixes) run as time chunks of long paths: ask for 16
    // resident per SM (<= 128 registers), the latency of one warp's reversal hidden by the others
    // GNS: the constant top-level gradient G_N lives in shared memory, not in registers (each
    // thread's block of C^(N-P) floats stored as float4 columns, [j/4][thread][4], conflict-free):
    // frees C^(N-P) registers per thread so that two CTAs fit per SM (plain and chunked calls,
    // not stream mode).  Each G_N value feeds two FMAs per step (gz and beta), one LDS.128 per four.
    static constexpr bool GNS = SIG_BWD_GNS && (C % 4 == 0) && (SH::own(N) >= 16) && (SH::CP % 32 == 0) &&
                                (SH::P > 0) && ((size_t)NT * SH::own(N) * 4 <= SIG_BWD_GNS_MAXKB * 1024);
    static constexpr int GNF = GNS ? NT * SH::own(N) : 0;  // floats of the G_N region
    static constexpr int MINB = (NT == 32 && SH::OWN + SH::OWNA <= 64) ? SIG_BWD_WARP_CTAS : (GNS ? SIG_BWD_GNS_MINB : 1);
    static constexpr int RECS = FAST ? HW : NT;      // records per step
    // shared memory of a tile of T steps: the tile's increments, T + 1 record slots, the per-step
    // totals, gprev, and the low-level partials of grad_initial
    __host__ __device__ static size_t smem_bytes_tile(int T) {
        return ((size_t)(T * C + 3) / 4 * 4 + (size_t)(T + 1) * RECS * REC + (size_t)T * C + 32 + (size_t)PL * NT) *
               sizeof(float);
    }
    // Largest power-of-two tile (<= SIG_BWD_TMAX, <= M) whose shared memory fits `budget` bytes.
    // The increments are staged per tile, so the chunk length does not enter: any path fits.
    static int tile(int64_t M, size_t budget) {
        int T = SIG_BWD_TMAX;
        while (T > 1 && smem_bytes_tile(T) > budget) T >>= 1;
        return (int)(T < M ? T : (M > 0 ? M : 1));
    }
};
// VJP of the level-K Horner chain, depth-first over the thread's word tree (post-order).
// Node (I, W) with chain value BI = B_I[p.W] returns beta_I[p.W] = (1/s) sum_c beta_{I+1}[p.W.c] z_c
// (s = K-I), after adding the level-(I+1) gz contributions (1/s) B_I[p.W] beta_{I+1}[p.W.c] and
// G_I += beta_I for owned levels I < K.  The leaves are beta_K = G_K (read before any chain
// k' > K adds into it: chains run bottom-up).
// GNS (top chain only): the leaves G_N[p.W.c] come from shared memory, gns = the thread's column
// (element j of its block at gns[(j/4) * 4 NT + j%4]).
template <class SH, int K, int I, int W, int SA, bool GNS = false>
__device__ __forceinline__ float vjp_visit(float BI, float (&G)[SH::OWN], const float (&A)[SA], const float (&z)[SH::C],
                                           float (&gz)[SH::C], const float* gns = nullptr) {
    // channel pairs with the packed FFMA2 (see horner_visit): gz += bs * x and acc += x * z
    constexpr int C = SH::C;
    constexpr float sc = inv_int(K - I);
    const float bs = BI * sc;
    const float2 bs2 = make_float2(bs, bs);
    float2 acc2 = make_float2(0.0f, 0.0f);
    float gl[(GNS && I + 1 == K) ? C : 1];
    if constexpr (GNS && I + 1 == K) {
        static_for<0, C / 4>([&](auto qq) {
            constexpr int q = decltype(qq)::value;
            constexpr int j = W * C + 4 * q;
            const float4 v = *reinterpret_cast<const float4*>(gns + (j / 4) * (4 * BwdLayout<SH>::NT));
            gl[4 * q] = v.x;
            gl[4 * q + 1] = v.y;
            gl[4 * q + 2] = v.z;
            gl[4 * q + 3] = v.w;
        });
    }
    static_for<0, C / 2>([&](auto cc) {
        constexpr int c = 2 * decltype(cc)::value;
        constexpr int ch = W * C + c;
        const float2 z2 = make_float2(z[c], z[c + 1]);
        float2 x;
        if constexpr (I + 1 == K) {
            if constexpr (GNS) x = make_float2(gl[c], gl[c + 1]);
            else x = make_float2(G[SH::own_off(K) + ch], G[SH::own_off(K) + ch + 1]);
        } else {
            constexpr int o = SH::own_off(I + 1) + ch;
            const float2 Bc = __ffma2_rn(bs2, z2, make_float2(A[o], A[o + 1]));
            x.x = vjp_visit<SH, K, I + 1, ch, SA, GNS>(Bc.x, G, A, z, gz, gns);
            x.y = vjp_visit<SH, K, I + 1, ch + 1, SA, GNS>(Bc.y, G, A, z, gz, gns);
        }
        const float2 g2 = __ffma2_rn(bs2, x, make_float2(gz[c], gz[c + 1]));
        gz[c] = g2.x;
        gz[c + 1] = g2.y;
        if constexpr (SIG_BWD_SDOT) {
            acc2.x = fmaf(x.x, z2.x, acc2.x);
            acc2.x = fmaf(x.y, z2.y, acc2.x);
        } else {
            acc2 = __ffma2_rn(x, z2, acc2);
        }
    });
    float acc = SIG_BWD_SDOT ? acc2.x : acc2.x + acc2.y;
    if constexpr (C % 2 == 1) {
        constexpr int c = C - 1;
        constexpr int ch = W * C + c;
        float x;
        if constexpr (I + 1 == K) {
            x = G[SH::own_off(K) + ch];
        } else {
            const float Bc = fmaf(bs, z[c], A[SH::own_off(I + 1) + ch]);
            x = vjp_visit<SH, K, I + 1, ch>(Bc, G, A, z, gz);
        }
        gz[c] = fmaf(bs, x, gz[c]);
        acc = fmaf(x, z[c], acc);
    }
    const float beta = acc * sc;
    if constexpr (I >= SH::K0) G[SH::own_off(I) + W] += beta;
    return beta;
}

// Fused VJP walk of the two top chains K = N-1 and K = N from node (I, W), P <= I <= N-2, carrying
// both chain values b1 = B^(N-1)_I[p.W] and b2 = B^(N)_I[p.W]; returns beta1 = beta^(N-1)_I[p.W] and
// beta2 = beta^(N)_I[p.W] and adds both to G_I (owned levels).  Same arithmetic as two vjp_visit
// walks, reorganised at the level-(N-2) nodes so that no horizontal add and no separate
// "G_{N-1} += beta_{N-1}" remain:
//   * chain N's level-(N-1) betas are accumulated straight into G_{N-1} (beta_{N-1}[Wc] =
//     sum_c' G_N[Wc c'] z_c' is a scalar FFMA chain seeded with G_{N-1}[Wc]);
//   * chain N-1 must read G_{N-1} before that update (chains run bottom-up), and chain N's
//     contributions at node W need beta_{N-1} = G_new - G_old, so the node's gz terms are
//     bs1 G_old + bs2 (G_new - G_old) = (bs1 - bs2) G_old + bs2 G_new, and
//     sum_c beta_{N-1}[Wc] z_c = sum_c G_new[Wc] z_c - sum_c G_old[Wc] z_c.
// Dot products over channels are scalar FFMA chains (an FFMA2 dot product needs a horizontal add,
// which costs an FP32 pipe cycle); the rank-1 gz updates are FFMA2 on channel pairs.
template <class SH, int I, int W, int SA>
__device__ __forceinline__ void vjp_top2(float b1, float b2, float (&G)[SH::OWN], const float (&A)[SA],
                                         const float (&z)[SH::C], float (&gz)[SH::C], float& beta1, float& beta2) {
    constexpr int C = SH::C, N = SH::N;
    constexpr float s1 = inv_int(N - 1 - I), s2 = inv_int(N - I);
    const float bs1 = (N - 1 - I == 1) ? b1 : b1 * s1;
    const float bs2 = b2 * s2;
    if constexpr (I == N - 2) {
        constexpr int o1 = SH::own_off(N - 1) + W * C;  // G_{N-1}[W c] and A_{N-1}[W c]
        constexpr int oN = SH::own_off(N) + W * C * C;  // G_N[W c c']
        // chain N-1 at this node, on the old G_{N-1}
        const float d = bs1 - bs2;
        const float2 d2 = make_float2(d, d);
        float acc1 = 0.0f;
        static_for<0, C / 2>([&](auto cc) {
            constexpr int c = 2 * decltype(cc)::value;
            const float2 g2 = __ffma2_rn(d2, make_float2(G[o1 + c], G[o1 + c + 1]), make_float2(gz[c], gz[c + 1]));
            gz[c] = g2.x;
            gz[c + 1] = g2.y;
        });
        if constexpr (C % 2 == 1) gz[C - 1] = fmaf(d, G[o1 + C - 1], gz[C - 1]);
        static_for<0, C>([&](auto cc) {
            constexpr int c = decltype(cc)::value;
            acc1 = fmaf(G[o1 + c], z[c], acc1);
        });
        // chain N: the level-(N-1) chain values of the children, B_c = bs2 z_c + A_{N-1}[W c]
        float Bc[C];
        const float2 bs22 = make_float2(bs2, bs2);
        static_for<0, C / 2>([&](auto cc) {
            constexpr int c = 2 * decltype(cc)::value;
            const float2 r = __ffma2_rn(bs22, make_float2(z[c], z[c + 1]), make_float2(A[o1 + c], A[o1 + c + 1]));
            Bc[c] = r.x;
            Bc[c + 1] = r.y;
        });
        if constexpr (C % 2 == 1) Bc[C - 1] = fmaf(bs2, z[C - 1], A[o1 + C - 1]);
        // the top level: gz[c'] += B_c G_N[W c c'] (FFMA2 over c' pairs); G_{N-1}[W c] += sum_c' G_N[W c c'] z_c'
        static_for<0, C>([&](auto cc) {
            constexpr int c = decltype(cc)::value;
            const float2 b2c = make_float2(Bc[c], Bc[c]);
            static_for<0, C / 2>([&](auto qq) {
                constexpr int q = 2 * decltype(qq)::value;
                const float2 g2 = __ffma2_rn(b2c, make_float2(G[oN + c * C + q], G[oN + c * C + q + 1]),
                                             make_float2(gz[q], gz[q + 1]));
                gz[q] = g2.x;
                gz[q + 1] = g2.y;
            });
            if constexpr (C % 2 == 1) gz[C - 1] = fmaf(Bc[c], G[oN + c * C + C - 1], gz[C - 1]);
            float g = G[o1 + c];
            static_for<0, C>([&](auto qq) {
                constexpr int q = decltype(qq)::value;
                g = fmaf(G[oN + c * C + q], z[q], g);
            });
            G[o1 + c] = g;
        });
        // chain N at this node, on the new G_{N-1}
        float acc2 = -acc1;
        static_for<0, C / 2>([&](auto cc) {
            constexpr int c = 2 * decltype(cc)::value;
            const float2 g2 = __ffma2_rn(bs22, make_float2(G[o1 + c], G[o1 + c + 1]), make_float2(gz[c], gz[c + 1]));
            gz[c] = g2.x;
            gz[c + 1] = g2.y;
        });
        if constexpr (C % 2 == 1) gz[C - 1] = fmaf(bs2, G[o1 + C - 1], gz[C - 1]);
        static_for<0, C>([&](auto cc) {
            constexpr int c = decltype(cc)::value;
            acc2 = fmaf(G[o1 + c], z[c], acc2);
        });
        beta1 = acc1;  // s1 = 1
        beta2 = acc2 * s2;
    } else {
        float acc1 = 0.0f, acc2 = 0.0f;
        static_for<0, C>([&](auto cc) {
            constexpr int c = decltype(cc)::value;
            constexpr int o = SH::own_off(I + 1) + W * C + c;
            float x1, x2;
            vjp_top2<SH, I + 1, W * C + c>(fmaf(bs1, z[c], A[o]), fmaf(bs2, z[c], A[o]), G, A, z, gz, x1, x2);
            gz[c] = fmaf(bs1, x1, fmaf(bs2, x2, gz[c]));
            acc1 = fmaf(x1, z[c], acc1);
            acc2 = fmaf(x2, z[c], acc2);
        });
        beta1 = acc1 * s1;
        beta2 = acc2 * s2;
    }
    if constexpr (I >= SH::K0) G[SH::own_off(I) + W] += beta1 + beta2;
}

// Prefix chain of chain K: Bp[j] = B^(K)_j[p[:j]] for j = 1..min(K-1, P) (Bp[0] = 1).
template <class SH, int K, int SA>
__device__ __forceinline__ void prefix_chain_all(float (&Bp)[SH::PL1], const float (&A)[SA], const float (&low)[SH::LOWA],
                                                 const float (&zp)[SH::PD]) {
    constexpr int P = SH::P;
    constexpr int J = (K - 1 < P) ? K - 1 : P;
    Bp[0] = 1.0f;
    static_for<1, J + 1>([&](auto jc) {
        constexpr int j = decltype(jc)::value;
        float Aj;
        if constexpr (j < P) Aj = low[j];
        else Aj = A[SH::own_off(P)];
        if constexpr (j == 1) Bp[j] = fmaf(zp[0], inv_int(K), Aj);
        else Bp[j] = fmaf(Bp[j - 1] * inv_int(K - j + 1), zp[j - 1], Aj);
    });
}

// Low tail of chain K from level I0 (<= P) down to 1 along the thread's prefix, on the partial
// b = beta_{I0}(p): level-i gz contributions go to acc[i] (channel p_{i-1}); partials of
// beta_{i-1} are added to Gh[i-1].
template <class SH, int K, int I0>
__device__ __forceinline__ void low_tail(float b, const float (&Bp)[SH::PL1], const float (&zp)[SH::PD],
                                         float (&acc)[SH::PL1], float (&Gh)[SH::LOWA]) {
    static_for<0, I0>([&](auto iic) {
        constexpr int i = I0 - decltype(iic)::value;  // I0 .. 1
        constexpr float sc = inv_int(K - i + 1);
        acc[i] = fmaf(Bp[i - 1] * sc, b, acc[i]);
        if constexpr (i >= 2) {
            b = b * zp[i - 1] * sc;
            Gh[i - 1] += b;
        }
    });
}

// STREAM (a template flag so that the plain kernel carries no stream-mode register pressure):
// the gradient w.r.t. every prefix signature, grad_out[t], is added before step t is reversed.
template <class SH, bool STREAM>
__global__ void __launch_bounds__(BwdLayout<SH>::NT, BwdLayout<SH>::MINB) sig_bwd_kernel(const BwdParams prm) {
    using LY = BwdLayout<SH>;
    constexpr int C = SH::C, N = SH::N, P = SH::P;
    constexpr int HW = LY::HW;
    constexpr int64_t S = SH::S;
    extern __shared__ __align__(16) float sm_base[];
    constexpr bool GNS = LY::GNS && !STREAM;
    float* const gn = sm_base;                                   // GNS: [own(N)/4][NT][4] G_N columns
    float* const sm = sm_base + (GNS ? LY::GNF : 0);
    const int64_t unit = blockIdx.x;
    const int64_t bidx = unit / prm.n_chunks;            // path
    const int64_t jc = unit - bidx * prm.n_chunks;       // time chunk
    const int64_t s0 = jc * prm.chunk_len;               // its first increment
    const int64_t M = (prm.chunk_len < prm.M - s0) ? prm.chunk_len : prm.M - s0;  // its increments
    const int T = prm.tile;
    float* zbuf = sm;                                        // [T][C] increments of the current tile
    float* part = zbuf + (T * C + 3) / 4 * 4;                // [1 + T][RECS][REC] per-step partials
    float* tot = part + (size_t)(T + 1) * LY::RECS * LY::REC;  // [T][C] per-step gz totals
    float* gprev = tot + (size_t)T * C;                      // [C] gz of the step processed before
    float* lowred = gprev + 32;                              // [P-1][NT] low-level partials (grad_initial)

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int has_bp = prm.bp_mode != 0;
    const float* sigrow = prm.sig_final + (size_t)unit * prm.sf_stride;  // state after this unit

    // increments of tile steps j = 0..tn-1 (step t = M-1-(n0+j)) into zbuf[j][c]; the caller
    // synchronises.  Staged per tile, so shared memory does not grow with the chunk length.
    const float* xr = prm.path + bidx * prm.L * C;
    auto stage_tile = [&](int64_t n0, int tn) {
        for (int e = tid; e < tn * C; e += blockDim.x) {
            const int j = e / C, c = e % C;
            const int64_t s = s0 + (M - 1 - (n0 + j));
            const int64_t r1 = s + 1 - has_bp, r0 = s - has_bp;
            const float x1 = __ldg(xr + r1 * C + c);
            const float x0 = (r0 >= 0) ? __ldg(xr + r0 * C + c) : ((prm.bp_mode == 2) ? prm.basepoint[bidx * C + c] : 0.0f);
            zbuf[e] = prm.zsign * (x1 - x0);
        }
    };
    if (tid < C) gprev[tid] = 0.0f;

    const bool valid = tid < SH::CP;
    const int prefix = valid ? tid : 0;
    int p[SH::PD];
    prefix_digits<SH>(prefix, p);
    float A[SH::OWNA];     // owned levels K0..N-1 of the current state
    float G[SH::OWN];      // owned levels K0..N of the gradient
    float low[SH::LOWA];   // A_i[p[:i]], i < P
    float Gh[SH::LOWA];    // partial low-level gradients Ghat_i(p), i < P
    static_for<SH::K0, N>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        load_run<SH::own(k), SH::own_off(k)>(A, sigrow + SH::lvl_off(k) + (int64_t)prefix * SH::own(k));
    });
    const float* gns = gn + 4 * tid;
    static_for<SH::K0, N + 1>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        if constexpr (GNS && k == N) {
            // the thread's own column: written and read by this thread only (no barrier needed)
            float tmp[SH::own(N)];
            if (valid) {
                load_run<SH::own(N), 0>(tmp, prm.grad_out + (size_t)unit * prm.go_stride + SH::lvl_off(N) +
                                                 (int64_t)prefix * SH::own(N));
            } else {
#pragma unroll
                for (int q = 0; q < SH::own(N); ++q) tmp[q] = 0.0f;
            }
#pragma unroll
            for (int q = 0; q < SH::own(N) / 4; ++q)
                *reinterpret_cast<float4*>(gn + q * 4 * LY::NT + 4 * tid) =
                    make_float4(tmp[4 * q], tmp[4 * q + 1], tmp[4 * q + 2], tmp[4 * q + 3]);
        } else if (STREAM || !valid) {
#pragma unroll
            for (int q = 0; q < SH::own(k); ++q) G[SH::own_off(k) + q] = 0.0f;
        } else {
            load_run<SH::own(k), SH::own_off(k)>(G, prm.grad_out + (size_t)unit * prm.go_stride + SH::lvl_off(k) +
                                                        (int64_t)prefix * SH::own(k));
        }
    });
    low[0] = 0.0f;
    Gh[0] = 0.0f;
    // the low-level gradient coefficient u = p[:i] is owned by the thread with p[i:] == 0
    static_for<1, P>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        constexpr int tail = (int)ipow(C, P - i);
        low[i] = sigrow[SH::lvl_off(i) + prefix / tail];
        Gh[i] = (!STREAM && valid && prefix % tail == 0)
                    ? prm.grad_out[(size_t)unit * prm.go_stride + SH::lvl_off(i) + prefix / tail]
                    : 0.0f;
    });
    __syncthreads();
    if (SIG_BWD_STAGGER > 0 && HW == 8 && ((warp >> 2) & 1)) __nanosleep(SIG_BWD_STAGGER);

    auto grad_row = [&](int64_t r) -> float* {
        // augmented point r (r == 0 is the basepoint when one is given)
        if (has_bp) {
            if (r == 0) return (prm.bp_mode == 2 && prm.grad_bp) ? prm.grad_bp + bidx * C : nullptr;
            return prm.grad_path + (bidx * prm.L + (r - 1)) * C;
        }
        return prm.grad_path + (bidx * prm.L + r) * C;
    };

    // one reversed step t: (1) reversibility A <- A [x] exp(-z) on levels < N (FIRST: the exact start
    // state at t == 0 instead), (2)+(3) chains k = 1..N bottom-up; leaves gz and the low-level
    // channel partials acc[i] (channel p_{i-1})
    auto stream_add = [&](int64_t t) {
        if (STREAM && valid) {
            const float* gr = prm.grad_out + ((size_t)bidx * prm.M + s0 + t) * S;  // stream: one chunk
            static_for<SH::K0, N + 1>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                add_run<SH::own(k), SH::own_off(k)>(G, gr + SH::lvl_off(k) + (int64_t)prefix * SH::own(k));
            });
            static_for<1, P>([&](auto ic) {
                constexpr int i = decltype(ic)::value;
                constexpr int tail = (int)ipow(C, P - i);
                if (prefix % tail == 0) Gh[i] += gr[SH::lvl_off(i) + prefix / tail];
            });
        }
    };
    auto load_z = [&](int j, float (&z)[C], float (&zp)[SH::PD]) {  // tile step j
#pragma unroll
        for (int c = 0; c < C; ++c) z[c] = zbuf[j * C + c];
#pragma unroll
        for (int q = 0; q < SH::PD; ++q) zp[q] = (P > 0) ? zbuf[j * C + p[q]] : 0.0f;
    };
    // the exact start state at t == 0: the product of the earlier chunks, the user's initial, or 1
    auto start_state = [&]() {
        if (jc > 0 || prm.initial != nullptr) {
            const float* ir = (jc > 0) ? prm.chunk_init + (size_t)(unit - 1) * S : prm.initial + (size_t)bidx * S;
            static_for<SH::K0, N>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                load_run<SH::own(k), SH::own_off(k)>(A, ir + SH::lvl_off(k) + (int64_t)prefix * SH::own(k));
            });
            static_for<1, P>([&](auto ic) {
                constexpr int i = decltype(ic)::value;
                low[i] = ir[SH::lvl_off(i) + prefix / (int)ipow(C, P - i)];
            });
        } else {
#pragma unroll
            for (int q = 0; q < SH::OWNA; ++q) A[q] = 0.0f;
#pragma unroll
            for (int q = 0; q < SH::LOWA; ++q) low[q] = 0.0f;
        }
    };
    // (2)+(3): chains k = 1..N bottom-up on the rebuilt state; leaves gz and the low-level channel
    // partials acc[i] (channel p_{i-1}).  Split in two (k < N, then k = N) so that the caller can
    // place work in between.
    auto chains_lower = [&](const float (&z)[C], const float (&zp)[SH::PD], float (&gz)[C], float (&acc)[SH::PL1]) {
#pragma unroll
        for (int c = 0; c < C; ++c) gz[c] = 0.0f;
#pragma unroll
        for (int q = 0; q < SH::PL1; ++q) acc[q] = 0.0f;
        // chains entirely below P: read Ghat_k, tail from level k
        static_for<1, (P < N ? P : N)>([&](auto kc) {
            constexpr int k = decltype(kc)::value;
            float Bp[SH::PL1];
            prefix_chain_all<SH, k>(Bp, A, low, zp);
            low_tail<SH, k, k>(Gh[k], Bp, zp, acc, Gh);
        });
        // chains max(P,1) <= k < N: owned levels depth-first, then the low tail from level P
        static_for<SH::K0, N>([&](auto kc) {
            constexpr int k = decltype(kc)::value;
            float Bp[SH::PL1];
            prefix_chain_all<SH, k>(Bp, A, low, zp);
            float bP;
            if constexpr (k == P) bP = G[SH::own_off(P)];
            else bP = vjp_visit<SH, k, P, 0>(Bp[P], G, A, z, gz);
            if constexpr (P >= 1) low_tail<SH, k, P>(bP, Bp, zp, acc, Gh);
        });
    };
    auto chain_top = [&](const float (&z)[C], const float (&zp)[SH::PD], float (&gz)[C], float (&acc)[SH::PL1]) {
        constexpr int k = N;
        float Bp[SH::PL1];
        prefix_chain_all<SH, k>(Bp, A, low, zp);
        float bP;
        if constexpr (k == P) bP = G[SH::own_off(P)];
        else bP = vjp_visit<SH, k, P, 0, SH::OWNA, GNS>(Bp[P], G, A, z, gz, gns);
        if constexpr (P >= 1) low_tail<SH, k, P>(bP, Bp, zp, acc, Gh);
    };

    // per-step gz of tile step j into record slot j + 1 (slot 0: dummy), in three stages so that
    // the caller can spread them over the next step's arithmetic.  FAST: rv[] holds the
    // reduce-scatter state (lane l ends with channel l % C summed over its group of C lanes).
    auto reduce_a = [&](float (&v)[C]) {
        if constexpr (LY::FAST) {
            static_for<0, ilog2(C)>([&](auto sc_) {
                constexpr int m = C >> (decltype(sc_)::value + 1);  // C/2, C/4, .., 1
                const bool up = (lane & m) != 0;
#pragma unroll
                for (int q = 0; q < m; ++q) {
                    const float send = up ? v[q] : v[q + m];
                    const float keep = up ? v[q + m] : v[q];
                    v[q] = keep + __shfl_xor_sync(0xffffffffu, send, m);
                }
            });
        }
    };
    auto reduce_b = [&](const float (&v)[C], const float (&acc)[SH::PL1]) -> float {
        float tv = 0.0f;
        if constexpr (LY::FAST) {
            tv = v[0];
            if constexpr (P >= 1) tv += acc[P];  // its channel p_{P-1} is lane % C
            static_for<1, P>([&](auto ic) {
                constexpr int i = decltype(ic)::value;  // channel p_{i-1}: constant over the group
                float gsum = acc[i];
#pragma unroll
                for (int m = 1; m < C; m <<= 1) gsum += __shfl_xor_sync(0xffffffffu, gsum, m);
                if ((lane % C) == p[i - 1]) tv += gsum;
            });
        }
        return tv;
    };
    auto reduce_c = [&](float tv, const float (&v)[C], const float (&acc)[SH::PL1], int j) {
        float* rec = part + (size_t)(j + 1) * LY::RECS * LY::REC;
        if constexpr (LY::FAST) {
#pragma unroll
            for (int m = C; m < 32; m <<= 1) tv += __shfl_xor_sync(0xffffffffu, tv, m);
            if (lane < C) rec[warp * C + lane] = tv;
        } else {
            float* r = rec + (size_t)tid * LY::REC;
#pragma unroll
            for (int c = 0; c < C; ++c) {
                float vc = v[c];
                static_for<1, P + 1>([&](auto ic) {  // acc[i] belongs to channel p_{i-1}
                    constexpr int i = decltype(ic)::value;
                    if (p[i - 1] == c) vc += acc[i];
                });
                r[c] = valid ? vc : 0.0f;
            }
        }
    };

    for (int64_t n0 = 0; n0 < M; n0 += T) {
        const int tn = (int)((M - n0) < T ? (M - n0) : T);
        stage_tile(n0, tn);
        __syncthreads();
        // Software pipelining: the gz reduction of step j is issued at the top of step j+1, in the
        // same basic block as that step's arithmetic, so its shuffle latency overlaps the FMAs
        // (the reduction is independent of the next step's state).  The step with t == 0 (exact
        // start state instead of the reversal) is peeled out of the loop to keep the body one
        // block.  rec slot 0 is a dummy that absorbs the reduction of the zero vector at j = 0.
        const bool last_tile = n0 + tn == M;  // holds the step t == 0
        const int jn = last_tile ? tn - 1 : tn;
        float gz[C], acc[SH::PL1];
#pragma unroll
        for (int c = 0; c < C; ++c) gz[c] = 0.0f;
#pragma unroll
        for (int q = 0; q < SH::PL1; ++q) acc[q] = 0.0f;
        for (int j = 0; j < jn; ++j) {
            const int64_t t = M - 1 - (n0 + j);
            if constexpr (STREAM) {
                // stream mode adds a grad_out row per step: no room to carry the previous gz
                // through the step, reduce it first
                float v[C];
#pragma unroll
                for (int c = 0; c < C; ++c) v[c] = gz[c];
                reduce_a(v);
                reduce_c(reduce_b(v, acc), v, acc, j - 1);
                stream_add(t);
                float z[C], zp[SH::PD];
                load_z(j, z, zp);
                fused_mulexp<SH, N - 1, true>(A, low, z, zp);
                chains_lower(z, zp, gz, acc);
                chain_top(z, zp, gz, acc);
                continue;
            }
            stream_add(t);
            float z[C], zp[SH::PD];
            load_z(j, z, zp);
            float v[C], ac[SH::PL1];  // previous step's gz, reduced while this step computes
#pragma unroll
            for (int c = 0; c < C; ++c) v[c] = gz[c];
#pragma unroll
            for (int q = 0; q < SH::PL1; ++q) ac[q] = acc[q];
            reduce_a(v);
            fused_mulexp<SH, N - 1, true>(A, low, z, zp);  // (1) reversibility, levels < N
            const float tv = reduce_b(v, ac);
            chains_lower(z, zp, gz, acc);
            reduce_c(tv, v, ac, j - 1);
            chain_top(z, zp, gz, acc);
        }
        if (last_tile) {
            float v[C];
#pragma unroll
            for (int c = 0; c < C; ++c) v[c] = gz[c];
            reduce_a(v);
            reduce_c(reduce_b(v, acc), v, acc, tn - 2);
            stream_add(0);
            float z[C], zp[SH::PD];
            load_z(tn - 1, z, zp);
            start_state();
            chains_lower(z, zp, gz, acc);
            chain_top(z, zp, gz, acc);
        }
        {
            float v[C];
#pragma unroll
            for (int c = 0; c < C; ++c) v[c] = gz[c];
            reduce_a(v);
            reduce_c(reduce_b(v, acc), v, acc, tn - 1);
        }
        // ---- flush: per-step totals in a fixed order, then the gradient rows
        __syncthreads();
        for (int e = tid; e < tn * C; e += blockDim.x) {
            const int j = e / C, c = e % C;
            const float* rec = part + (size_t)(j + 1) * LY::RECS * LY::REC;
            float s = 0.0f;
            if constexpr (LY::FAST) {
                for (int w = 0; w < HW; ++w) s += rec[w * C + c];
            } else {
                for (int th = 0; th < SH::CP; ++th) s += rec[(size_t)th * LY::REC + c];
            }
            tot[j * C + c] = s;
        }
        __syncthreads();
        for (int e = tid; e < tn * C; e += blockDim.x) {
            const int j = e / C, c = e % C;
            const int64_t t = M - 1 - (n0 + j);
            const float before = (j == 0) ? gprev[c] : tot[(j - 1) * C + c];
            float* gr = grad_row(s0 + t + 1);
            if (gr) gr[c] = prm.zsign * (tot[j * C + c] - before);  // grad x_{t+1} = gz_t - gz_{t+1}
            if (t == 0) {
                if (jc == 0) {
                    float* g0 = grad_row(0);
                    if (g0) g0[c] = -prm.zsign * tot[j * C + c];
                } else {  // the point shared with the previous chunk: added by the fix-up kernel
                    prm.edge[unit * C + c] = -prm.zsign * tot[j * C + c];
                }
            }
        }
        __syncthreads();
        if (tid < C) gprev[tid] = tot[(tn - 1) * C + tid];
        __syncthreads();
    }
    if (prm.grad_initial != nullptr && jc == 0) {
        // G now holds dL/d(start state): owned levels directly; a level i < P coefficient u is the
        // fixed-order sum of the partials Ghat_i(p) over the C^(P-i) prefixes p extending u
        float* gi = prm.grad_initial + (size_t)bidx * S;
        if (valid) {
            static_for<SH::K0, N + 1>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                if constexpr (GNS && k == N) {
                    float tmp[SH::own(N)];
#pragma unroll
                    for (int q = 0; q < SH::own(N) / 4; ++q) {
                        const float4 v = *reinterpret_cast<const float4*>(gn + q * 4 * LY::NT + 4 * tid);
                        tmp[4 * q] = v.x;
                        tmp[4 * q + 1] = v.y;
                        tmp[4 * q + 2] = v.z;
                        tmp[4 * q + 3] = v.w;
                    }
                    store_run<SH::own(N), 0, false>(gi + SH::lvl_off(N) + (int64_t)prefix * SH::own(N), tmp);
                } else {
                    store_run<SH::own(k), SH::own_off(k), false>(gi + SH::lvl_off(k) + (int64_t)prefix * SH::own(k), G);
                }
            });
        }
        static_for<1, P>([&](auto ic) {
            constexpr int i = decltype(ic)::value;
            lowred[(i - 1) * LY::NT + tid] = valid ? Gh[i] : 0.0f;
        });
        __syncthreads();
        static_for<1, P>([&](auto ic) {
            constexpr int i = decltype(ic)::value;
            constexpr int bs = (int)ipow(C, P - i);
            for (int u = tid; u < (int)ipow(C, i); u += blockDim.x) {
                float sum = 0.0f;
                for (int q = 0; q < bs; ++q) sum += lowred[(i - 1) * LY::NT + u * bs + q];
                gi[SH::lvl_off(i) + u] = sum;
            }
        });
    }
}

#ifndef SIG_BWD_TOP2
#define SIG_BWD_TOP2 1
#endif
// prefix-pair K2: the top level's G_N in natural per-prefix order (1) or in pairs too (0)
#ifndef SIG_BWD2P_NATTOP
#define SIG_BWD2P_NATTOP 0
#endif
// dev-only ablations of the prefix-pair kernel (wrong results; timing attribution only)
#ifndef SIG_ABL_NOREV
#define SIG_ABL_NOREV 0
#endif
#ifndef SIG_ABL_NOTOP
#define SIG_ABL_NOTOP 0
#endif
#ifndef SIG_ABL_NORED
#define SIG_ABL_NORED 0
#endif
#ifndef SIG_BWD2_STAGGER
#define SIG_BWD2_STAGGER 0
#endif
// ---------------------------------------------------------------------------------------------
// K2 with two sibling prefixes per thread ("R = 2").  Everything a thread computes below level P
// -- the replicated prefix values low[], the prefix-chain values B_i (i < P), the partial
// low-level gradient Ghat and the low tails of every chain, the C-vector gz -- is the same for the
// sibling prefixes pa = 2t and pb = 2t + 1 (same p[:P-1]); only level P and above differ.  One
// thread therefore carries both blocks and does the shared work once: per useful FMA this halves
// the scalar overhead and the gz reduction.  Half the threads (CP/2 per path) with twice the
// registers (up to 255): two warps per SM sub-partition instead of four.
// Used for plain calls (no stream, no time chunks, no initial state) of shapes with even C, P >= 2
// and CP/2 a multiple of 32 (BwdLayout2::OK); everything else runs sig_bwd_kernel.
// ---------------------------------------------------------------------------------------------
template <class SH>
struct BwdLayout2 {
    static constexpr int C = SH::C, N = SH::N, P = SH::P;
    // ... and a state small enough for two copies plus ~60 working registers in the per-thread share
    // of the register file (c2's (8,5,3): 2 x 82 floats; c4's (4,7,4) with 2 x 106 spills and ran
    // 16% slower than the one-prefix kernel)
    static constexpr int NT = SH::CP / 2;
    static constexpr int REGS = (65536 / (NT > 0 ? NT : 1)) < 255 ? (65536 / (NT > 0 ? NT : 1)) : 255;
    static constexpr bool OK = (C % 2 == 0) && (32 % C == 0) && ((C & (C - 1)) == 0) && P >= 2 && (NT % 32 == 0) &&
                               NT <= 512 && 2 * (SH::OWN + SH::OWNA) + 48 + 4 * P <= REGS;
    static constexpr int HW = NT / 32;
    __host__ __device__ static int tile(int64_t M) {
        int T = 128;
        while (T > 1 && (size_t)T * HW * C * sizeof(float) > 96 * 1024) T >>= 1;
        return (int)(T < M ? T : M);
    }
    static size_t smem_bytes(int64_t M) {
        const size_t zf = (size_t)((M * C + 3) / 4 * 4);
        const size_t T = (size_t)tile(M);
        return (zf + T * HW * C + T * C + 32) * sizeof(float);
    }
    // floats of the TMA staging area for a path of L points (its 16-byte-aligned cover)
    static size_t raw_floats(int64_t L) { return (size_t)((L * C + 8 + 3) / 4 * 4); }
};

// the prefix chain of chain K up to level J (J <= P-1): Bp[j] = B^(K)_j[p[:j]], j = 1..J (Bp[0] = 1)
template <class SH, int K, int J>
__device__ __forceinline__ void chain_low(float (&Bp)[SH::PL1], const float (&low)[SH::LOWA], const float (&zp)[SH::PD]) {
    Bp[0] = 1.0f;
    static_for<1, J + 1>([&](auto jc) {
        constexpr int j = decltype(jc)::value;
        if constexpr (j == 1) Bp[j] = fmaf(zp[0], inv_int(K), low[j]);
        else Bp[j] = fmaf(Bp[j - 1] * inv_int(K - j + 1), zp[j - 1], low[j]);
    });
}

template <class SH>
__global__ void __launch_bounds__(BwdLayout2<SH>::NT, 1) sig_bwd2_kernel(const BwdParams prm) {
    using LY = BwdLayout2<SH>;
    constexpr int C = SH::C, N = SH::N, P = SH::P;
    constexpr int HW = LY::HW;
    extern __shared__ __align__(16) float sm[];
    const int64_t bidx = blockIdx.x;
    const int64_t M = prm.M;
    const int T = LY::tile(M);
    float* zbuf = sm;                                 // [M][C] increments
    float* part = zbuf + (M * C + 3) / 4 * 4;         // [T][HW][C] per-warp gz records
    float* tot = part + (size_t)T * HW * C;           // [T][C] per-step gz totals
    float* gprev = tot + (size_t)T * C;               // [C]

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int has_bp = prm.bp_mode != 0;
    const float* sigrow = prm.sig_final + (size_t)bidx * prm.sf_stride;
    const float* gorow = prm.grad_out + (size_t)bidx * prm.go_stride;

    __shared__ uint64_t stage_bar;
    stage_path_increments<C>(prm, bidx, M, zbuf, sm, &stage_bar);
    if (tid < C) gprev[tid] = 0.0f;

    const int pa = 2 * tid;  // prefixes pa, pa + 1 (siblings: same p[:P-1], last digit p[P-1], p[P-1] + 1)
    int p[SH::PD];
    prefix_digits<SH>(pa, p);
    float Aa[SH::OWNA], Ab[SH::OWNA], Ga[SH::OWN], Gb[SH::OWN];
    float low[SH::LOWA], Gh[SH::LOWA];
    static_for<SH::K0, N>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        load_run<SH::own(k), SH::own_off(k)>(Aa, sigrow + SH::lvl_off(k) + (int64_t)pa * SH::own(k));
        load_run<SH::own(k), SH::own_off(k)>(Ab, sigrow + SH::lvl_off(k) + (int64_t)(pa + 1) * SH::own(k));
    });
    static_for<SH::K0, N + 1>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        load_run<SH::own(k), SH::own_off(k)>(Ga, gorow + SH::lvl_off(k) + (int64_t)pa * SH::own(k));
        load_run<SH::own(k), SH::own_off(k)>(Gb, gorow + SH::lvl_off(k) + (int64_t)(pa + 1) * SH::own(k));
    });
    low[0] = 0.0f;
    Gh[0] = 0.0f;
    static_for<1, P>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        constexpr int tail = (int)ipow(C, P - i);
        low[i] = sigrow[SH::lvl_off(i) + pa / tail];
        Gh[i] = (pa % tail == 0) ? gorow[SH::lvl_off(i) + pa / tail] : 0.0f;
    });
    __syncthreads();
    if (SIG_BWD2_STAGGER > 0 && ((warp >> 2) & 1)) __nanosleep(SIG_BWD2_STAGGER);

    // channels of the level-P (pa, pb) and level-(P-1) partials in the reduction (see below)
    constexpr int HC = C / 2;
    const int gbase = lane & ~(C - 1);
    const int ch = lane & (C - 1);
    const int chP1_g0 = ((tid & ~(C - 1)) / HC) % C;        // ... of sub-group 0 of its C-lane group
    const int chP1_g1 = (((tid & ~(C - 1)) + HC) / HC) % C; // ... of sub-group 1

    for (int64_t n0 = 0; n0 < M; n0 += T) {
        const int tn = (int)((M - n0) < T ? (M - n0) : T);
        for (int j = 0; j < tn; ++j) {
            const int64_t t = M - 1 - (n0 + j);
            float z[C], zp[SH::PD];
#pragma unroll
            for (int c = 0; c < C; ++c) z[c] = zbuf[t * C + c];
#pragma unroll
            for (int q = 0; q < SH::PD; ++q) zp[q] = zbuf[t * C + p[q]];
            const float zpb = zbuf[t * C + p[P - 1] + 1];
            // (1) reversibility: levels < N; the exact start state (identity) at t = 0
            if (t > 0) {
                mulexp2<SH, N - 1, true>(Aa, Ab, low, z, zp, zpb);
            } else {
#pragma unroll
                for (int q = 0; q < SH::OWNA; ++q) Aa[q] = Ab[q] = 0.0f;
#pragma unroll
                for (int q = 0; q < SH::LOWA; ++q) low[q] = 0.0f;
            }
            // (2)+(3): chains k = 1..N bottom-up
            float gz[C];
#pragma unroll
            for (int c = 0; c < C; ++c) gz[c] = 0.0f;
            float acc[SH::PL1];
#pragma unroll
            for (int q = 0; q < SH::PL1; ++q) acc[q] = 0.0f;
            float accPb = 0.0f;  // level-P partial of pb (acc[P] is pa's)
            static_for<1, P>([&](auto kc) {  // chains entirely below P
                constexpr int k = decltype(kc)::value;
                float Bp[SH::PL1];
                chain_low<SH, k, k - 1>(Bp, low, zp);
                low_tail<SH, k, k>(Gh[k], Bp, zp, acc, Gh);
            });
            // level P of the low tail of chain k per prefix (betas ba, bb at level P), then one shared
            // tail from level P-1
            auto tail_k = [&](auto kc, const float (&Bp)[SH::PL1], float ba, float bb) {
                constexpr int k = decltype(kc)::value;
                constexpr float sc = inv_int(k - P + 1);
                const float bps = Bp[P - 1] * sc;
                acc[P] = fmaf(bps, ba, acc[P]);
                accPb = fmaf(bps, bb, accPb);
                const float b1 = fmaf(ba * zp[P - 1], sc, (bb * zpb) * sc);
                Gh[P - 1] += b1;
                low_tail<SH, k, P - 1>(b1, Bp, zp, acc, Gh);
            };
            constexpr bool TOP2 = SIG_BWD_TOP2 && (N - 2 >= P);
            static_for<P, (TOP2 ? N - 1 : N + 1)>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                constexpr float sc = inv_int(k - P + 1);
                float Bp[SH::PL1];
                chain_low<SH, k, P - 1>(Bp, low, zp);
                float ba, bb;
                if constexpr (k == P) {
                    ba = Ga[SH::own_off(P)];
                    bb = Gb[SH::own_off(P)];
                } else {
                    const float bs = Bp[P - 1] * sc;
                    ba = vjp_visit<SH, k, P, 0>(fmaf(bs, zp[P - 1], Aa[SH::own_off(P)]), Ga, Aa, z, gz);
                    bb = vjp_visit<SH, k, P, 0>(fmaf(bs, zpb, Ab[SH::own_off(P)]), Gb, Ab, z, gz);
                }
                tail_k(kc, Bp, ba, bb);
            });
            if constexpr (TOP2) {
                // chains N-1 and N walked together (vjp_top2)
                constexpr float sc1 = inv_int(N - 1 - P + 1), sc2 = inv_int(N - P + 1);
                float Bp1[SH::PL1], Bp2[SH::PL1];
                chain_low<SH, N - 1, P - 1>(Bp1, low, zp);
                chain_low<SH, N, P - 1>(Bp2, low, zp);
                const float bs1 = Bp1[P - 1] * sc1, bs2 = Bp2[P - 1] * sc2;
                float b1a, b2a, b1b, b2b;
                vjp_top2<SH, P, 0>(fmaf(bs1, zp[P - 1], Aa[SH::own_off(P)]), fmaf(bs2, zp[P - 1], Aa[SH::own_off(P)]),
                                   Ga, Aa, z, gz, b1a, b2a);
                vjp_top2<SH, P, 0>(fmaf(bs1, zpb, Ab[SH::own_off(P)]), fmaf(bs2, zpb, Ab[SH::own_off(P)]), Gb, Ab, z,
                                   gz, b1b, b2b);
                tail_k(std::integral_constant<int, N - 1>{}, Bp1, b1a, b1b);
                tail_k(std::integral_constant<int, N>{}, Bp2, b2a, b2b);
            }

            // ---- per-step gz: warp reduction into the tile
            float v[C];
#pragma unroll
            for (int c = 0; c < C; ++c) v[c] = gz[c];
            static_for<0, ilog2(C)>([&](auto sc_) {
                constexpr int m = C >> (decltype(sc_)::value + 1);
                const bool up = (lane & m) != 0;
#pragma unroll
                for (int q = 0; q < m; ++q) {
                    const float send = up ? v[q] : v[q + m];
                    const float keep = up ? v[q + m] : v[q];
                    v[q] = keep + __shfl_xor_sync(0xffffffffu, send, m);
                }
            });
            float tv = v[0];  // channel ch = lane % C, summed over the C-lane group
            {
                // level P: pa -> channel 2 (tid % HC), pb -> +1; lanes j and j + HC of a group share them
                const float u0 = acc[P] + __shfl_xor_sync(0xffffffffu, acc[P], HC);
                const float u1 = accPb + __shfl_xor_sync(0xffffffffu, accPb, HC);
                const float t0 = __shfl_sync(0xffffffffu, u0, gbase + (ch >> 1));
                const float t1 = __shfl_sync(0xffffffffu, u1, gbase + (ch >> 1));
                tv += (ch & 1) ? t1 : t0;
            }
            {
                // level P-1: channel p_{P-2}, constant over each half (HC lanes) of the group
                float gs = acc[P - 1];
#pragma unroll
                for (int m = 1; m < HC; m <<= 1) gs += __shfl_xor_sync(0xffffffffu, gs, m);
                const float s0 = __shfl_sync(0xffffffffu, gs, gbase);
                const float s1 = __shfl_sync(0xffffffffu, gs, gbase + HC);
                if (ch == chP1_g0) tv += s0;
                if (ch == chP1_g1) tv += s1;
            }
            static_for<1, P - 1>([&](auto ic) {  // levels below P-1: channel constant over the group
                constexpr int i = decltype(ic)::value;
                float gsum = acc[i];
#pragma unroll
                for (int m = 1; m < C; m <<= 1) gsum += __shfl_xor_sync(0xffffffffu, gsum, m);
                if (ch == p[i - 1]) tv += gsum;
            });
#pragma unroll
            for (int m = C; m < 32; m <<= 1) tv += __shfl_xor_sync(0xffffffffu, tv, m);
            if (lane < C) part[((size_t)j * HW + warp) * C + lane] = tv;
        }
        // ---- flush
        __syncthreads();
        for (int e = tid; e < tn * C; e += blockDim.x) {
            const int j = e / C, c = e % C;
            float s = 0.0f;
            for (int w = 0; w < HW; ++w) s += part[((size_t)j * HW + w) * C + c];
            tot[j * C + c] = s;
        }
        __syncthreads();
        for (int e = tid; e < tn * C; e += blockDim.x) {
            const int j = e / C, c = e % C;
            const int64_t t = M - 1 - (n0 + j);
            const float before = (j == 0) ? gprev[c] : tot[(j - 1) * C + c];
            const int64_t r = t + 1;  // augmented point t + 1
            float* gr = has_bp ? prm.grad_path + (bidx * prm.L + (r - 1)) * C : prm.grad_path + (bidx * prm.L + r) * C;
            gr[c] = prm.zsign * (tot[j * C + c] - before);
            if (t == 0) {
                float* g0 = has_bp ? ((prm.bp_mode == 2 && prm.grad_bp) ? prm.grad_bp + bidx * C : nullptr)
                                   : prm.grad_path + bidx * prm.L * C;
                if (g0) g0[c] = -prm.zsign * tot[j * C + c];
            }
        }
        __syncthreads();
        if (tid < C) gprev[tid] = tot[(tn - 1) * C + tid];
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------------
// K2 with the two sibling prefixes as the two lanes of every FFMA2 ("prefix-pair" layout).
// Same algorithm and launch geometry as sig_bwd2_kernel, for shapes whose two top chains meet at the
// prefix level (N - 2 == P, e.g. c2's (8, 5, 3)).  Everything at levels >= P is computed for both
// prefixes at once: the state is held as float2 pairs (A[pa.w], A[pb.w]), z enters as a broadcast
// scalar, and every dot product over channels accumulates a pair -- so there is no horizontal add
// anywhere above P, and the instruction stream above P is pure FFMA2 (a mix of FFMA and FFMA2 runs
// measurably slower at two warps per SM sub-partition, K2).  gz then holds one partial
// per prefix, summed once per step.  The two top chains are walked together as in vjp_top2.
// ---------------------------------------------------------------------------------------------
template <class SH>
struct BwdLayout2P {
    static constexpr bool OK = BwdLayout2<SH>::OK && (SH::N - 2 == SH::P);
};

__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }

// reversal Horner walk in pair layout: node (I, W) with BI = (B_I[pa.W], B_I[pb.W]); children
// B_{I+1}[p.W.c] = B_I[p.W] (-z_c) / (K-I) + A_{I+1}[p.W.c]; at I+1 = K A is updated in place
template <class SH, int K, int I, int W, int SZ>
__device__ __forceinline__ void horner_pp_neg(float2 BI, float2 (&AP)[SZ], const float (&z)[SH::C]) {
    constexpr int C = SH::C;
    const float2 bs = (K - I == 1) ? BI : __fmul2_rn(BI, f2(inv_int(K - I)));
    static_for<0, C>([&](auto cc) {
        constexpr int c = decltype(cc)::value;
        constexpr int o = SH::own_off(I + 1) + W * C + c;
        const float2 r = __ffma2_rn(bs, f2(-z[c]), AP[o]);
        if constexpr (I + 1 == K) AP[o] = r;
        else horner_pp_neg<SH, K, I + 1, W * C + c>(r, AP, z);
    });
}

template <class SH>
__global__ void __launch_bounds__(BwdLayout2<SH>::NT, 1) sig_bwd2p_kernel(const BwdParams prm) {
    using LY = BwdLayout2<SH>;
    constexpr int C = SH::C, N = SH::N, P = SH::P;
    static_assert(N - 2 == P && P >= 2 && C % 2 == 0, "prefix-pair K2: the top chains meet at level P");
    constexpr int HW = LY::HW;
    constexpr int NA = SH::OWNA;  // owned levels P..N-1
    constexpr int NG = SH::OWN;   // owned levels P..N
    extern __shared__ __align__(16) float sm[];
    const int64_t bidx = blockIdx.x;
    const int64_t M = prm.M;
    const int T = LY::tile(M);
    float* zbuf = sm;                                 // [M][C] increments
    float* part = zbuf + (M * C + 3) / 4 * 4;         // [T][HW][C] per-warp gz records
    float* tot = part + (size_t)T * HW * C;           // [T][C] per-step gz totals
    float* gprev = tot + (size_t)T * C;               // [C]

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int has_bp = prm.bp_mode != 0;
    const float* sigrow = prm.sig_final + (size_t)bidx * prm.sf_stride;
    const float* gorow = prm.grad_out + (size_t)bidx * prm.go_stride;

    __shared__ uint64_t stage_bar;
    stage_path_increments<C>(prm, bidx, M, zbuf, sm, &stage_bar);
    if (tid < C) gprev[tid] = 0.0f;

    const int pa = 2 * tid;  // prefixes pa, pa + 1: same p[:P-1], last digits p[P-1], p[P-1] + 1
    int p[SH::PD];
    prefix_digits<SH>(pa, p);
    // levels P..N-1 in pairs; the top level G_N per prefix in natural order (NT: the top loop's gz
    // update is then an FFMA2 with a broadcast chain value, K2)
    constexpr int CN = SH::own(N);
    float2 AP[NA], GP[NG];
    float GNa[SIG_BWD2P_NATTOP ? CN : 1], GNb[SIG_BWD2P_NATTOP ? CN : 1];
    float low[SH::LOWA], Gh[SH::LOWA];
    static_for<SH::K0, N + 1>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        constexpr int n = SH::own(k);
        float ta[n], tb[n];
        auto ld = [&](float* dst, const float* src) { load_run<n, 0>(*reinterpret_cast<float(*)[n]>(dst), src); };
        if constexpr (k < N) {
            ld(ta, sigrow + SH::lvl_off(k) + (int64_t)pa * n);
            ld(tb, sigrow + SH::lvl_off(k) + (int64_t)(pa + 1) * n);
#pragma unroll
            for (int q = 0; q < n; ++q) AP[SH::own_off(k) + q] = make_float2(ta[q], tb[q]);
        }
        if constexpr (k == N && SIG_BWD2P_NATTOP) {
            ld(GNa, gorow + SH::lvl_off(k) + (int64_t)pa * n);
            ld(GNb, gorow + SH::lvl_off(k) + (int64_t)(pa + 1) * n);
        } else {
            ld(ta, gorow + SH::lvl_off(k) + (int64_t)pa * n);
            ld(tb, gorow + SH::lvl_off(k) + (int64_t)(pa + 1) * n);
#pragma unroll
            for (int q = 0; q < n; ++q) GP[SH::own_off(k) + q] = make_float2(ta[q], tb[q]);
        }
    });
    low[0] = 0.0f;
    Gh[0] = 0.0f;
    static_for<1, P>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        constexpr int tail = (int)ipow(C, P - i);
        low[i] = sigrow[SH::lvl_off(i) + pa / tail];
        Gh[i] = (pa % tail == 0) ? gorow[SH::lvl_off(i) + pa / tail] : 0.0f;
    });
    __syncthreads();

    constexpr int HC = C / 2;
    const int gbase = lane & ~(C - 1);
    const int ch = lane & (C - 1);
    const int chP1_g0 = ((tid & ~(C - 1)) / HC) % C;
    const int chP1_g1 = (((tid & ~(C - 1)) + HC) / HC) % C;
    constexpr int oP = SH::own_off(P), o1 = SH::own_off(N - 1), oN = SH::own_off(N);

    for (int64_t n0 = 0; n0 < M; n0 += T) {
        const int tn = (int)((M - n0) < T ? (M - n0) : T);
        for (int j = 0; j < tn; ++j) {
            const int64_t t = M - 1 - (n0 + j);
            float z[C], zp[SH::PD];
#pragma unroll
            for (int c = 0; c < C; ++c) z[c] = zbuf[t * C + c];
#pragma unroll
            for (int q = 0; q < SH::PD; ++q) zp[q] = zbuf[t * C + p[q]];
            const float zpb = zbuf[t * C + p[P - 1] + 1];
            const float2 zpp = make_float2(zp[P - 1], zpb);
            // (1) reversibility A <- A [x] exp(-z) on levels < N; the exact start state at t = 0
            if (!SIG_ABL_NOREV && t > 0) {
                static_for<0, N - 1 - P + 1>([&](auto kkc) {
                    constexpr int k = N - 1 - decltype(kkc)::value;  // N-1 .. P
                    float b = 1.0f;
                    static_for<1, P>([&](auto ic) {
                        constexpr int i = decltype(ic)::value;
                        if constexpr (i == 1) b = fmaf(zp[0], -inv_int(k), low[i]);
                        else b = fmaf(b * (-inv_int(k - i + 1)), zp[i - 1], low[i]);
                    });
                    const float2 BP = __ffma2_rn(f2(b * (-inv_int(k - P + 1))), zpp, AP[oP]);
                    if constexpr (k == P) AP[oP] = BP;
                    else horner_pp_neg<SH, k, P, 0>(BP, AP, z);
                });
                static_for<0, P - 1>([&](auto kkc) {
                    constexpr int k = P - 1 - decltype(kkc)::value;
                    float b = 1.0f;
                    static_for<1, k + 1>([&](auto ic) {
                        constexpr int i = decltype(ic)::value;
                        if constexpr (i == 1) b = fmaf(zp[0], -inv_int(k), low[i]);
                        else b = fmaf(b * (-inv_int(k - i + 1)), zp[i - 1], low[i]);
                    });
                    low[k] = b;
                });
            } else {
#pragma unroll
                for (int q = 0; q < NA; ++q) AP[q] = make_float2(0.0f, 0.0f);
#pragma unroll
                for (int q = 0; q < SH::LOWA; ++q) low[q] = 0.0f;
            }
            // (2)+(3): chains k = 1..N bottom-up
            float acc[SH::PL1];
#pragma unroll
            for (int q = 0; q < SH::PL1; ++q) acc[q] = 0.0f;
            float accPb = 0.0f;
            auto tail_k = [&](auto kc, const float (&Bp)[SH::PL1], float ba, float bb) {
                constexpr int k = decltype(kc)::value;
                constexpr float sc = inv_int(k - P + 1);
                const float bps = Bp[P - 1] * sc;
                acc[P] = fmaf(bps, ba, acc[P]);
                accPb = fmaf(bps, bb, accPb);
                const float b1 = fmaf(ba * zp[P - 1], sc, (bb * zpb) * sc);
                Gh[P - 1] += b1;
                low_tail<SH, k, P - 1>(b1, Bp, zp, acc, Gh);
            };
            static_for<1, P>([&](auto kc) {  // chains entirely below P
                constexpr int k = decltype(kc)::value;
                float Bp[SH::PL1];
                chain_low<SH, k, k - 1>(Bp, low, zp);
                low_tail<SH, k, k>(Gh[k], Bp, zp, acc, Gh);
            });
            {  // chain P: its leaf is G_P itself
                float Bp[SH::PL1];
                chain_low<SH, P, P - 1>(Bp, low, zp);
                tail_k(std::integral_constant<int, P>{}, Bp, GP[oP].x, GP[oP].y);
            }
            // chains N-1 and N together (see vjp_top2), both prefixes per FFMA2
            float Bp1[SH::PL1], Bp2[SH::PL1];
            chain_low<SH, N - 1, P - 1>(Bp1, low, zp);
            chain_low<SH, N, P - 1>(Bp2, low, zp);
            const float2 b1 = __ffma2_rn(f2(Bp1[P - 1] * inv_int(N - P)), zpp, AP[oP]);      // B^(N-1)_P
            const float2 bs2 = __fmul2_rn(__ffma2_rn(f2(Bp2[P - 1] * inv_int(N - P + 1)), zpp, AP[oP]),
                                          f2(0.5f));                                        // B^(N)_P / 2
            const float2 d = __ffma2_rn(bs2, f2(-1.0f), b1);
            float2 acc1 = make_float2(0.0f, 0.0f);
            float2 Bc[C];
            static_for<0, C>([&](auto cc) {
                constexpr int c = decltype(cc)::value;
                Bc[c] = __ffma2_rn(bs2, f2(z[c]), AP[o1 + c]);
            });
            float v[C];
            if constexpr (SIG_BWD2P_NATTOP) {
                float gza[C], gzb[C];  // per-prefix gz partials, natural channel pairs
                static_for<0, C>([&](auto cc) {  // chain N-1 on the old G_{N-1}
                    constexpr int c = decltype(cc)::value;
                    gza[c] = d.x * GP[o1 + c].x;
                    gzb[c] = d.y * GP[o1 + c].y;
                    acc1 = __ffma2_rn(GP[o1 + c], f2(z[c]), acc1);
                });
                if (!SIG_ABL_NOTOP) static_for<0, C>([&](auto cc) {  // the top level
                    constexpr int c = decltype(cc)::value;
                    static_for<0, C / 2>([&](auto qq) {
                        constexpr int q = 2 * decltype(qq)::value;
                        const float2 ra = __ffma2_rn(f2(Bc[c].x), make_float2(GNa[c * C + q], GNa[c * C + q + 1]),
                                                     make_float2(gza[q], gza[q + 1]));
                        gza[q] = ra.x;
                        gza[q + 1] = ra.y;
                        const float2 rb = __ffma2_rn(f2(Bc[c].y), make_float2(GNb[c * C + q], GNb[c * C + q + 1]),
                                                     make_float2(gzb[q], gzb[q + 1]));
                        gzb[q] = rb.x;
                        gzb[q + 1] = rb.y;
                    });
                    float ga = GP[o1 + c].x, gb = GP[o1 + c].y;
                    static_for<0, C>([&](auto qq) {
                        constexpr int q = decltype(qq)::value;
                        ga = fmaf(GNa[c * C + q], z[q], ga);
                        gb = fmaf(GNb[c * C + q], z[q], gb);
                    });
                    GP[o1 + c] = make_float2(ga, gb);
                });
                static_for<0, C>([&](auto cc) {  // chain N on the new G_{N-1}
                    constexpr int c = decltype(cc)::value;
                    gza[c] = fmaf(bs2.x, GP[o1 + c].x, gza[c]);
                    gzb[c] = fmaf(bs2.y, GP[o1 + c].y, gzb[c]);
                    v[c] = gza[c] + gzb[c];
                });
            } else {
                float2 gzab[C];
                static_for<0, C>([&](auto cc) {  // chain N-1 on the old G_{N-1}
                    constexpr int c = decltype(cc)::value;
                    gzab[c] = __fmul2_rn(d, GP[o1 + c]);
                    acc1 = __ffma2_rn(GP[o1 + c], f2(z[c]), acc1);
                });
                // the top level, in blocks of C independent accumulators sharing one operand: row k of
                // the rank-1 gz update (B_k reused), then column k of the dot products (z_k reused)
                if (!SIG_ABL_NOTOP) static_for<0, C>([&](auto kk) {
                    constexpr int k = decltype(kk)::value;
                    static_for<0, C>([&](auto qq) {
                        constexpr int q = decltype(qq)::value;
                        gzab[q] = __ffma2_rn(Bc[k], GP[oN + k * C + q], gzab[q]);
                    });
                    static_for<0, C>([&](auto cc) {
                        constexpr int c = decltype(cc)::value;
                        GP[o1 + c] = __ffma2_rn(GP[oN + c * C + k], f2(z[k]), GP[o1 + c]);
                    });
                });
                static_for<0, C>([&](auto cc) {  // chain N on the new G_{N-1}
                    constexpr int c = decltype(cc)::value;
                    gzab[c] = __ffma2_rn(bs2, GP[o1 + c], gzab[c]);
                    v[c] = gzab[c].x + gzab[c].y;
                });
            }
            float2 acc2 = make_float2(-acc1.x, -acc1.y);
            static_for<0, C>([&](auto cc) {
                constexpr int c = decltype(cc)::value;
                acc2 = __ffma2_rn(GP[o1 + c], f2(z[c]), acc2);
            });
            const float2 beta2 = __fmul2_rn(acc2, f2(0.5f));
            GP[oP] = __fadd2_rn(GP[oP], __fadd2_rn(acc1, beta2));
            tail_k(std::integral_constant<int, N - 1>{}, Bp1, acc1.x, acc1.y);
            tail_k(std::integral_constant<int, N>{}, Bp2, beta2.x, beta2.y);

            // ---- per-step gz (the two prefix partials were summed into v): warp reduction into the tile
            if (SIG_ABL_NORED) {
                float sv = accPb + acc[P] + acc[P - 1];
#pragma unroll
                for (int c = 0; c < C; ++c) sv += v[c];
                if (lane < C) part[((size_t)j * HW + warp) * C + lane] = sv;
                continue;
            }
            static_for<0, ilog2(C)>([&](auto sc_) {
                constexpr int m = C >> (decltype(sc_)::value + 1);
                const bool up = (lane & m) != 0;
#pragma unroll
                for (int q = 0; q < m; ++q) {
                    const float send = up ? v[q] : v[q + m];
                    const float keep = up ? v[q + m] : v[q];
                    v[q] = keep + __shfl_xor_sync(0xffffffffu, send, m);
                }
            });
            float tv = v[0];
            {
                const float u0 = acc[P] + __shfl_xor_sync(0xffffffffu, acc[P], HC);
                const float u1 = accPb + __shfl_xor_sync(0xffffffffu, accPb, HC);
                const float t0 = __shfl_sync(0xffffffffu, u0, gbase + (ch >> 1));
                const float t1 = __shfl_sync(0xffffffffu, u1, gbase + (ch >> 1));
                tv += (ch & 1) ? t1 : t0;
            }
            {
                float gs = acc[P - 1];
#pragma unroll
                for (int m = 1; m < HC; m <<= 1) gs += __shfl_xor_sync(0xffffffffu, gs, m);
                const float s0 = __shfl_sync(0xffffffffu, gs, gbase);
                const float s1 = __shfl_sync(0xffffffffu, gs, gbase + HC);
                if (ch == chP1_g0) tv += s0;
                if (ch == chP1_g1) tv += s1;
            }
            static_for<1, P - 1>([&](auto ic) {
                constexpr int i = decltype(ic)::value;
                float gsum = acc[i];
#pragma unroll
                for (int m = 1; m < C; m <<= 1) gsum += __shfl_xor_sync(0xffffffffu, gsum, m);
                if (ch == p[i - 1]) tv += gsum;
            });
#pragma unroll
            for (int m = C; m < 32; m <<= 1) tv += __shfl_xor_sync(0xffffffffu, tv, m);
            if (lane < C) part[((size_t)j * HW + warp) * C + lane] = tv;
        }
        // ---- flush
        __syncthreads();
        for (int e = tid; e < tn * C; e += blockDim.x) {
            const int j = e / C, c = e % C;
            float s = 0.0f;
            for (int w = 0; w < HW; ++w) s += part[((size_t)j * HW + w) * C + c];
            tot[j * C + c] = s;
        }
        __syncthreads();
        for (int e = tid; e < tn * C; e += blockDim.x) {
            const int j = e / C, c = e % C;
            const int64_t t = M - 1 - (n0 + j);
            const float before = (j == 0) ? gprev[c] : tot[(j - 1) * C + c];
            const int64_t r = t + 1;
            float* gr = has_bp ? prm.grad_path + (bidx * prm.L + (r - 1)) * C : prm.grad_path + (bidx * prm.L + r) * C;
            gr[c] = prm.zsign * (tot[j * C + c] - before);
            if (t == 0) {
                float* g0 = has_bp ? ((prm.bp_mode == 2 && prm.grad_bp) ? prm.grad_bp + bidx * C : nullptr)
                                   : prm.grad_path + bidx * prm.L * C;
                if (g0) g0[c] = -prm.zsign * tot[j * C + c];
            }
        }
        __syncthreads();
        if (tid < C) gprev[tid] = tot[(tn - 1) * C + tid];
        __syncthreads();
    }
}

#ifndef SIG_BWD2
#define SIG_BWD2 1
#endif
#ifndef SIG_BWD_TMA_STAGE
#define SIG_BWD_TMA_STAGE 1
#endif
#ifndef SIG_BWD2P
#define SIG_BWD2P 1
#endif

template <class SH>
int64_t bwd_slots();

template <class SH>
cudaError_t launch_bwd(const BwdParams& prm, cudaStream_t st) {
    if constexpr (SIG_BWD2 && BwdLayout2<SH>::OK) {
        using LY2 = BwdLayout2<SH>;
        if (!prm.stream && prm.n_chunks == 1 && prm.initial == nullptr && prm.grad_initial == nullptr) {
            const size_t smem2 = LY2::smem_bytes(prm.M);
            if (smem2 <= 227 * 1024) {
                auto kern = sig_bwd2_kernel<SH>;
                size_t smem = smem2;
                unsigned grid = (unsigned)prm.B;
                if constexpr (SIG_BWD2P && BwdLayout2P<SH>::OK) kern = sig_bwd2p_kernel<SH>;
                BwdParams q = prm;
                q.raw_off = 0;
                // TMA staging of the points when the cover stays inside the path tensor (16-byte
                // aligned start and end) and fits next to the rest
                const bool aligned = (reinterpret_cast<uintptr_t>(prm.path) & 15) == 0 && (prm.B * prm.L * SH::C) % 4 == 0;
                const int64_t roff = ((int64_t)(smem2 / sizeof(float)) + 3) / 4 * 4;  // 16-byte aligned
                const size_t with_raw = ((size_t)roff + LY2::raw_floats(prm.L)) * sizeof(float);
                if (SIG_BWD_TMA_STAGE && aligned && with_raw <= 227 * 1024) {
                    q.raw_off = roff;
                    smem = with_raw;
                }
                if (smem > 48 * 1024) {
                    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                    if (e != cudaSuccess) return e;
                }
                kern<<<grid, LY2::NT, smem, st>>>(q);
                return cudaGetLastError();
            }
        }
    }
    using LY = BwdLayout<SH>;
    auto kern = prm.stream ? sig_bwd_kernel<SH, true> : sig_bwd_kernel<SH, false>;
    const int slots = bwd_slots<SH>();
    if (slots <= 0) return cudaErrorInvalidConfiguration;
    // the shared memory that leaves the register-limited number of CTAs resident (c5's chunked
    // backward: 1-warp CTAs, 16 per SM), at most SIG_BWD_TILE_KB
    size_t budget = (size_t)228 * 1024 / slots - 1024;
    if (budget > (size_t)SIG_BWD_TILE_KB * 1024) budget = (size_t)SIG_BWD_TILE_KB * 1024;
    const size_t gnb = prm.stream ? 0 : (size_t)LY::GNF * sizeof(float);  // GNS region (plain kernel)
    budget = budget > gnb + 4096 ? budget - gnb : 4096;
    BwdParams q = prm;
    q.tile = LY::tile(prm.chunk_len, budget);
    const size_t smem = LY::smem_bytes_tile(q.tile) + gnb;
    if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    kern<<<(unsigned)(prm.B * prm.n_chunks), LY::NT, smem, st>>>(q);
    return cudaGetLastError();
}

// CTAs of sig_bwd_kernel resident per SM as limited by registers and warps (the tile is then sized
// so that shared memory does not lower it); 0 if the kernel cannot be queried.
template <class SH>
int64_t bwd_slots() {
    static int cached = -1;
    if (cached < 0) {
        cudaFuncAttributes a{};
        if (cudaFuncGetAttributes(&a, sig_bwd_kernel<SH, false>) != cudaSuccess) return 0;
        constexpr int NT = BwdLayout<SH>::NT;
        const int regs_per_warp = (a.numRegs * 32 + 255) / 256 * 256;
        int n = 65536 / (regs_per_warp * (NT / 32));
        if (n > 64 / (NT / 32)) n = 64 / (NT / 32);
        if (n > 32) n = 32;
        cached = n;
    }
    return cached;
}

}  // namespace sigb200
