// sig_fwd.cuh -- K1: the fused multiply-exponentiate scan (forward signature), sm_100a.
//
// Method (Appendix A.1.2): Sig = exp(z_0) [x] exp(z_1) [x] ... is a
// reduction with the fused operation A <- A [x] exp(z), whose level-k term is evaluated in
// Horner form (eq-fusedterm):
//     B_1 = z/k + A_1,   B_i = B_{i-1} (x) z/(k-i+1) + A_i  (i = 2..k),   A_k <- B_k,
// for k = N down to 1, so that every A_i read while updating level k is still the old value.
// The first exponential is the same update applied to the identity (A = 0).
//
// B200 design: FP32 FMA on the CUDA cores (no contraction dimension here, so
// tensor cores do not apply), state register-resident with the prefix decomposition described in
// sig_common.cuh -- no inter-thread communication inside the scan.  Increments are staged into
// shared memory per tile; every thread reads the same z_t (broadcast LDS).  A "unit" is one time
// chunk of one path ("splitting the computation up into chunks"); chunk results are
// folded afterwards by the combine kernels (K3).
#pragma once
#include "combine.cuh"
#include "sig_common.cuh"

// increments staged per tile of the grouped-chunk scan (at most SIG_FWD_TILE steps and
// SIG_FWD_TILE_KB of shared memory for all units of the CTA)
#ifndef SIG_FWD_TILE
#define SIG_FWD_TILE 1024
#endif
#ifndef SIG_FWD_TILE_KB
#define SIG_FWD_TILE_KB 160
#endif
#ifndef SIG_FWD_TMA_STAGE
#define SIG_FWD_TMA_STAGE 1
#endif
// one-prefix forward prefix chains written as b * (z_p / m) + A instead of (b / m) z_p + A (same
// operation count; measured: c5's scan 410 -> 400 us; the two-prefix mulexp2 keeps the other form:
// c2's forward 237 -> 243 us with it).  The backward's reversal keeps the other form: there
// the scaled increments become common subexpressions of the reversal, the VJP chains and the low
// tails, and the extra live registers measured slower (c5b +1.6%, c4 +0.4%).
// threads of the blocked chunk scan's CTA (one group of up to 16 chunk signatures, scanned in
// order with one barrier per element): 1024 puts about one coefficient of each product on a thread
// (c5b: ~2.4 us less per scan launch than with 512, 10 launches per step)
// threads of the compiled group fold (K3) CTA; with groups of SIG_FOLD_G = 8 (api.cu): c5's six
// fold launches of 512-thread CTAs in groups of 4 become four, forward 400 -> 390 us
#ifndef SIG_FOLD_THREADS
#define SIG_FOLD_THREADS 1024
#endif
#ifndef SIG_SCAN_THREADS
#define SIG_SCAN_THREADS 1024
#endif
#ifndef SIG_ZS_CSE
#define SIG_ZS_CSE 1
#endif

namespace sigb200 {

struct FwdParams {
    const float* path;       // [B, L, C]
    const float* basepoint;  // [B, C] when bp_mode == 2
    int bp_mode;             // 0 none, 1 zero, 2 given  (reading R4)
    int stream;              // 1: write every prefix
    int64_t B, L;
    int64_t M;               // increments per path = L - 1 + (bp_mode != 0)
    int64_t chunk_len;       // increments per unit
    int64_t n_chunks;        // units per path (stream => 1)
    int64_t n_units;         // B * n_chunks
    int tile;                // increments staged per tile
    int upc;                 // > 0: grouped chunks -- each CTA holds upc consecutive chunks of one
                             //      path and writes their ordered product to out + (u / upc) * S
    TensorDims dims;         // level tables for the in-CTA fold (upc > 0)
    float* out;              // stream: [B, M, S]; upc = 0: unit u -> out + u * S
    float zsign;             // +1, or -1: scan the negated path (the inverse option, R18)
    const float* initial;    // [B, S] start state of each path's first chunk, or nullptr (identity)
    int64_t raw_off;         // > 0: sig_fwd_kernel stages each tile's points by TMA bulk copies into the
                             // shared area at this float offset (nu * RawLayout::unit(tile, C) floats)
};

// TMA staging of path points (sig_fwd_kernel): a unit's tile needs the rows r0 .. r0 + cnt of its
// path (r0 = -1 is the basepoint); the 16-byte-aligned cover of those rows is bulk-copied into a
// per-unit slot, and the increments are formed from shared memory.  One copy and one barrier wait
// per unit and tile, instead of several dependent rounds of global loads (c1 is latency-bound).
struct RawLayout {
    __host__ __device__ static int64_t unit(int tile, int C) { return (((int64_t)tile + 1) * C + 8 + 3) / 4 * 4; }
};

// Depth-first walk of the thread's word tree for the level-K Horner chain (eq-fusedterm):
// node (I, W) is the word p.W at level I (W indexes the C^(I-P) words below the prefix), BI is
// B_I[p.W].  Children: B_{I+1}[p.W.c] = B_I[p.W] * z_c / (K-I) + A_{I+1}[p.W.c]; at I+1 = K the
// child is A_K itself, updated in place.  Walking depth-first keeps one chain value per level live
// (a breadth-first sweep would hold whole blocks of B_i in registers).
template <class SH, int K, int I, int W, bool NEG, int SZ>
__device__ __forceinline__ void horner_visit(float BI, float (&own)[SZ], const float (&z)[SH::C]) {
    // Channels are processed in pairs with the packed FFMA2 (fma.rn.f32x2): the same FLOP rate as
    // FFMA in half the issue slots (measured, scripts/fma_peak.cu), which matters because the
    // scan is issue-bound.  z and the owned blocks sit in natural order, so (c, c+1) pairs are
    // aligned register pairs straight from the vector loads.
    constexpr int C = SH::C;
    constexpr float sg = NEG ? -1.0f : 1.0f;  // NEG: multiply by -z (the reversibility step)
    const float bs = (K - I == 1) ? sg * BI : BI * (sg * inv_int(K - I));
    const float2 bs2 = make_float2(bs, bs);
    static_for<0, C / 2>([&](auto cc) {
        constexpr int c = 2 * decltype(cc)::value;
        constexpr int ch = W * C + c;
        const float2 z2 = make_float2(z[c], z[c + 1]);
        if constexpr (I + 1 == K) {
            constexpr int o = SH::own_off(K) + ch;
            const float2 r = __ffma2_rn(bs2, z2, make_float2(own[o], own[o + 1]));
            own[o] = r.x;
            own[o + 1] = r.y;
        } else {
            constexpr int o = SH::own_off(I + 1) + ch;
            const float2 Bc = __ffma2_rn(bs2, z2, make_float2(own[o], own[o + 1]));
            horner_visit<SH, K, I + 1, ch, NEG>(Bc.x, own, z);
            horner_visit<SH, K, I + 1, ch + 1, NEG>(Bc.y, own, z);
        }
    });
    if constexpr (C % 2 == 1) {
        constexpr int c = C - 1;
        constexpr int ch = W * C + c;
        if constexpr (I + 1 == K) {
            own[SH::own_off(K) + ch] = fmaf(bs, z[c], own[SH::own_off(K) + ch]);
        } else {
            const float Bc = fmaf(bs, z[c], own[SH::own_off(I + 1) + ch]);
            horner_visit<SH, K, I + 1, ch, NEG>(Bc, own, z);
        }
    }
}

// b = B^(k)_P[p] along the thread's own prefix (B_0 = 1): the scalar part of the chain.
template <class SH, int K, bool NEG, int SZ>
__device__ __forceinline__ float prefix_chain(const float (&own)[SZ], const float (&low)[SH::LOWA],
                                              const float (&zp)[SH::PD]) {
    constexpr int P = SH::P;
    constexpr float sg = NEG ? -1.0f : 1.0f;
    float b = 1.0f;
    static_for<1, P + 1>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        float Ai;
        if constexpr (i < P) Ai = low[i];
        else Ai = own[SH::own_off(P)];
        if constexpr (i == 1) b = fmaf(zp[0], sg * inv_int(K), Ai);
        else if constexpr (SIG_ZS_CSE && !NEG) b = fmaf(b, zp[i - 1] * inv_int(K - i + 1), Ai);
        else b = fmaf(b * (sg * inv_int(K - i + 1)), zp[i - 1], Ai);
    });
    return b;
}

// A <- A [x] exp(z) on owned levels KTOP..K0 (top-down) and then on the replicated prefix levels
// P-1..1.  own: owned coefficients (levels K0..KTOP or more); low[i] (i = 1..P-1): A_i[p_0..p_{i-1}];
// z[c]: the increment; zp[j] = z[p_j].  With z negated this is the reversibility step
// (eq-reverse) used by the backward.
template <class SH, int KTOP, bool NEG, int SZ>
__device__ __forceinline__ void fused_mulexp(float (&own)[SZ], float (&low)[SH::LOWA], const float (&z)[SH::C],
                                             const float (&zp)[SH::PD]) {
    constexpr int P = SH::P;
    constexpr float sg = NEG ? -1.0f : 1.0f;
    static_for<0, (KTOP >= SH::K0 ? KTOP - SH::K0 + 1 : 0)>([&](auto kkc) {
        constexpr int k = KTOP - decltype(kkc)::value;
        const float b = prefix_chain<SH, k, NEG>(own, low, zp);
        if constexpr (k == P) own[SH::own_off(P)] = b;
        else horner_visit<SH, k, P, 0, NEG>(b, own, z);
    });
    static_for<0, (P > 1 ? P - 1 : 0)>([&](auto kkc) {
        constexpr int k = P - 1 - decltype(kkc)::value;
        float b = 1.0f;
        static_for<1, k + 1>([&](auto ic) {
            constexpr int i = decltype(ic)::value;
            if constexpr (i == 1) b = fmaf(zp[0], sg * inv_int(k), low[i]);
            else if constexpr (SIG_ZS_CSE && !NEG) b = fmaf(b, zp[i - 1] * inv_int(k - i + 1), low[i]);
            else b = fmaf(b * (sg * inv_int(k - i + 1)), zp[i - 1], low[i]);
        });
        low[k] = b;
    });
}

// A <- A [x] exp(+-z) for two sibling prefixes pa, pb = pa + 1 held by one thread (same p[:P-1]; the
// last letters are p[P-1] and p[P-1] + 1, zpb = z[p[P-1] + 1]): the prefix chain below level P and
// the replicated low levels are computed once, level P and above per prefix (the two-prefix
// kernels sig_fwd2_kernel / sig_bwd2_kernel; P >= 2).
template <class SH, int KTOP, bool NEG, int SZ>
__device__ __forceinline__ void mulexp2(float (&Aa)[SZ], float (&Ab)[SZ], float (&low)[SH::LOWA], const float (&z)[SH::C],
                                        const float (&zp)[SH::PD], float zpb) {
    constexpr int P = SH::P;
    constexpr float sg = NEG ? -1.0f : 1.0f;
    static_for<0, KTOP - P + 1>([&](auto kkc) {
        constexpr int k = KTOP - decltype(kkc)::value;  // KTOP .. P
        float b = 1.0f;
        static_for<1, P>([&](auto ic) {
            constexpr int i = decltype(ic)::value;
            if constexpr (i == 1) b = fmaf(zp[0], sg * inv_int(k), low[i]);
            else b = fmaf(b * (sg * inv_int(k - i + 1)), zp[i - 1], low[i]);
        });
        const float bs = b * (sg * inv_int(k - P + 1));
        const float ba = fmaf(bs, zp[P - 1], Aa[SH::own_off(P)]);
        const float bb = fmaf(bs, zpb, Ab[SH::own_off(P)]);
        if constexpr (k == P) {
            Aa[SH::own_off(P)] = ba;
            Ab[SH::own_off(P)] = bb;
        } else {
            horner_visit<SH, k, P, 0, NEG>(ba, Aa, z);
            horner_visit<SH, k, P, 0, NEG>(bb, Ab, z);
        }
    });
    static_for<0, P - 1>([&](auto kkc) {
        constexpr int k = P - 1 - decltype(kkc)::value;
        float b = 1.0f;
        static_for<1, k + 1>([&](auto ic) {
            constexpr int i = decltype(ic)::value;
            if constexpr (i == 1) b = fmaf(zp[0], sg * inv_int(k), low[i]);
            else b = fmaf(b * (sg * inv_int(k - i + 1)), zp[i - 1], low[i]);
        });
        low[k] = b;
    });
}

// Write the thread's coefficients of the current state to a row of S floats.
template <class SH, bool STREAMING>
__device__ __forceinline__ void store_state(float* row, int prefix, const float (&own)[SH::OWN],
                                            const float (&low)[SH::LOWA]) {
    static_for<SH::K0, SH::N + 1>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        store_run<SH::own(k), SH::own_off(k), STREAMING>(row + SH::lvl_off(k) + (int64_t)prefix * SH::own(k), own);
    });
    // replicated prefix level i is written by the thread whose trailing digits are zero
    static_for<1, SH::P>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        constexpr int tail = (int)ipow(SH::C, SH::P - i);
        if (prefix % tail == 0) row[SH::lvl_off(i) + prefix / tail] = low[i];
    });
}

// Read a state row into the thread's registers (the inverse of store_state).
template <class SH>
__device__ __forceinline__ void load_state(const float* row, int prefix, float (&own)[SH::OWN], float (&low)[SH::LOWA]) {
    static_for<SH::K0, SH::N + 1>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        load_run<SH::own(k), SH::own_off(k)>(own, row + SH::lvl_off(k) + (int64_t)prefix * SH::own(k));
    });
    static_for<1, SH::P>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        low[i] = row[SH::lvl_off(i) + prefix / (int)ipow(SH::C, SH::P - i)];
    });
}

// In-register right product A <- A [x] B for the thread's share of a state (prefix p of length P:
// own levels >= max(P,1), replicated prefix values low[i] = A_i[p[:i]], i < P), B a full row in
// shared memory.  (A [x] B)_k[w] = A_k[w] + B_k[w] + sum_{i=1}^{k-1} A_i[w[:i]] B_{k-i}[w[i:]]
// (eq-tensorproduct): every A factor along the thread's own words is in its registers,
// every B factor an LDS at a compile-time offset (plus a per-thread base below P).  Levels are
// updated top-down in place (level k reads only levels < k of A and its own coefficient).
template <class SH>
__device__ __forceinline__ void mul_right_regs(float (&own)[SH::OWN], float (&low)[SH::LOWA], const float* Bs,
                                               int prefix) {
    constexpr int C = SH::C, N = SH::N, P = SH::P;
    static_for<0, N - SH::K0 + 1>([&](auto kkc) {
        constexpr int k = N - decltype(kkc)::value;  // N .. K0
        constexpr int NW = SH::own(k);                // C^(k-P) owned words p.w'
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            float acc = own[SH::own_off(k) + w] + Bs[SH::lvl_off(k) + prefix * NW + w];
            static_for<1, k>([&](auto ic) {
                constexpr int i = decltype(ic)::value;
                constexpr int D = (int)ipow(C, k - i);  // size of the B block
                if constexpr (i >= SH::K0) {
                    acc = fmaf(own[SH::own_off(i) + w / D], Bs[SH::lvl_off(k - i) + w % D], acc);
                } else {
                    // A_i[p[:i]] = low[i]; B index (p[i:] . w') = (p mod C^(P-i)) C^(k-P) + w'
                    const int pb = prefix % (int)ipow(C, P - i);
                    acc = fmaf(low[i], Bs[SH::lvl_off(k - i) + pb * NW + w], acc);
                }
            });
            own[SH::own_off(k) + w] = acc;
        }
    });
    static_for<0, (P > 1 ? P - 1 : 0)>([&](auto iic) {
        constexpr int i = P - 1 - decltype(iic)::value;  // P-1 .. 1
        const int pi = prefix / (int)ipow(C, P - i);      // p[:i]
        float acc = low[i] + Bs[SH::lvl_off(i) + pi];
        static_for<1, i>([&](auto jc) {
            constexpr int j = decltype(jc)::value;
            const int pj = pi % (int)ipow(C, i - j);      // p[j:i]
            acc = fmaf(low[j], Bs[SH::lvl_off(i - j) + pj], acc);
        });
        low[i] = acc;
    });
}

// Ordered fold of the nu consecutive units of a CTA (time order = unit order) with the states in
// registers: tree level s, unit u = 2sq + s writes its state to shared-memory slot q, unit 2sq
// multiplies it in from the right (mul_right_regs).  Unit 0 ends with the product.  `slots` holds
// ceil(nu/2) rows of S floats.  Every thread of the CTA must call it.
template <class SH>
__device__ __forceinline__ void fold_units_regs(float (&own)[SH::OWN], float (&low)[SH::LOWA], float* slots, int ul,
                                                int nu, int prefix) {
    for (int st = 1; st < nu; st <<= 1) {
        __syncthreads();  // the previous level's reads of the slots are done
        if (ul % (2 * st) == st) store_state<SH, false>(slots + (size_t)(ul / (2 * st)) * SH::S, prefix, own, low);
        __syncthreads();
        if (ul % (2 * st) == 0 && ul + st < nu) mul_right_regs<SH>(own, low, slots + (size_t)(ul / (2 * st)) * SH::S, prefix);
    }
}

// (a [x] b) at flat coefficient f with compile-time shapes// (a [x] b) at flat coefficient f with compile-time shapes (cf. mul_coef in combine.cuh): the level
// of f selects an unrolled sum whose word splits are divisions by compile-time powers of C.
template <class SH>
__device__ __forceinline__ float mul_coef_t(const float* a, const float* b, int f) {
    constexpr int C = SH::C;
    float r = 0.0f;
    static_for<1, SH::N + 1>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        if (f >= (int)SH::lvl_off(k) && f < (int)SH::lvl_off(k + 1)) {
            const int w = f - (int)SH::lvl_off(k);
            float acc = a[f] + b[f];
            static_for<1, k>([&](auto ic) {
                constexpr int i = decltype(ic)::value;
                constexpr int D = (int)ipow(C, k - i);
                const int u = w / D, v = w - u * D;
                acc = fmaf(a[(int)SH::lvl_off(i) + u], b[(int)SH::lvl_off(k - i) + v], acc);
            });
            r = acc;
        }
    });
    return r;
}

// Ordered tree fold of cnt signatures gs[0..cnt) (time order) with one barrier per tree level:
// level results are written compactly into the other buffer (ping-pong gs <-> tmp, tmp holding
// ceil(cnt/2) signatures).  Returns the buffer holding the product.
template <class SH>
__device__ __forceinline__ const float* block_fold_t(float* gs, float* tmp, int cnt) {
    constexpr int S = (int)SH::S;
    float* src = gs;
    float* dst = tmp;
    while (cnt > 1) {
        const int np = (cnt + 1) / 2;
        for (int e = threadIdx.x; e < np * S; e += blockDim.x) {
            const int pr = e / S, f = e - pr * S;
            const float* x = src + (size_t)(2 * pr) * S;
            dst[e] = (2 * pr + 1 < cnt) ? mul_coef_t<SH>(x, x + S, f) : x[f];
        }
        __syncthreads();
        float* t = src;
        src = dst;
        dst = t;
        cnt = np;
    }
    return src;
}

// K3 group fold compiled per shape: CTA (g, b) folds elements g*G .. g*G+G-1 of path b in time
// order (block_fold_t: one barrier per tree level) -- the fold of the time-chunk partials.
template <class SH>
__global__ void __launch_bounds__(SIG_FOLD_THREADS) fold_group_t_kernel(const GroupParams p) {
    extern __shared__ __align__(16) float gs[];  // [G][S] + [ceil(G/2)][S]
    constexpr int S = (int)SH::S;
    const int64_t g = blockIdx.x;
    const int64_t j0 = g * p.G;
    const int cnt = (int)((p.n - j0) < p.G ? (p.n - j0) : p.G);
    for (int64_t b = blockIdx.y; b < p.B; b += gridDim.y) {  // gridDim.y is capped at 65535
        if (p.in_sj == S) {
            stage_to_smem(gs, p.in + j0 * p.in_sj + b * p.in_sb, cnt * S);
        } else {
            for (int jj = 0; jj < cnt; ++jj) stage_to_smem(gs + (size_t)jj * S, p.in + (j0 + jj) * p.in_sj + b * p.in_sb, S);
        }
        __syncthreads();
        const float* prod = block_fold_t<SH>(gs, gs + (size_t)p.G * S, cnt);
        float* o = p.out + g * p.out_sj + b * p.out_sb;
        for (int f = threadIdx.x; f < S; f += blockDim.x) o[f] = prod[f];
        __syncthreads();
    }
}

// Blocked ordered scan compiled per shape (the time-parallel backward's prefix and suffix products,
// SURVEY 8(f)1): CTA (grp, b) scans elements grp*g .. grp*g+g-1 of path b sequentially in shared
// memory, one barrier per element, started from the carry E (the product of all earlier groups for
// a prefix scan, of all later groups for a suffix scan; none for the first / last group):
//   prefix: Y_0 = E [x] X_0, Y_i = Y_{i-1} [x] X_i;   suffix: Y_{n-1} = X_{n-1} [x] E, Y_i = X_i [x] Y_{i+1}.
// Writes Y to out (if given) and the group total (prefix: Y_{n-1}, suffix: Y_0) to tot[b, grp].
template <class SH>
__global__ void __launch_bounds__(SIG_SCAN_THREADS) scan_group_t_kernel(const ScanParams p) {
    extern __shared__ __align__(16) float ss[];  // X[g][S], Y[g][S], E[S]
    constexpr int S = (int)SH::S;
    const int g = p.g;
    const int64_t ng = (p.m + g - 1) / g;
    const int64_t grp = blockIdx.x;
    const int64_t j0 = grp * g;
    const int cnt = (int)((p.m - j0) < g ? (p.m - j0) : g);
    float* X = ss;
    float* Y = X + (size_t)g * S;
    float* E = Y + (size_t)g * S;
    const bool has_e = p.carry != nullptr && (p.suffix ? grp + 1 < ng : grp > 0);
    for (int64_t b = blockIdx.y; b < p.B; b += gridDim.y) {
        stage_to_smem(X, p.in + ((size_t)b * p.m + j0) * S, cnt * S);
        if (has_e) stage_to_smem(E, p.carry + ((size_t)b * ng + (p.suffix ? grp + 1 : grp - 1)) * S, S);
        __syncthreads();
        for (int ii = 0; ii < cnt; ++ii) {
            const int i = p.suffix ? cnt - 1 - ii : ii;
            const float* l;
            const float* r;
            if (!p.suffix) {
                l = (i == 0) ? (has_e ? E : nullptr) : Y + (size_t)(i - 1) * S;
                r = X + (size_t)i * S;
            } else {
                l = X + (size_t)i * S;
                r = (i == cnt - 1) ? (has_e ? E : nullptr) : Y + (size_t)(i + 1) * S;
            }
            float* y = Y + (size_t)i * S;
            if (l == nullptr) {
                for (int f = threadIdx.x; f < S; f += blockDim.x) y[f] = r[f];
            } else if (r == nullptr) {
                for (int f = threadIdx.x; f < S; f += blockDim.x) y[f] = l[f];
            } else {
                for (int f = threadIdx.x; f < S; f += blockDim.x) y[f] = mul_coef_t<SH>(l, r, f);
            }
            __syncthreads();
        }
        if (p.out) {
            float* dst = p.out + ((size_t)b * p.m + j0) * S;
            for (int e = threadIdx.x; e < cnt * S; e += blockDim.x) dst[e] = Y[e];
        }
        if (p.tot) {
            const float* t = Y + (size_t)(p.suffix ? 0 : cnt - 1) * S;
            float* dst = p.tot + ((size_t)b * ng + grp) * S;
            for (int f = threadIdx.x; f < S; f += blockDim.x) dst[f] = t[f];
        }
        __syncthreads();
    }
}

template <class SH>
cudaError_t launch_scan_group_t(const ScanParams& p, cudaStream_t st) {
    const size_t smem = (size_t)(2 * p.g + 1) * SH::S * sizeof(float);
    if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(scan_group_t_kernel<SH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const int64_t ng = (p.m + p.g - 1) / p.g;
    scan_group_t_kernel<SH><<<dim3((unsigned)ng, p.B < 65535 ? (unsigned)p.B : 65535u), SIG_SCAN_THREADS, smem, st>>>(p);
    return cudaGetLastError();
}

template <class SH>
cudaError_t launch_fold_group_t(const GroupParams& p, unsigned ngroups, unsigned B, cudaStream_t st) {
    const size_t smem = (size_t)(p.G + (p.G + 1) / 2) * SH::S * sizeof(float);
    if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fold_group_t_kernel<SH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    fold_group_t_kernel<SH><<<dim3(ngroups, B < 65535u ? B : 65535u), SIG_FOLD_THREADS, smem, st>>>(p);
    return cudaGetLastError();
}

// Staging of grouped time chunks held in one tile (see sig_fwd_kernel): one bulk copy of the CTA's
// contiguous points, then the increments of all its units.
template <int C>
__device__ __noinline__ void stage_contig_units(const FwdParams& prm, float* zs, uint64_t* bar, unsigned& stage_phase,
                                                int64_t unit0, int nu, int T, int has_bp) {
    float* raw = zs + prm.raw_off;
    const int64_t b0 = unit0 / prm.n_chunks;
    const int64_t j0 = unit0 - b0 * prm.n_chunks;
    const int64_t cl = prm.chunk_len;
    const int64_t s_lo = j0 * cl;                                               // first increment
    const int64_t s_hi = ((j0 + nu) * cl < prm.M ? (j0 + nu) * cl : prm.M);    // one past the last
    const int64_t r_lo = s_lo - has_bp;                                         // its x0 point (-1: basepoint)
    const float* lo = prm.path + (b0 * prm.L + (r_lo < 0 ? 0 : r_lo)) * C;
    const float* hi = prm.path + (b0 * prm.L + (s_hi - has_bp) + 1) * C;        // past the last x1
    const uintptr_t a = reinterpret_cast<uintptr_t>(lo) & ~(uintptr_t)15;
    const uintptr_t e = (reinterpret_cast<uintptr_t>(hi) + 15) & ~(uintptr_t)15;
    if (s_hi > s_lo) {
        if (threadIdx.x == 0) {
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(bar, (unsigned)(e - a));
            bulk_g2s_big(raw, reinterpret_cast<const void*>(a), e - a, bar);
        }
        mbar_wait(bar, stage_phase);
        stage_phase ^= 1u;
    }
    const float* base = raw + ((reinterpret_cast<uintptr_t>(lo) & 15) >> 2);  // point max(r_lo, 0)
    const int TC = T * C;
    for (int uu = 0; uu < nu; ++uu) {  // per unit: no division in the element loop
        const int64_t su = (j0 + uu) * cl;  // the unit's first increment
        const int64_t rem = s_hi - su;
        const int len = (int)(rem <= 0 ? 0 : (rem < cl ? rem : cl));
        const int64_t rel0 = su - s_lo + (r_lo < 0 ? -1 : 0);  // its first x0 row relative to base
        const float* ub = base + rel0 * C;
        float* zu = zs + (size_t)uu * TC;
        for (int i = threadIdx.x; i < TC; i += blockDim.x) {
            float zv = 0.0f;
            if (i < len * C) {
                const float x1 = ub[i + C];
                float x0;
                if (rel0 >= 0 || i >= C) x0 = ub[i];
                else x0 = (prm.bp_mode == 2) ? prm.basepoint[b0 * C + i] : 0.0f;  // the path's first x0
                zv = prm.zsign * (x1 - x0);
            }
            const int t = i / C, c = i - t * C;
            zu[t * C + zswz(C, c)] = zv;
        }
    }
}

// in-CTA fold of grouped time chunks with the states in registers (fold_units_regs); 0: the
// shared-memory tree fold block_fold_t
#ifndef SIG_FOLD_REGS
#define SIG_FOLD_REGS 1
#endif
// grouped chunks in one tile: one bulk copy of the CTA's contiguous points (0: one per unit)
#ifndef SIG_FWD_CONTIG
#define SIG_FWD_CONTIG 1
#endif
template <class SH>
__global__ void __launch_bounds__(512, 1) sig_fwd_kernel(const FwdParams prm) {
    constexpr int C = SH::C;
    extern __shared__ float zs[];  // [units in CTA][tile][C]
    const int64_t g0 = (int64_t)blockIdx.x * blockDim.x;
    const int64_t gt = g0 + threadIdx.x;
    const int64_t unit = gt / SH::CP;
    const int prefix = (int)(gt % SH::CP);
    const int64_t unit0 = g0 / SH::CP;
    const int64_t unit1 = (g0 + blockDim.x - 1) / SH::CP;
    const int nu = (int)(unit1 - unit0 + 1);
    const int ul = (int)(unit - unit0);
    const bool valid = unit < prm.n_units;
    const int64_t b = valid ? unit / prm.n_chunks : 0;
    const int64_t j = valid ? unit % prm.n_chunks : 0;
    const int64_t s0 = j * prm.chunk_len;
    const int64_t my_len = valid ? (prm.chunk_len < prm.M - s0 ? prm.chunk_len : prm.M - s0) : 0;
    const int T = prm.tile;
    const int has_bp = prm.bp_mode != 0;

    int p[SH::PD];
    prefix_digits<SH>(prefix, p);

    float own[SH::OWN];
    float low[SH::LOWA];
#pragma unroll
    for (int i = 0; i < SH::OWN; ++i) own[i] = 0.0f;
#pragma unroll
    for (int i = 0; i < SH::LOWA; ++i) low[i] = 0.0f;
    // the update case: the path's first chunk starts from the given signature
    if (prm.initial != nullptr && valid && j == 0) load_state<SH>(prm.initial + (size_t)b * SH::S, prefix, own, low);

    __shared__ uint64_t stage_bar;
    unsigned stage_phase = 0;
    if (prm.raw_off > 0 && threadIdx.x == 0) mbar_init(&stage_bar, 1);
    for (int64_t t0 = 0; t0 < prm.chunk_len; t0 += T) {
        __syncthreads();
        if (SIG_FWD_CONTIG && prm.raw_off > 0 && prm.upc > 0 && T >= prm.chunk_len) {
            // ---- TMA, grouped chunks in one tile: the CTA's units are consecutive chunks of one
            // path, so their points are ONE contiguous run -- one bulk copy, then all threads form
            // the increments of all units at once (a copy and a serial loop per unit cost c1's
            // latency plan ~0.4 us per unit; c1 10.3 -> 6.2 us per call).  Out of line so that it
            // does not enter the register allocation of the scan loop.
            stage_contig_units<C>(prm, zs, &stage_bar, stage_phase, unit0, nu, T, has_bp);
        } else if (prm.raw_off > 0) {
            // ---- TMA: the 16-byte-aligned cover of every unit's rows, one bulk copy per unit
            float* raw = zs + prm.raw_off;
            const int64_t ru = RawLayout::unit(T, C);
            auto unit_rows = [&](int uu, int64_t& bb, int64_t& r0, int& cnt) {
                const int64_t un = unit0 + uu;
                cnt = 0;
                bb = 0;
                r0 = 0;
                if (un < prm.n_units) {
                    bb = un / prm.n_chunks;
                    const int64_t jj = un - bb * prm.n_chunks;
                    const int64_t ulen = (prm.chunk_len < prm.M - jj * prm.chunk_len ? prm.chunk_len
                                                                                      : prm.M - jj * prm.chunk_len);
                    cnt = (int)(ulen - t0 < T ? (ulen - t0 > 0 ? ulen - t0 : 0) : T);
                    r0 = jj * prm.chunk_len + t0 - has_bp;  // point of the tile's first x0 (-1: basepoint)
                }
            };
            if (threadIdx.x == 0) {
                unsigned total = 0;
                for (int uu = 0; uu < nu; ++uu) {
                    int64_t bb, r0;
                    int cnt;
                    unit_rows(uu, bb, r0, cnt);
                    if (cnt == 0) continue;
                    const float* lo = prm.path + (bb * prm.L + (r0 < 0 ? 0 : r0)) * C;
                    const float* hi = prm.path + (bb * prm.L + r0 + cnt + 1) * C;
                    const uintptr_t a = reinterpret_cast<uintptr_t>(lo) & ~(uintptr_t)15;
                    const uintptr_t e = (reinterpret_cast<uintptr_t>(hi) + 15) & ~(uintptr_t)15;
                    total += (unsigned)(e - a);
                }
                fence_proxy_async_smem();
                mbar_arrive_expect_tx(&stage_bar, total);
                for (int uu = 0; uu < nu; ++uu) {
                    int64_t bb, r0;
                    int cnt;
                    unit_rows(uu, bb, r0, cnt);
                    if (cnt == 0) continue;
                    const float* lo = prm.path + (bb * prm.L + (r0 < 0 ? 0 : r0)) * C;
                    const float* hi = prm.path + (bb * prm.L + r0 + cnt + 1) * C;
                    const uintptr_t a = reinterpret_cast<uintptr_t>(lo) & ~(uintptr_t)15;
                    const uintptr_t e = (reinterpret_cast<uintptr_t>(hi) + 15) & ~(uintptr_t)15;
                    bulk_g2s(raw + uu * ru, reinterpret_cast<const void*>(a), (unsigned)(e - a), &stage_bar);
                }
            }
            mbar_wait(&stage_bar, stage_phase);
            stage_phase ^= 1u;
            for (int uu = 0; uu < nu; ++uu) {
                int64_t bb, r0;
                int cnt;
                unit_rows(uu, bb, r0, cnt);
                const float* lo = prm.path + (bb * prm.L + (r0 < 0 ? 0 : r0)) * C;
                const int sh = (int)((reinterpret_cast<uintptr_t>(lo) & 15) >> 2);  // floats before row max(r0, 0)
                const float* ru_base = raw + uu * ru + sh;  // point row max(r0, 0) of the unit
                float* zu = zs + (size_t)uu * T * C;
                for (int i = threadIdx.x; i < T * C; i += blockDim.x) {
                    const int t = i / C, c = i - (i / C) * C;
                    float zv = 0.0f;
                    if (t < cnt) {
                        const int64_t row = r0 + t;  // x0 = point row, x1 = point row + 1
                        const int64_t rel = row - (r0 < 0 ? 0 : r0);
                        const float x1 = ru_base[(rel + 1) * C + c];
                        const float x0 = (row >= 0) ? ru_base[rel * C + c]
                                                    : ((prm.bp_mode == 2) ? prm.basepoint[bb * C + c] : 0.0f);
                        zv = prm.zsign * (x1 - x0);
                    }
                    zu[t * C + zswz(C, c)] = zv;
                }
            }
        } else
        // ---- stage the increments z = X[s+1] - X[s] of this tile for the CTA's units.  Per unit
        // the points are one contiguous run of the path (coalesced, independent loads unrolled for
        // memory-level parallelism); index math is 32-bit inside the tile.
        for (int uu = 0; uu < nu; ++uu) {
            const int64_t un = unit0 + uu;
            int cnt = 0;          // valid increments of this unit in this tile
            int64_t rowbase = 0;  // element offset of augmented point (s - has_bp) of the tile start
            int64_t bb = 0;
            if (un < prm.n_units) {
                bb = un / prm.n_chunks;
                const int64_t jj = un - bb * prm.n_chunks;
                const int64_t s = jj * prm.chunk_len + t0;
                const int64_t ulen = (prm.chunk_len < prm.M - jj * prm.chunk_len ? prm.chunk_len
                                                                                  : prm.M - jj * prm.chunk_len);
                cnt = (int)(ulen - t0 < T ? (ulen - t0 > 0 ? ulen - t0 : 0) : T);
                rowbase = (bb * prm.L + (s - has_bp)) * C;
            }
            float* zu = zs + (size_t)uu * T * C;
            const float* xb = prm.path;
#pragma unroll 4
            for (int i = threadIdx.x; i < T * C; i += blockDim.x) {
                const int t = i / C, c = i - (i / C) * C;
                float zv = 0.0f;
                if (t < cnt) {
                    const int64_t g0 = rowbase + i;  // point (s + t - has_bp), channel c
                    const float x1 = __ldg(xb + g0 + C);
                    float x0;
                    if (g0 >= bb * prm.L * C) x0 = __ldg(xb + g0);
                    else x0 = (prm.bp_mode == 2) ? prm.basepoint[bb * C + c] : 0.0f;
                    zv = prm.zsign * (x1 - x0);
                }
                zu[t * C + zswz(C, c)] = zv;  // pair-swapped staging when enabled (see zswz)
            }
        }
        __syncthreads();
        const int tl = (int)((int64_t)T < prm.chunk_len - t0 ? (int64_t)T : prm.chunk_len - t0);
        const int tn = (int)((int64_t)tl < my_len - t0 ? (int64_t)tl : (my_len - t0 > 0 ? my_len - t0 : 0));
        // running pointers into the staged increments: z_t and the thread's prefix letters z_t[p_q]
        const float* zrow = zs + (size_t)ul * T * C;
        const float* zq[SH::PD];
#pragma unroll
        for (int q = 0; q < SH::PD; ++q) zq[q] = zrow + (SH::P > 0 ? zswz(C, p[q]) : 0);
        for (int t = 0; t < tn; ++t) {
            float z[C];
            float zp[SH::PD];
#pragma unroll
            for (int c = 0; c < C; ++c) z[c] = zrow[zswz(C, c)];
#pragma unroll
            for (int q = 0; q < SH::PD; ++q) zp[q] = *zq[q];
            zrow += C;
#pragma unroll
            for (int q = 0; q < SH::PD; ++q) zq[q] += C;
            fused_mulexp<SH, SH::N, false>(own, low, z, zp);
            if (prm.stream) {
                float* row = prm.out + ((size_t)b * prm.M + (s0 + t0 + t)) * SH::S;
                store_state<SH, true>(row, prefix, own, low);
            }
        }
    }
    if (prm.upc > 0) {
        // grouped time chunks: this CTA's units are consecutive chunks of one path; fold
        // their signatures in time order in shared memory (Chen's identity, eq-grouplike) and write
        // one partial product.  Units past the end hold the identity (zero state).
#if SIG_FOLD_REGS
        fold_units_regs<SH>(own, low, zs, ul, nu, prefix);
        if (ul == 0) store_state<SH, false>(prm.out + (size_t)blockIdx.x * SH::S, prefix, own, low);
#else
        __syncthreads();
        store_state<SH, false>(zs + (size_t)ul * SH::S, prefix, own, low);
        __syncthreads();
        const float* prod = block_fold_t<SH>(zs, zs + (size_t)nu * SH::S, nu);
        float* o = prm.out + (size_t)blockIdx.x * SH::S;
        for (int f = threadIdx.x; f < (int)SH::S; f += blockDim.x) o[f] = prod[f];
#endif
        return;
    }
    if (valid && !prm.stream) store_state<SH, false>(prm.out + (size_t)unit * SH::S, prefix, own, low);
}

// ---------------------------------------------------------------------------------------------
// Stream mode with staged output (A4): the output [B, M, S] is written once and never
// read back, so the store path decides the speed.  Each thread owns scattered runs of a row (its
// prefix blocks), and storing them directly touches every 32-byte sector several times.  Here a CTA
// holds whole units (paths); every step, its threads write their coefficients into a row image in
// shared memory, and after OT steps one thread writes the unit's OT consecutive rows -- one
// contiguous run of global memory -- with a TMA bulk copy (cp.async.bulk, shared -> global).  The
// run is only 8-byte aligned in general, so the image sits at the same phase mod 16 bytes as its
// global destination; the 16-byte-aligned interior goes by TMA, the <= 3 floats at each end by
// plain stores.  Two images per unit alternate, so the copy of one tile overlaps the next tile.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

struct StreamStage {
    int nu;       // units (paths) per CTA
    int ot;       // steps per output image
    int64_t img;  // floats per image (ot * S + 4, rounded up to 4)
};

__host__ __device__ inline int64_t stream_img_floats(int ot, int64_t S) { return ((int64_t)ot * S + 4 + 3) / 4 * 4; }

template <class SH>
__global__ void __launch_bounds__(512, 1) sig_fwd_stream_kernel(const FwdParams prm, const StreamStage sg) {
    constexpr int C = SH::C;
    constexpr int64_t S = SH::S;
    extern __shared__ __align__(16) float sm[];
    const int nu = sg.nu, OT = sg.ot;
    const int T = prm.tile;
    float* zs = sm;                                        // [nu][T][C]
    float* img = sm + ((int64_t)nu * T * C + 3) / 4 * 4;  // [2][nu][img]
    const int ul = threadIdx.x / SH::CP;
    const int prefix = threadIdx.x % SH::CP;
    const int64_t unit0 = (int64_t)blockIdx.x * nu;
    const int64_t b = unit0 + ul;
    const bool valid = ul < nu && b < prm.B;
    const int has_bp = prm.bp_mode != 0;
    const int64_t M = prm.M;

    int p[SH::PD];
    prefix_digits<SH>(prefix, p);
    float own[SH::OWN];
    float low[SH::LOWA];
#pragma unroll
    for (int i = 0; i < SH::OWN; ++i) own[i] = 0.0f;
#pragma unroll
    for (int i = 0; i < SH::LOWA; ++i) low[i] = 0.0f;
    if (prm.initial != nullptr && valid) load_state<SH>(prm.initial + (size_t)b * S, prefix, own, low);

    // flush image `buf` holding steps [s, s + n) of every unit of the CTA
    auto flush = [&](int buf, int64_t s, int n) {
        fence_proxy_async_smem();
        __syncthreads();
        for (int u = 0; u < nu; ++u) {
            const int64_t bb = unit0 + u;
            if (bb >= prm.B) break;
            const int64_t g0 = (bb * M + s) * S, g1 = g0 + (int64_t)n * S;
            const int ph = (int)(g0 & 3);
            const float* im = img + ((int64_t)buf * nu + u) * sg.img;  // row data at im[ph ..]
            const int64_t a0 = (g0 + 3) & ~(int64_t)3, a1 = g1 & ~(int64_t)3;
            if (a1 > a0) {
                if (threadIdx.x == 0) bulk_s2g(prm.out + a0, im + ph + (a0 - g0), (uint32_t)((a1 - a0) * sizeof(float)));
                const int e = (int)threadIdx.x - 1;  // edges: threads 1..6
                if (e >= 0 && e < 3 && g0 + e < a0) prm.out[g0 + e] = im[ph + e];
                if (e >= 3 && e < 6 && a1 + (e - 3) < g1) prm.out[a1 + (e - 3)] = im[ph + (a1 - g0) + (e - 3)];
            } else {
                for (int64_t g = g0 + threadIdx.x; g < g1; g += blockDim.x) prm.out[g] = im[ph + (g - g0)];
            }
        }
        if (threadIdx.x == 0) {
            bulk_commit();
            bulk_wait_read1();  // the other image (flushed last time) has been read: free to refill
        }
        __syncthreads();
    };

    int buf = 0, fill = 0;  // image being filled, steps in it
    int64_t fs = 0;         // first step of the image
    for (int64_t t0 = 0; t0 < M; t0 += T) {
        __syncthreads();
        for (int uu = 0; uu < nu; ++uu) {
            const int64_t bb = unit0 + uu;
            const int cnt = (bb < prm.B) ? (int)(M - t0 < T ? M - t0 : T) : 0;
            const int64_t rowbase = (bb * prm.L + (t0 - has_bp)) * C;
            float* zu = zs + (size_t)uu * T * C;
            for (int i = threadIdx.x; i < T * C; i += blockDim.x) {
                const int t = i / C, c = i - (i / C) * C;
                float zv = 0.0f;
                if (t < cnt) {
                    const int64_t g = rowbase + i;
                    const float x1 = __ldg(prm.path + g + C);
                    float x0;
                    if (g >= bb * prm.L * C) x0 = __ldg(prm.path + g);
                    else x0 = (prm.bp_mode == 2) ? prm.basepoint[bb * C + c] : 0.0f;
                    zv = prm.zsign * (x1 - x0);
                }
                zu[t * C + zswz(C, c)] = zv;
            }
        }
        __syncthreads();
        const int tl = (int)(M - t0 < T ? M - t0 : T);
        const float* zrow = zs + (size_t)(valid ? ul : 0) * T * C;
        for (int t = 0; t < tl; ++t) {
            float z[C];
            float zp[SH::PD];
#pragma unroll
            for (int c = 0; c < C; ++c) z[c] = zrow[t * C + zswz(C, c)];
#pragma unroll
            for (int q = 0; q < SH::PD; ++q) zp[q] = (SH::P > 0) ? zrow[t * C + zswz(C, p[q])] : 0.0f;
            fused_mulexp<SH, SH::N, false>(own, low, z, zp);
            if (valid) {
                const int64_t g0 = (b * M + fs) * S;
                float* row = img + ((int64_t)buf * nu + ul) * sg.img + (g0 & 3) + (int64_t)fill * S;
                store_state<SH, false>(row, prefix, own, low);
            }
            if (++fill == OT) {
                flush(buf, fs, fill);
                buf ^= 1;
                fs += fill;
                fill = 0;
            }
        }
    }
    if (fill > 0) flush(buf, fs, fill);
    if (threadIdx.x == 0) bulk_wait_all();
}

template <class SH>
cudaError_t launch_fwd_stream_staged(const FwdParams& prm_in, cudaStream_t st, bool* done) {
    *done = false;
    constexpr int64_t S = SH::S;
    constexpr int CP = SH::CP;
    if (!prm_in.stream || prm_in.n_chunks != 1 || CP > 512) return cudaSuccess;
    // units per CTA: enough threads for a few warps, but at least ~2 CTAs per SM
    int nu = 1;
    while ((nu * 2) * CP <= 256 && (prm_in.B + nu * 2 - 1) / (nu * 2) >= 2 * 148) nu *= 2;
    const size_t budget = 100 * 1024;
    int ot = 16;
    while (ot > 1 && 2 * (size_t)nu * stream_img_floats(ot, S) * sizeof(float) > budget) ot /= 2;
    if (2 * (size_t)nu * stream_img_floats(ot, S) * sizeof(float) > budget || ot < 2) return cudaSuccess;
    FwdParams prm = prm_in;
    int tile = (int)(prm.M < 256 ? prm.M : 256);
    while (tile > 8 && (size_t)nu * tile * SH::C * 4 > 16 * 1024) tile /= 2;
    prm.tile = tile;
    StreamStage sg{nu, ot, stream_img_floats(ot, S)};
    const size_t smem = (((size_t)nu * tile * SH::C + 3) / 4 * 4 + 2 * (size_t)nu * sg.img) * sizeof(float);
    if (smem > 227 * 1024) return cudaSuccess;
    auto kern = sig_fwd_stream_kernel<SH>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const int bd = (nu * CP + 31) / 32 * 32;
    const int64_t grid = (prm.B + nu - 1) / nu;
    kern<<<(unsigned)grid, bd, smem, st>>>(prm, sg);
    *done = true;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Forward with two sibling prefixes per thread (cf. sig_bwd2_kernel): one path per CTA of CP/2
// threads; the prefix chains below level P and the replicated low levels are computed once for both
// prefixes.  Plain calls only (no stream, no time chunks, no initial state).
// ---------------------------------------------------------------------------------------------
template <class SH>
struct FwdLayout2 {
    static constexpr int NT = SH::CP / 2;
    // both prefixes' state plus ~48 working registers must fit the per-thread share of the register
    // file (c2's (8,5,3): 2 x 73 at 256 threads; c4's (4,7,4): 2 x 85 at 128 threads)
    static constexpr int REGS = (65536 / (NT > 0 ? NT : 1)) < 255 ? (65536 / (NT > 0 ? NT : 1)) : 255;
    static constexpr bool OK = (SH::C % 2 == 0) && SH::P >= 2 && (NT % 32 == 0) && NT <= 512 &&
                               2 * SH::OWN + 48 <= REGS;
};

template <class SH>
__global__ void __launch_bounds__(FwdLayout2<SH>::NT, 1) sig_fwd2_kernel(const FwdParams prm) {
    constexpr int C = SH::C, P = SH::P;
    extern __shared__ __align__(16) float zs[];  // [T][C]
    const int64_t b = blockIdx.x;
    const int64_t M = prm.M;
    const int T = prm.tile;
    const int has_bp = prm.bp_mode != 0;
    const int pa = 2 * threadIdx.x;
    int p[SH::PD];
    prefix_digits<SH>(pa, p);
    float Aa[SH::OWN], Ab[SH::OWN], low[SH::LOWA];
#pragma unroll
    for (int i = 0; i < SH::OWN; ++i) Aa[i] = Ab[i] = 0.0f;
#pragma unroll
    for (int i = 0; i < SH::LOWA; ++i) low[i] = 0.0f;
    for (int64_t t0 = 0; t0 < M; t0 += T) {
        __syncthreads();
        const int tl = (int)(M - t0 < T ? M - t0 : T);
        const int64_t rowbase = (b * prm.L + (t0 - has_bp)) * C;
        for (int i = threadIdx.x; i < tl * C; i += blockDim.x) {
            const int c = i % C;
            const int64_t g = rowbase + i;
            const float x1 = __ldg(prm.path + g + C);
            float x0;
            if (g >= b * prm.L * C) x0 = __ldg(prm.path + g);
            else x0 = (prm.bp_mode == 2) ? prm.basepoint[b * C + c] : 0.0f;
            zs[i] = prm.zsign * (x1 - x0);
        }
        __syncthreads();
        for (int t = 0; t < tl; ++t) {
            float z[C], zp[SH::PD];
#pragma unroll
            for (int c = 0; c < C; ++c) z[c] = zs[t * C + c];
#pragma unroll
            for (int q = 0; q < SH::PD; ++q) zp[q] = zs[t * C + p[q]];
            const float zpb = zs[t * C + p[P - 1] + 1];
            mulexp2<SH, SH::N, false>(Aa, Ab, low, z, zp, zpb);
        }
    }
    float* row = prm.out + (size_t)b * SH::S;
    store_state<SH, false>(row, pa, Aa, low);
    store_state<SH, false>(row, pa + 1, Ab, low);  // pa + 1 is odd: writes no replicated level
}

#ifndef SIG_FWD2
#define SIG_FWD2 1
#endif

// The two-prefix forward runs one CTA per path: from 64 paths on it beats the wider-prefix
// variant (c2's shape at B = 128: 0.140 ms with P = 4, one CTA per path of 256 threads ~0.04 ms).
constexpr int64_t kFwd2MinBatch = 64;

template <class SH>
cudaError_t launch_fwd(const FwdParams& prm_in, cudaStream_t st) {
    if constexpr (SIG_FWD2 && FwdLayout2<SH>::OK) {
        if (!prm_in.stream && prm_in.n_chunks == 1 && prm_in.upc == 0 && prm_in.initial == nullptr &&
            prm_in.B >= kFwd2MinBatch) {
            FwdParams prm = prm_in;
            prm.tile = (int)(prm.M < 256 ? prm.M : 256);
            const size_t smem = (size_t)prm.tile * SH::C * sizeof(float);
            sig_fwd2_kernel<SH><<<(unsigned)prm.B, FwdLayout2<SH>::NT, smem, st>>>(prm);
            return cudaGetLastError();
        }
    }
#if !defined(SIG_STREAM_DIRECT)
    {
        bool done = false;
        cudaError_t e = launch_fwd_stream_staged<SH>(prm_in, st, &done);
        if (e != cudaSuccess || done) return e;
    }
#endif
    FwdParams prm = prm_in;
    const int64_t threads = prm.n_units * (int64_t)SH::CP;
    int bd = 512;
    if (prm.upc > 0) {
        // grouped chunks: a CTA is exactly upc whole units (no unit straddles two CTAs)
        bd = prm.upc * SH::CP;
    } else {
        // CTA size: units never communicate, so any size works.  Small problems are spread over
        // more SMs (latency-bound, e.g. BASELINE config c1); otherwise pick the size whose CTA count
        // divides most evenly over the 148 SMs (c3 lost 31% to SMs holding 2 CTAs next to SMs
        // holding 1), preferring larger CTAs on ties.
        double best = -1.0;
        for (int cand = 512; cand >= 32; cand /= 2) {
            const int64_t ctas = (threads + cand - 1) / cand;
            const int64_t waves = (ctas + 147) / 148;
            const double eff = (double)ctas / (double)(waves * 148);  // average vs busiest SM
            if (eff > best + 1e-6) {
                best = eff;
                bd = cand;
            }
        }
    }
    const int64_t grid = (threads + bd - 1) / bd;
    const int nu = (prm.upc > 0) ? prm.upc : (int)((bd - 1) / SH::CP + 2);  // max units touched by one CTA
    // grouped chunks (one resident CTA per SM anyway) stage a whole chunk at once: one load phase
    // and one barrier per CTA instead of one per 128 steps (c5 596 -> 504 us); other scans keep
    // 48 KB so that small CTAs still fit several per SM
    const int tmax = prm.upc > 0 ? SIG_FWD_TILE : 256;
    const size_t tkb = prm.upc > 0 ? SIG_FWD_TILE_KB : 48;
    int tile = (int)(prm.chunk_len < tmax ? prm.chunk_len : tmax);
    while (tile > 8 && (size_t)nu * tile * SH::C * 4 > tkb * 1024) tile /= 2;
    prm.tile = tile;
    size_t smem = (size_t)nu * tile * SH::C * sizeof(float);
    // TMA staging of the points (RawLayout) after the increments, 16-byte aligned, when it fits
    prm.raw_off = 0;
    {
        const int64_t ro = ((int64_t)nu * tile * SH::C + 3) / 4 * 4;
        const size_t need = (size_t)(ro + (int64_t)nu * RawLayout::unit(tile, SH::C)) * sizeof(float);
        // the aligned covers stay inside the path tensor when it starts and ends on 16 bytes
        const bool aligned = (reinterpret_cast<uintptr_t>(prm.path) & 15) == 0 && (prm.B * prm.L * SH::C) % 4 == 0;
        if (SIG_FWD_TMA_STAGE && aligned && need <= 160 * 1024) {
            prm.raw_off = ro;
            smem = need;
        }
    }
    // grouped chunks: nu unit signatures plus the fold's second buffer of ceil(nu / 2)
    if (prm.upc > 0 && (size_t)(nu + (nu + 1) / 2) * SH::S * sizeof(float) > smem)
        smem = (size_t)(nu + (nu + 1) / 2) * SH::S * sizeof(float);
    if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(sig_fwd_kernel<SH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    sig_fwd_kernel<SH><<<(unsigned)grid, bd, smem, st>>>(prm);
    return cudaGetLastError();
}

}  // namespace sigb200
