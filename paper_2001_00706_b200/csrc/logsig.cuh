// logsig.cuh -- K4/K5: tensor logarithm + Lyndon projections, and their VJP, sm_100a.
//
// log of a group-like element A = 1 + x as the truncated series
//   log(1 + x) = sum_{n=1}^{N} (-1)^{n+1} x^n / n,
// evaluated in Horner form (reading R7):  H_N = 1/N,  H_n = 1/n - x H_{n+1},  log = x H_1.
// H_n is only needed on levels 0..N-n (it is multiplied by x, which has no scalar part, n times).
// Projections (Appendix A.2): WORDS = psi(log) -- gather the Lyndon coefficients;
// BRACKETS = (psi o phi)^{-1} psi(log) as a sparse mat-vec with the exact integer
// inverse built on the host; EXPAND = log itself.
//
// One CTA (1024 threads) per signature row; x and the H_n live in shared memory.  The series
// cancels heavily at deep levels (at C=4, N=7 a float evaluation loses ~1e-4 relative at level 7
// while the log is well conditioned in its input: ~1e-6), so the forward (K4) computes in float64
// with float32 inputs and outputs; the backward (K5) has no such cancellation and stays float32
// (DESIGN.md "K4").
// Index arithmetic is 32-bit; divisions by C use a precomputed magic multiplier.
#pragma once
#include "combine.cuh"

namespace sigb200 {

struct LogsigTables {
    int w;                        // Witt dimension
    const int64_t* lyn_idx;       // [w] flat index of each Lyndon word
    const int* minv_rowptr;       // [w+1] CSR of (psi o phi)^{-1}
    const int* minv_col;
    const float* minv_val;
    const int* minvT_rowptr;      // [w+1] CSR of its transpose
    const int* minvT_col;
    const float* minvT_val;
};

// 32-bit level tables of one (C, N), built on the host
struct LDims {
    int C, N, S;
    int pw[17];    // C^k
    int off[18];   // flat offset of level k (1-based) in the S layout; off[N+1] = S
    int hoff[18];  // offset of level m (0-based, scalar level 0 included) in an H array
    uint32_t magic;  // n / C == __umulhi(n, magic) for n < 2^24
};

inline LDims make_ldims(int C, int N) {
    LDims d{};
    d.C = C;
    d.N = N;
    d.pw[0] = 1;
    for (int k = 1; k <= 16; ++k) d.pw[k] = (k <= N + 1) ? d.pw[k - 1] * C : 0;
    d.off[1] = 0;
    for (int k = 1; k <= N; ++k) d.off[k + 1] = d.off[k] + d.pw[k];
    d.S = d.off[N + 1];
    d.hoff[0] = 0;
    for (int m = 0; m <= N; ++m) d.hoff[m + 1] = d.hoff[m] + d.pw[m];
    // magic = ceil(2^32 / C): floor(n * magic / 2^32) == floor(n / C) exactly for n < 2^32 / C
    d.magic = (uint32_t)((((uint64_t)1 << 32) + (uint64_t)C - 1) / (uint64_t)C);
    return d;
}

__device__ __forceinline__ int divC(const LDims& d, int n) {
    return (d.C == 1) ? n : (int)__umulhi((uint32_t)n, d.magic);
}

// level of flat coefficient f (1..N) -- at most N compares, no division
__device__ __forceinline__ int lvl_of(const LDims& d, int f) {
    int k = 1;
    while (k < d.N && f >= d.off[k + 1]) ++k;
    return k;
}
// level m of an index e into an H array (levels 0..)
__device__ __forceinline__ int hlvl_of(const LDims& d, int e) {
    int m = 0;
    while (e >= d.hoff[m + 1]) ++m;
    return m;
}

// (x H)_k[w] = sum_{i=1}^{k} x_i[w / C^(k-i)] H_{k-i}[w mod C^(k-i)]   (H given on levels 0..k-1)
__device__ __forceinline__ double xh_coef(const LDims& d, const float* xs, const double* H, int k, int w) {
    double acc = 0.0;
    int u = w, v = 0, q = 1;  // i = k: prefix w, empty suffix
    for (int i = k; i >= 1; --i) {
        acc = fma((double)xs[d.off[i] + u], H[d.hoff[k - i] + v], acc);
        const int u2 = divC(d, u);
        v += (u - u2 * d.C) * q;
        q *= d.C;
        u = u2;
    }
    return acc;
}

struct LogsigParams {
    LDims d;
    int mode;                     // 0 expand, 1 brackets, 2 words
    LogsigTables tb;
    int64_t rows;
    const float* sig;             // [rows, S]
    float* out;                   // fwd: [rows, w|S]
    const float* gout;            // bwd: [rows, w|S]
    float* gsig;                  // bwd: [rows, S] output (accumulated in place)
    float* glog_ws;               // bwd scratch [rows, S]: dense dL/dlog (words / brackets)
    int gl_smem;                  // bwd: dense dL/dlog staged in shared memory (else glog_ws)
};

constexpr int LOGSIG_THREADS = 1024;

#ifdef SIG_DEFINE_LOGSIG_KERNELS  // non-template kernels: defined in api.cu only
__global__ void __launch_bounds__(LOGSIG_THREADS, 1) logsig_fwd_kernel(const LogsigParams p) {
    const LDims& d = p.d;
    const int N = d.N, S = d.S;
    const int64_t row = blockIdx.x;
    extern __shared__ __align__(16) double lsd[];
    const int HS = d.hoff[N];  // levels 0..N-1
    double* Ha = lsd;
    double* Hb = Ha + HS;
    float* xs = reinterpret_cast<float*>(Hb + HS);  // [S]
    float* psi = xs + S;                            // [w] (brackets only)
    const float* src = p.sig + row * S;
    for (int f = threadIdx.x; f < S; f += blockDim.x) xs[f] = src[f];
    if (threadIdx.x == 0) Ha[0] = 1.0 / (double)N;
    __syncthreads();
    double* Hc = Ha;
    double* Hn = Hb;
    for (int n = N - 1; n >= 1; --n) {
        const int top = N - n;  // H_n on levels 0..top
        for (int e = threadIdx.x; e < d.hoff[top + 1]; e += blockDim.x) {
            if (e == 0) {
                Hn[0] = 1.0 / (double)n;
                continue;
            }
            const int m = hlvl_of(d, e);
            Hn[e] = -xh_coef(d, xs, Hc, m, e - d.hoff[m]);
        }
        __syncthreads();
        double* t = Hc;
        Hc = Hn;
        Hn = t;
    }
    // log = x H_1
    if (p.mode == 0) {
        float* o = p.out + row * S;
        for (int f = threadIdx.x; f < S; f += blockDim.x) {
            const int k = lvl_of(d, f);
            o[f] = (float)xh_coef(d, xs, Hc, k, f - d.off[k]);
        }
        return;
    }
    float* o = p.out + row * p.tb.w;
    for (int j = threadIdx.x; j < p.tb.w; j += blockDim.x) {
        const int f = (int)p.tb.lyn_idx[j];
        const int k = lvl_of(d, f);
        const double v = xh_coef(d, xs, Hc, k, f - d.off[k]);
        if (p.mode == 2) o[j] = (float)v;
        else psi[j] = (float)v;
    }
    if (p.mode == 1) {
        __syncthreads();
        // exact integer coefficients of (psi o phi)^{-1}
        for (int r = threadIdx.x; r < p.tb.w; r += blockDim.x) {
            double acc = 0.0;
            for (int e = p.tb.minv_rowptr[r]; e < p.tb.minv_rowptr[r + 1]; ++e)
                acc = fma((double)p.tb.minv_val[e], (double)psi[p.tb.minv_col[e]], acc);
            o[r] = (float)acc;
        }
    }
}

// Reverse mode through the Horner recursion.  With g = dL/dlog:
//   log = x H_1:            gx_i[u] = sum_m sum_v g_{i+m}[u v] H_1,m[v];
//                           gH1_m[v] = sum_i sum_u x_i[u] g_{i+m}[u v]          (m >= 1)
//   H_n = c_n - x H_{n+1}:  gx_i[u] -= sum_m sum_v gHn_{i+m}[u v] H_{n+1},m[v];
//                           gH{n+1}_m[v] = -sum_i sum_u x_i[u] gHn_{i+m}[u v]   (m >= 1)
// float32 arithmetic (the backward has no cancellation problem: ~1e-5 measured vs the 5e-4 bar).
// Every pass is a set of independent dot products of very different lengths (a level-1 coefficient
// sums over most of the tensor, a top-level one over one term), so each pass flattens all its
// outputs into one list of warp slots: short outputs take one lane each, long ones a group of up to
// 32 lanes that split the inner index and combine with an xor-shuffle tree (fixed order:
// deterministic).  gH is double-buffered so all levels of a pass are independent.  Each dL/dSig
// coefficient has one owner and accumulates in place in the output row.
#endif  // SIG_DEFINE_LOGSIG_KERNELS

__device__ __forceinline__ int group_for(int work) {
    int G = 1;
    while (G < 32 && G * 16 < work) G <<= 1;
    return G;
}

__device__ __forceinline__ float group_sum(float v, int G) {
    for (int m = G >> 1; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    return v;
}

#ifdef SIG_DEFINE_LOGSIG_KERNELS  // non-template kernels: defined in api.cu only
__global__ void __launch_bounds__(LOGSIG_THREADS, 1) logsig_bwd_kernel(const LogsigParams p) {
    const LDims& d = p.d;
    const int N = d.N, S = d.S;
    const int64_t row = blockIdx.x;
    extern __shared__ __align__(16) float lsf[];
    const int HS = d.hoff[N];
    auto hb = [&](int n) -> int {  // offset of H_n (levels 0..N-n); H_N first
        int s = 0;
        for (int q = N; q > n; --q) s += d.hoff[N - q + 1];
        return s;
    };
    float* Hall = lsf;                 // all H_n
    float* gHa = Hall + hb(0);         // [HS] dL/dH, double-buffered
    float* gHb = gHa + HS;             // [HS]
    float* xs = gHb + HS;              // [off[N]] levels 1..N-1 of x (level N is never read)
    const float* src = p.sig + row * S;
    for (int f = threadIdx.x; f < d.off[N]; f += blockDim.x) xs[f] = src[f];
    if (threadIdx.x == 0) Hall[hb(N)] = 1.0f / (float)N;
    // dense dL/dlog: shared memory when it fits (the passes below read it many times)
    float* gw = p.gl_smem ? xs + d.off[N] : p.glog_ws + row * S;
    if (p.mode == 0) {
        if (p.gl_smem) {
            const float* go = p.gout + row * S;
            for (int f = threadIdx.x; f < S; f += blockDim.x) gw[f] = go[f];
        } else {
            gw = const_cast<float*>(p.gout + row * S);
        }
    } else {
        for (int f = threadIdx.x; f < S; f += blockDim.x) gw[f] = 0.0f;
    }
    __syncthreads();
    if (p.mode != 0) {
        const float* go = p.gout + row * p.tb.w;
        for (int j = threadIdx.x; j < p.tb.w; j += blockDim.x) {
            double v;
            if (p.mode == 2) {
                v = go[j];
            } else {
                v = 0.0;
                for (int e = p.tb.minvT_rowptr[j]; e < p.tb.minvT_rowptr[j + 1]; ++e)
                    v = fma((double)p.tb.minvT_val[e], (double)go[p.tb.minvT_col[e]], v);
            }
            gw[(int)p.tb.lyn_idx[j]] = (float)v;
        }
    }
    const float* gl = gw;
    for (int n = N - 1; n >= 1; --n) {
        const int top = N - n;
        float* Hn = Hall + hb(n);
        const float* Hc = Hall + hb(n + 1);
        for (int e = threadIdx.x; e < d.hoff[top + 1]; e += blockDim.x) {
            if (e == 0) {
                Hn[0] = 1.0f / (float)n;
                continue;
            }
            const int m = hlvl_of(d, e);
            const int w = e - d.hoff[m];
            float acc = 0.0f;
            int u = w, v = 0, q = 1;
            for (int i = m; i >= 1; --i) {
                acc = fmaf(xs[d.off[i] + u], Hc[d.hoff[m - i] + v], acc);
                const int u2 = divC(d, u);
                v += (u - u2 * d.C) * q;
                q *= d.C;
                u = u2;
            }
            Hn[e] = -acc;
        }
        __syncthreads();
    }
    float* gx = p.gsig + row * S;
    __syncthreads();
    // Both passes walk the output levels in turn; within a level, G lanes (a power of two <= 32,
    // so groups never straddle a warp) share one output.  There is no barrier between levels, so
    // threads done with a small level go straight on to the next one.
    auto lg2 = [](int G) { return 31 - __clz(G); };
    // gx_i[u] (+)= sgn * sum_{m=0}^{top-i} sum_v src_{i+m}[u C^m + v] * Hm[v],  i = 1..top
    // src(level k, idx) = gl[off[k] + idx] (step A) or gHs[hoff[k] + idx]
    auto gx_pass = [&](int top, const float* gHs, const float* Hm, float sgn, bool init) {
        for (int i = 1; i <= top; ++i) {
            const int nout = d.pw[i];
            const int G = group_for(d.hoff[top - i + 1]), sh = lg2(G);
            const int items = ((nout << sh) + 31) & ~31;
            for (int idx = threadIdx.x; idx < items; idx += blockDim.x) {
                const int u = idx >> sh, gq = idx & (G - 1);
                float acc = 0.0f;
                if (u < nout) {
                    const float* sb = gHs ? gHs + d.hoff[i] : gl + d.off[i];
                    for (int m = 0; m <= top - i; ++m) {
                        const int nv = d.pw[m];
                        const float* srow = sb + u * nv;
                        const float* hrow = Hm + d.hoff[m];
#pragma unroll 4
                        for (int v = gq; v < nv; v += G) acc = fmaf(srow[v], hrow[v], acc);
                        sb += d.pw[i + m];  // next level's block
                    }
                }
                acc = group_sum(acc, G);
                if (gq == 0 && u < nout) {
                    float* dst = &gx[d.off[i] + u];
                    *dst = init ? sgn * acc : fmaf(sgn, acc, *dst);
                }
            }
        }
    };
    // gHo_m[v] = sgn * sum_{i=1}^{top-m} sum_u x_i[u] src_{i+m}[u C^m + v],  m = 1..top-1
    auto gh_pass = [&](int top, const float* gHs, float* gHo, float sgn) {
        for (int m = 1; m <= top - 1; ++m) {
            const int nout = d.pw[m];
            const int G = group_for(d.off[top - m + 1]), sh = lg2(G);
            const int items = ((nout << sh) + 31) & ~31;
            for (int idx = threadIdx.x; idx < items; idx += blockDim.x) {
                const int v = idx >> sh, gq = idx & (G - 1);
                float acc = 0.0f;
                if (v < nout) {
                    const int stride = nout;
                    for (int i = 1; i <= top - m; ++i) {
                        const int nu = d.pw[i];
                        const float* xrow = xs + d.off[i];
                        const float* srow = gHs ? gHs + d.hoff[i + m] + v : gl + d.off[i + m] + v;
#pragma unroll 4
                        for (int u = gq; u < nu; u += G) acc = fmaf(xrow[u], srow[u * stride], acc);
                    }
                }
                acc = group_sum(acc, G);
                if (gq == 0 && v < nout) gHo[d.hoff[m] + v] = sgn * acc;
            }
        }
    };
    // step A: log = x H_1 (H_1 on levels 0..N-1)
    gx_pass(N, nullptr, Hall + hb(1), 1.0f, true);
    gh_pass(N, nullptr, gHa, 1.0f);
    __syncthreads();
    float* gc = gHa;
    float* gn = gHb;
    for (int n = 1; n <= N - 1; ++n) {
        const int top = N - n;  // gc = dL/dH_n on levels 1..top
        gx_pass(top, gc, Hall + hb(n + 1), -1.0f, false);
        if (n <= N - 2) gh_pass(top, gc, gn, -1.0f);
        __syncthreads();
        float* t = gc;
        gc = gn;
        gn = t;
    }
}

#endif  // SIG_DEFINE_LOGSIG_KERNELS

// ---------------------------------------------------------------------------------------------
// K5, owned-prefix form (used whenever its shared-memory layout fits; logsig_bwd_kernel above is
// the general fallback).  Each pass of the Horner VJP is a pair of contractions of a source
// tensor s (dL/dlog, then dL/dH_n) on levels 1..top:
//   GX: gx_i[u]  (+)= sgn * sum_{m=0}^{top-i} sum_v s_{i+m}[u v] H_m[v]          (trailing contraction)
//   GH: gH_m[v]   = sgn * sum_{i=1}^{top-m} sum_u x_i[u] s_{i+m}[u v]            (leading contraction)
// GX is split by word PREFIX: thread p (a word of length P' = min(P, top)) computes every output
// gx_i[u] with u[:P'] = p outright (i >= P'), and for i < P' one partial over the words it owns,
// which an aligned block of C^(P'-i) threads then sums.  GH is split the same way by word SUFFIX.
// Every thread does about the same number of FMAs; source reads are thread-strided blocks, so the
// shared arrays carry one pad float per 32 (lpad) to keep them conflict-free.  All sums have a
// fixed order.
__host__ __device__ constexpr inline int lpad(int e) { return e + (e >> 5); }

struct OwnedLayout {
    int P;                                       // ownership prefix length (C^P <= 1024)
    int o_gha, o_ghb, o_xs, o_gl, o_scr, total;  // float offsets into shared memory (H_n at 0)
};

__host__ __device__ inline int hall_size(const LDims& d) {
    int hall = 0;
    for (int n = 1; n <= d.N; ++n) hall += d.hoff[d.N - n + 1];
    return hall;
}

__host__ __device__ inline OwnedLayout owned_layout(const LDims& d) {
    OwnedLayout L;
    int P = 1;
    while (P < d.N && d.pw[P + 1] <= LOGSIG_THREADS) ++P;
    L.P = P;
    const int hs = d.hoff[d.N];
    const int scr = (P > 1 ? P - 1 : 1) * d.pw[P];
    L.o_gha = lpad(hall_size(d)) + 1;
    L.o_ghb = L.o_gha + lpad(hs) + 1;
    L.o_xs = L.o_ghb + lpad(hs) + 1;
    L.o_gl = L.o_xs + d.off[d.N];
    L.o_scr = L.o_gl + lpad(d.S) + 1;
    L.total = L.o_scr + lpad(scr) + 1;
    return L;
}

// sum aligned blocks of a partial row: level l (1..Lp-1) has C^l outputs, each the sum of the
// C^(Lp-l) consecutive entries of row l-1 (rows of np entries); G lanes per output
template <class Emit>
__device__ __forceinline__ void owned_block_reduce(const LDims& d, const float* scr, int Lp, int np, Emit&& emit) {
    for (int l = 1; l < Lp; ++l) {
        const int nout = d.pw[l], bs = d.pw[Lp - l];
        int G = 1;
        while (G < 32 && 2 * G <= bs) G <<= 1;
        const int sh = 31 - __clz(G);
        const int items = ((nout << sh) + 31) & ~31;
        for (int idx = threadIdx.x; idx < items; idx += blockDim.x) {
            const int o = idx >> sh, g = idx & (G - 1);
            float sum = 0.0f;
            if (o < nout) {
                const int base = (l - 1) * np + o * bs;
                for (int e = g; e < bs; e += G) sum += scr[lpad(base + e)];
            }
            for (int q = G >> 1; q >= 1; q >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, q);
            if (g == 0 && o < nout) emit(l, o, sum);
        }
    }
}

// one pass: src levels k at src[lpad(soff[k] + idx)], H_m at Hall[lpad(hbase + hoff[m] + idx)]
__device__ __forceinline__ void owned_pass(const LDims& d, int P, int top, const float* src, const int* soff,
                                           const float* Hall, int hbase, const float* xs, float* scr, float* gx,
                                           float* gHo, float sgn, bool init) {
    const int tid = threadIdx.x, nth = blockDim.x;
    auto Sv = [&](int e) { return src[lpad(e)]; };
    auto Hv = [&](int e) { return Hall[lpad(hbase + e)]; };
    // ---- GX, by prefix
    const int Pg = P < top ? P : top;
    const int np = d.pw[Pg];
    for (int pf = tid; pf < np; pf += nth) {
        for (int i = Pg; i <= top; ++i) {  // owned outputs u = pf u'
            const int nu = d.pw[i - Pg];
            for (int up = 0; up < nu; ++up) {
                const int u = pf * nu + up;
                float acc = 0.0f;
                for (int m = 0; m <= top - i; ++m) {
                    const int nv = d.pw[m];
                    const int rb = soff[i + m] + u * nv, hb0 = d.hoff[m];
                    for (int v = 0; v < nv; ++v) acc = fmaf(Sv(rb + v), Hv(hb0 + v), acc);
                }
                float* dst = gx + d.off[i] + u;
                *dst = init ? sgn * acc : fmaf(sgn, acc, *dst);
            }
        }
        for (int i = 1; i < Pg; ++i) {  // partial of gx_i[p[:i]] over the words this thread owns
            const int ps = pf % d.pw[Pg - i];  // p[i:]
            float acc = 0.0f;
            for (int k = Pg; k <= top; ++k) {  // words p v'
                const int nv = d.pw[k - Pg];
                const int sb = soff[k] + pf * nv, hb0 = d.hoff[k - i] + ps * nv;
                for (int v = 0; v < nv; ++v) acc = fmaf(Sv(sb + v), Hv(hb0 + v), acc);
            }
            for (int k = i; k < Pg; ++k) {  // short words w (|w| = k < P'), owned by p = w 0..0
                const int q = d.pw[Pg - k];
                if (pf % q == 0) {
                    const int w = pf / q;
                    acc = fmaf(Sv(soff[k] + w), Hv(d.hoff[k - i] + w % d.pw[k - i]), acc);
                }
            }
            scr[lpad((i - 1) * np + pf)] = acc;
        }
    }
    __syncthreads();
    owned_block_reduce(d, scr, Pg, np, [&](int i, int u, float sum) {
        float* dst = gx + d.off[i] + u;
        *dst = init ? sgn * sum : fmaf(sgn, sum, *dst);
    });
    if (!gHo || top < 2) return;
    __syncthreads();  // scratch reuse
    // ---- GH, by suffix
    const int Ph = P < top - 1 ? P : top - 1;
    const int ns = d.pw[Ph];
    for (int sf = tid; sf < ns; sf += nth) {
        for (int m = Ph; m <= top - 1; ++m) {  // owned outputs v = v'' s
            const int nvv = d.pw[m - Ph], stride = d.pw[m];
            for (int vv = 0; vv < nvv; ++vv) {
                const int v = vv * ns + sf;
                float acc = 0.0f;
                for (int i = 1; i <= top - m; ++i) {
                    const int nu = d.pw[i], xb = d.off[i], sb = soff[i + m] + v;
                    for (int u = 0; u < nu; ++u) acc = fmaf(xs[xb + u], Sv(sb + u * stride), acc);
                }
                gHo[lpad(d.hoff[m] + v)] = sgn * acc;
            }
        }
        for (int m = 1; m < Ph; ++m) {  // partial of gH_m[s[Ph-m:]] over the words this thread owns
            const int cm = d.pw[m], sq = sf / cm, cq = d.pw[Ph - m];
            float acc = 0.0f;
            for (int k = Ph; k <= top; ++k) {  // words y s, split u = (y s)[:k-m]
                const int ny = d.pw[k - Ph], xb = d.off[k - m] + sq, sb = soff[k] + sf;
                for (int y = 0; y < ny; ++y) acc = fmaf(xs[xb + y * cq], Sv(sb + y * ns), acc);
            }
            for (int k = m + 1; k < Ph; ++k)  // short words w = s (|w| = k), owned by s = 0..0 w
                if (sf < d.pw[k]) acc = fmaf(xs[d.off[k - m] + sq], Sv(soff[k] + sf), acc);
            scr[lpad((m - 1) * ns + (sf % cm) * cq + sq)] = acc;  // grouped by output
        }
    }
    __syncthreads();
    owned_block_reduce(d, scr, Ph, ns, [&](int m, int v, float sum) { gHo[lpad(d.hoff[m] + v)] = sgn * sum; });
}

#ifdef SIG_DEFINE_LOGSIG_KERNELS  // non-template kernels: defined in api.cu only
__global__ void __launch_bounds__(LOGSIG_THREADS, 1) logsig_bwd_owned_kernel(const LogsigParams p) {
    const LDims& d = p.d;
    const int N = d.N, S = d.S;
    const int64_t row = blockIdx.x;
    const OwnedLayout L = owned_layout(d);
    extern __shared__ __align__(16) float lsf[];
    auto hb = [&](int n) -> int {  // offset of H_n (levels 0..N-n) in Hall; H_N first
        int s = 0;
        for (int q = N; q > n; --q) s += d.hoff[N - q + 1];
        return s;
    };
    float* Hall = lsf;
    float* gHa = lsf + L.o_gha;
    float* gHb = lsf + L.o_ghb;
    float* xs = lsf + L.o_xs;  // levels 1..N-1 of x
    float* gl = lsf + L.o_gl;  // dense dL/dlog, padded
    float* scr = lsf + L.o_scr;
    const float* sg = p.sig + row * S;
    for (int f = threadIdx.x; f < d.off[N]; f += blockDim.x) xs[f] = sg[f];
    if (threadIdx.x == 0) Hall[lpad(hb(N))] = 1.0f / (float)N;
    if (p.mode == 0) {
        const float* go = p.gout + row * S;
        for (int f = threadIdx.x; f < S; f += blockDim.x) gl[lpad(f)] = go[f];
    } else {
        for (int f = threadIdx.x; f < S; f += blockDim.x) gl[lpad(f)] = 0.0f;
        __syncthreads();
        const float* go = p.gout + row * p.tb.w;
        for (int j = threadIdx.x; j < p.tb.w; j += blockDim.x) {
            double v;
            if (p.mode == 2) {
                v = go[j];
            } else {
                v = 0.0;
                for (int e = p.tb.minvT_rowptr[j]; e < p.tb.minvT_rowptr[j + 1]; ++e)
                    v = fma((double)p.tb.minvT_val[e], (double)go[p.tb.minvT_col[e]], v);
            }
            gl[lpad((int)p.tb.lyn_idx[j])] = (float)v;
        }
    }
    __syncthreads();
    // recompute H_{N-1} .. H_1 (float: the VJP has no cancellation problem)
    for (int n = N - 1; n >= 1; --n) {
        const int top = N - n, bn = hb(n), bc = hb(n + 1);
        for (int e = threadIdx.x; e < d.hoff[top + 1]; e += blockDim.x) {
            float val = 1.0f / (float)n;
            if (e > 0) {
                const int m = hlvl_of(d, e);
                float acc = 0.0f;
                int u = e - d.hoff[m], v = 0, q = 1;
                for (int i = m; i >= 1; --i) {
                    acc = fmaf(xs[d.off[i] + u], Hall[lpad(bc + d.hoff[m - i] + v)], acc);
                    const int u2 = divC(d, u);
                    v += (u - u2 * d.C) * q;
                    q *= d.C;
                    u = u2;
                }
                val = -acc;
            }
            Hall[lpad(bn + e)] = val;
        }
        __syncthreads();
    }
    float* gx = p.gsig + row * S;
    // step A: log = x H_1
    owned_pass(d, L.P, N, gl, d.off, Hall, hb(1), xs, scr, gx, N >= 2 ? gHa : nullptr, 1.0f, true);
    __syncthreads();
    float* gc = gHa;
    float* gn = gHb;
    for (int n = 1; n <= N - 1; ++n) {  // H_n = 1/n - x H_{n+1}; gc = dL/dH_n on levels 1..N-n
        owned_pass(d, L.P, N - n, gc, d.hoff, Hall, hb(n + 1), xs, scr, gx, n <= N - 2 ? gn : nullptr, -1.0f,
                   false);
        __syncthreads();
        float* t = gc;
        gc = gn;
        gn = t;
    }
}

#endif  // SIG_DEFINE_LOGSIG_KERNELS

inline size_t logsig_bwd_owned_smem(const LDims& d) { return (size_t)owned_layout(d).total * sizeof(float); }

inline size_t logsig_fwd_smem(const LDims& d, int w, bool brackets) {
    return (size_t)(2 * d.hoff[d.N]) * sizeof(double) + (size_t)(d.S + (brackets ? w : 0)) * sizeof(float);
}

inline size_t logsig_bwd_smem(const LDims& d, bool gl_smem) {
    int hall = 0;
    for (int n = 1; n <= d.N; ++n) hall += d.hoff[d.N - n + 1];
    return (size_t)(hall + 2 * d.hoff[d.N] + d.off[d.N] + (gl_smem ? d.S : 0)) * sizeof(float);
}

}  // namespace sigb200
