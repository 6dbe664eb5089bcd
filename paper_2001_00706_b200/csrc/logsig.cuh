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
};

constexpr int LOGSIG_THREADS = 1024;

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
__device__ __forceinline__ int group_for(int work) {
    int G = 1;
    while (G < 32 && G * 16 < work) G <<= 1;
    return G;
}

__device__ __forceinline__ float group_sum(float v, int G) {
    for (int m = G >> 1; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    return v;
}

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
    float* xs = gHb + HS;              // [S]
    const float* src = p.sig + row * S;
    for (int f = threadIdx.x; f < S; f += blockDim.x) xs[f] = src[f];
    if (threadIdx.x == 0) Hall[hb(N)] = 1.0f / (float)N;
    __syncthreads();
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
    // dense dL/dlog
    const float* gl;
    if (p.mode == 0) {
        gl = p.gout + row * S;
    } else {
        float* gw = p.glog_ws + row * S;
        for (int f = threadIdx.x; f < S; f += blockDim.x) gw[f] = 0.0f;
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
            gw[(int)p.tb.lyn_idx[j]] = (float)v;
        }
        gl = gw;
    }
    float* gx = p.gsig + row * S;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;

    // Work lists: level l of a pass needs ns[l] warp slots of (32 / G[l]) outputs each.
    __shared__ int s_G[17], s_ns[17];
    auto plan_pass = [&](int lo, int hi, bool gx_kind, int top) {
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int l = lo; l <= hi; ++l) {
                const int work = gx_kind ? d.hoff[top - l + 1] : d.off[top - l + 1];
                const int G = group_for(work);
                s_G[l] = G;
                s_ns[l] = (d.pw[l] * G + 31) / 32;
            }
        }
        __syncthreads();
    };
    // gx_i[u] (+)= sgn * sum_{m=0}^{top-i} sum_v src_{i+m}[u C^m + v] * Hm[v],  i = 1..top
    // src(level k, idx) = gl[off[k] + idx] (step A) or gHs[hoff[k] + idx]
    auto gx_pass = [&](int top, const float* gHs, const float* Hm, float sgn, bool init) {
        plan_pass(1, top, true, top);
        int total = 0;
        for (int i = 1; i <= top; ++i) total += s_ns[i];
        for (int slot = warp; slot < total; slot += nwarps) {
            int i = 1, base = slot;
            while (base >= s_ns[i]) {
                base -= s_ns[i];
                ++i;
            }
            const int G = s_G[i];
            const int u = base * (32 / G) + lane / G, gq = lane % G;
            float acc = 0.0f;
            if (u < d.pw[i]) {
                for (int m = 0; m <= top - i; ++m) {
                    const int nv = d.pw[m];
                    const float* srow = gHs ? gHs + d.hoff[i + m] + u * nv : gl + d.off[i + m] + u * nv;
                    const float* hrow = Hm + d.hoff[m];
                    for (int v = gq; v < nv; v += G) acc = fmaf(srow[v], hrow[v], acc);
                }
            }
            acc = group_sum(acc, G);
            if (gq == 0 && u < d.pw[i]) {
                float* dst = &gx[d.off[i] + u];
                *dst = init ? sgn * acc : fmaf(sgn, acc, *dst);
            }
        }
    };
    // gHo_m[v] = sgn * sum_{i=1}^{top-m} sum_u x_i[u] src_{i+m}[u C^m + v],  m = 1..top-1
    auto gh_pass = [&](int top, const float* gHs, float* gHo, float sgn) {
        if (top < 2) return;
        plan_pass(1, top - 1, false, top);
        int total = 0;
        for (int m = 1; m <= top - 1; ++m) total += s_ns[m];
        for (int slot = warp; slot < total; slot += nwarps) {
            int m = 1, base = slot;
            while (base >= s_ns[m]) {
                base -= s_ns[m];
                ++m;
            }
            const int G = s_G[m];
            const int v = base * (32 / G) + lane / G, gq = lane % G;
            float acc = 0.0f;
            if (v < d.pw[m]) {
                const int stride = d.pw[m];
                for (int i = 1; i <= top - m; ++i) {
                    const int nu = d.pw[i];
                    const float* xrow = xs + d.off[i];
                    const float* srow = gHs ? gHs + d.hoff[i + m] + v : gl + d.off[i + m] + v;
                    for (int u = gq; u < nu; u += G) acc = fmaf(xrow[u], srow[u * stride], acc);
                }
            }
            acc = group_sum(acc, G);
            if (gq == 0 && v < d.pw[m]) gHo[d.hoff[m] + v] = sgn * acc;
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

inline size_t logsig_fwd_smem(const LDims& d, int w, bool brackets) {
    return (size_t)(2 * d.hoff[d.N]) * sizeof(double) + (size_t)(d.S + (brackets ? w : 0)) * sizeof(float);
}

inline size_t logsig_bwd_smem(const LDims& d) {
    int hall = 0;
    for (int n = 1; n <= d.N; ++n) hall += d.hoff[d.N - n + 1];
    return (size_t)(hall + 2 * d.hoff[d.N] + d.S) * sizeof(float);
}

}  // namespace sigb200
