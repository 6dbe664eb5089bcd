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
// One CTA per signature row; x (float, as stored) and the H_n (double) live in shared memory.
// The series cancels heavily at deep levels (at C=4, N=7 the float evaluation loses ~1e-4
// relative at level 7 while the log is well conditioned in its input: ~1e-6), so the
// arithmetic of K4/K5 is float64 with float32 inputs and outputs.  The work is
// ~N*S FMAs per row (about 2-5% of the scan at the BASELINE shapes): a latency-bound epilogue,
// not a roofline kernel.  The backward (K5) walks the Horner recursion in reverse and produces the
// dense gradient w.r.t. the signature that seeds the reversible signature backward (K2).
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

struct LogsigParams {
    TensorDims d;
    int mode;                     // 0 expand, 1 brackets, 2 words
    LogsigTables tb;
    int64_t rows;
    const float* sig;             // [rows, S]
    float* out;                   // fwd: [rows, w|S]
    const float* gout;            // bwd: [rows, w|S]
    float* gsig;                  // bwd: [rows, S] output
    float* glog_ws;               // bwd scratch [rows, S] (brackets/words)
};

__device__ __forceinline__ int64_t hoff(const TensorDims& d, int m) {  // levels 0..m-1 sizes
    int64_t s = 0;
    for (int j = 0; j < m; ++j) s += d.pw[j];
    return s;
}

// (x H)_k[w] = sum_{i=1}^{k} x_i[w / C^(k-i)] H_{k-i}[w mod C^(k-i)]   (H given on levels 0..k-1)
__device__ __forceinline__ double xh_coef(const TensorDims& d, const float* xs, const double* H, int k, int64_t w) {
    double acc = 0.0;
    for (int i = 1; i <= k; ++i) {
        const int64_t q = d.pw[k - i];
        acc = fma((double)xs[d.off[i] + w / q], H[hoff(d, k - i) + w % q], acc);
    }
    return acc;
}

__global__ void logsig_fwd_kernel(const LogsigParams p) {
    const TensorDims& d = p.d;
    const int N = d.N;
    const int64_t S = d.S;
    const int64_t row = blockIdx.x;
    extern __shared__ __align__(16) double lsd[];
    const int64_t HS = hoff(d, N);  // levels 0..N-1
    double* Ha = lsd;
    double* Hb = Ha + HS;
    float* xs = reinterpret_cast<float*>(Hb + HS);  // [S]
    float* psi = xs + S;                            // [w] (brackets only)
    const float* src = p.sig + row * S;
    for (int64_t f = threadIdx.x; f < S; f += blockDim.x) xs[f] = src[f];
    if (threadIdx.x == 0) Ha[0] = 1.0 / (double)N;
    __syncthreads();
    double* Hc = Ha;
    double* Hn = Hb;
    for (int n = N - 1; n >= 1; --n) {
        const int top = N - n;  // H_n on levels 0..top
        for (int64_t e = threadIdx.x; e < hoff(d, top + 1); e += blockDim.x) {
            if (e == 0) {
                Hn[0] = 1.0 / (double)n;
                continue;
            }
            int m = 1;
            while (e >= hoff(d, m + 1)) ++m;
            Hn[e] = -xh_coef(d, xs, Hc, m, e - hoff(d, m));
        }
        __syncthreads();
        double* t = Hc;
        Hc = Hn;
        Hn = t;
    }
    // log = x H_1
    if (p.mode == 0) {
        float* o = p.out + row * S;
        for (int64_t f = threadIdx.x; f < S; f += blockDim.x) {
            const int k = level_of(d, f);
            o[f] = (float)xh_coef(d, xs, Hc, k, f - d.off[k]);
        }
        return;
    }
    float* o = p.out + row * p.tb.w;
    for (int j = threadIdx.x; j < p.tb.w; j += blockDim.x) {
        const int64_t f = p.tb.lyn_idx[j];
        const int k = level_of(d, f);
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
// Every thread owns a fixed set of gx coefficients across the steps (no races, fixed order).
__global__ void logsig_bwd_kernel(const LogsigParams p) {
    const TensorDims& d = p.d;
    const int N = d.N;
    const int64_t S = d.S;
    const int64_t row = blockIdx.x;
    extern __shared__ __align__(16) double lsd[];
    const int64_t HS = hoff(d, N);
    auto hb = [&](int n) -> int64_t {  // offset of H_n (levels 0..N-n) in Hall
        int64_t s = 0;
        for (int q = N; q > n; --q) s += hoff(d, N - q + 1);
        return s;
    };
    double* Hall = lsd;
    double* gH = Hall + hb(0);                      // [HS] gradient of the current H_n (in place)
    float* xs = reinterpret_cast<float*>(gH + HS);  // [S]
    const float* src = p.sig + row * S;
    for (int64_t f = threadIdx.x; f < S; f += blockDim.x) xs[f] = src[f];
    if (threadIdx.x == 0) Hall[hb(N)] = 1.0 / (double)N;
    __syncthreads();
    for (int n = N - 1; n >= 1; --n) {
        const int top = N - n;
        double* Hn = Hall + hb(n);
        const double* Hc = Hall + hb(n + 1);
        for (int64_t e = threadIdx.x; e < hoff(d, top + 1); e += blockDim.x) {
            if (e == 0) {
                Hn[0] = 1.0 / (double)n;
                continue;
            }
            int m = 1;
            while (e >= hoff(d, m + 1)) ++m;
            Hn[e] = -xh_coef(d, xs, Hc, m, e - hoff(d, m));
        }
        __syncthreads();
    }
    // dense dL/dlog (float32 in the workspace for words/brackets)
    const float* g;
    if (p.mode == 0) {
        g = p.gout + row * S;
    } else {
        float* gw = p.glog_ws + row * S;
        for (int64_t f = threadIdx.x; f < S; f += blockDim.x) gw[f] = 0.0f;
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
            gw[p.tb.lyn_idx[j]] = (float)v;
        }
        __syncthreads();
        g = gw;
    }
    float* gx = p.gsig + row * S;
    // step A: log = x H_1 (H_1 on levels 0..N-1)
    {
        const double* H1 = Hall + hb(1);
        for (int64_t f = threadIdx.x; f < S; f += blockDim.x) {
            const int i = level_of(d, f);
            const int64_t u = f - d.off[i];
            double acc = 0.0;
            for (int m = 0; m <= N - i; ++m) {
                const int64_t nv = d.pw[m];
                const float* gk = g + d.off[i + m] + u * nv;
                const double* hm = H1 + hoff(d, m);
                for (int64_t v = 0; v < nv; ++v) acc = fma((double)gk[v], hm[v], acc);
            }
            gx[f] = (float)acc;
        }
        for (int64_t e = threadIdx.x; e < HS; e += blockDim.x) {
            if (e == 0) continue;
            int m = 1;
            while (e >= hoff(d, m + 1)) ++m;
            const int64_t v = e - hoff(d, m);
            double acc = 0.0;
            for (int i = 1; i <= N - m; ++i) {
                const int64_t nu = d.pw[i];
                const float* gk = g + d.off[i + m] + v;
                const float* xi = xs + d.off[i];
                for (int64_t u = 0; u < nu; ++u) acc = fma((double)xi[u], (double)gk[u * d.pw[m]], acc);
            }
            gH[e] = acc;
        }
        __syncthreads();
    }
    for (int n = 1; n <= N - 1; ++n) {
        const int top = N - n;  // gH = dL/dH_n on levels 1..top
        const double* Hnext = Hall + hb(n + 1);  // levels 0..top-1
        for (int64_t f = threadIdx.x; f < d.off[top + 1]; f += blockDim.x) {
            const int i = level_of(d, f);
            const int64_t u = f - d.off[i];
            double acc = 0.0;
            for (int m = 0; m <= top - i; ++m) {
                const int64_t nv = d.pw[m];
                const double* gk = gH + hoff(d, i + m) + u * nv;
                const double* hm = Hnext + hoff(d, m);
                for (int64_t v = 0; v < nv; ++v) acc = fma(gk[v], hm[v], acc);
            }
            gx[f] = (float)((double)gx[f] - acc);
        }
        __syncthreads();
        // dL/dH_{n+1} in place, level by level upward: level m reads only levels > m
        if (n <= N - 2) {
            for (int m = 1; m <= top - 1; ++m) {
                for (int64_t v = threadIdx.x; v < d.pw[m]; v += blockDim.x) {
                    double acc = 0.0;
                    for (int i = 1; i <= top - m; ++i) {
                        const int64_t nu = d.pw[i];
                        const double* gk = gH + hoff(d, i + m) + v;
                        const float* xi = xs + d.off[i];
                        for (int64_t u = 0; u < nu; ++u) acc = fma((double)xi[u], gk[u * d.pw[m]], acc);
                    }
                    gH[hoff(d, m) + v] = -acc;
                }
                __syncthreads();
            }
        }
    }
}

inline size_t logsig_fwd_smem(const TensorDims& d, int w, bool brackets) {
    int64_t HS = 0;
    for (int j = 0; j < d.N; ++j) HS += d.pw[j];
    return (size_t)(2 * HS) * sizeof(double) + (size_t)(d.S + (brackets ? w : 0)) * sizeof(float);
}

inline size_t logsig_bwd_smem(const TensorDims& d) {
    int64_t HS = 0;
    for (int j = 0; j < d.N; ++j) HS += d.pw[j];
    int64_t hall = 0;
    for (int n = 1; n <= d.N; ++n)
        for (int j = 0; j <= d.N - n; ++j) hall += d.pw[j];
    return (size_t)(hall + HS) * sizeof(double) + (size_t)d.S * sizeof(float);
}

}  // namespace sigb200
