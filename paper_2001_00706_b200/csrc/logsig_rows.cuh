// logsig_rows.cuh -- K4 for many small rows (stream-mode logsignatures), sm_100a.
//
// Same computation as logsig_fwd_kernel (logsig.cuh): the truncated log in Horner form
// H_N = 1/N, H_n = 1/n - x H_{n+1} (levels 0..N-n), log = x H_1 (reading R7), float64
// inside, float32 in and out, then the words / brackets / expand projection (Appendix A.2).
// Layout: one WARP per signature row instead of one 1024-thread CTA per row.  A stream-mode
// logsignature has B*M rows of a small signature (c3's shape: 261,888 rows of S = 1554); a CTA per
// row spends its time launching, staging and synchronising 32 warps for ~2k multiply-adds.  Here a
// warp stages the row and its two H buffers in its own slice of shared memory, synchronises with
// __syncwarp only, and walks rows with a grid stride.  C is a template parameter so that the word splits are divisions by a
// compile-time constant; N and the level tables are runtime (a per-CTA copy in shared memory).
#pragma once
#include "logsig.cuh"

namespace sigb200 {

constexpr int LOGSIG_ROWS_THREADS = 256;

// the same kernel compiled per (C, N) (logsig_rows.cu); nullptr when (C, N) has no instance
using LogsigRowsLaunch = cudaError_t (*)(const LogsigParams&, cudaStream_t);
LogsigRowsLaunch find_logsig_rows_t(int C, int N);

// floats of shared memory per warp: the row (levels 1..N), two float64 H buffers (levels
// 0..N-1), psi (brackets)
inline size_t logsig_rows_warp_floats(const LDims& d, int w, bool brackets) {
    const size_t xs = ((size_t)d.S + 1) / 2 * 2;  // keeps the doubles 8-byte aligned
    return xs + 2 * 2 * (size_t)d.hoff[d.N] + (brackets ? ((size_t)w + 1) / 2 * 2 : 0);
}

#ifdef SIG_DEFINE_LOGSIG_KERNELS
template <int C>
__device__ __forceinline__ double xh_rows(const int* off, const int* hoff, const float* xs, const double* H, int k,
                                          int w) {
    // (x H)_k[w] = sum_{i=1}^{k} x_i[w[:i]] H_{k-i}[w[i:]], peeling one letter per term
    double acc = 0.0;
    int u = w, v = 0, q = 1;
    for (int i = k; i >= 1; --i) {
        acc = fma((double)xs[off[i] + u], H[hoff[k - i] + v], acc);
        const int u2 = u / C;
        v += (u - u2 * C) * q;
        q *= C;
        u = u2;
    }
    return acc;
}

template <int C>
__global__ void __launch_bounds__(LOGSIG_ROWS_THREADS) logsig_rows_kernel(const LogsigParams p, int wfloats) {
    extern __shared__ __align__(16) float lrs[];
    __shared__ int off[18], hoff[18];
    const int N = p.d.N, S = p.d.S;
    if (threadIdx.x < 18) {
        off[threadIdx.x] = p.d.off[threadIdx.x];
        hoff[threadIdx.x] = p.d.hoff[threadIdx.x];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int HS = hoff[N];                // H levels 0..N-1
    float* xs = lrs + (size_t)wib * wfloats;
    double* Ha = reinterpret_cast<double*>(xs + (S + 1) / 2 * 2);
    double* Hb = Ha + HS;
    float* psi = reinterpret_cast<float*>(Hb + HS);
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t row = gw; row < p.rows; row += nw) {
        const float* src = p.sig + row * S;
        // the whole row, many loads in flight per lane (one dependent global load per output word
        // cost the first version ~5x)
        {
            int f = lane;
            for (; f + 96 < S; f += 128) {
                const float a = __ldg(src + f), b = __ldg(src + f + 32), c = __ldg(src + f + 64), e = __ldg(src + f + 96);
                xs[f] = a;
                xs[f + 32] = b;
                xs[f + 64] = c;
                xs[f + 96] = e;
            }
            for (; f < S; f += 32) xs[f] = __ldg(src + f);
        }
        if (lane == 0) Ha[0] = 1.0 / (double)N;
        __syncwarp();
        double* Hc = Ha;
        double* Hn = Hb;
        for (int n = N - 1; n >= 1; --n) {
            const int top = N - n;  // H_n on levels 0..top
            for (int e = lane; e < hoff[top + 1]; e += 32) {
                if (e == 0) {
                    Hn[0] = 1.0 / (double)n;
                    continue;
                }
                int m = 1;
                while (e >= hoff[m + 1]) ++m;
                Hn[e] = -xh_rows<C>(off, hoff, xs, Hc, m, e - hoff[m]);
            }
            __syncwarp();
            double* t = Hc;
            Hc = Hn;
            Hn = t;
        }
        // log = x H_1
        auto coef = [&](int f) -> double {
            int k = 1;
            while (k < N && f >= off[k + 1]) ++k;
            return xh_rows<C>(off, hoff, xs, Hc, k, f - off[k]);
        };
        if (p.mode == 0) {
            float* o = p.out + row * S;
            for (int f = lane; f < S; f += 32) o[f] = (float)coef(f);
        } else {
            float* o = p.out + row * p.tb.w;
            for (int j = lane; j < p.tb.w; j += 32) {
                const double v = coef((int)__ldg(p.tb.lyn_idx + j));
                if (p.mode == 2) o[j] = (float)v;
                else psi[j] = (float)v;
            }
            if (p.mode == 1) {
                __syncwarp();
                // exact integer coefficients of (psi o phi)^{-1}
                for (int r = lane; r < p.tb.w; r += 32) {
                    double acc = 0.0;
                    for (int e = __ldg(p.tb.minv_rowptr + r); e < __ldg(p.tb.minv_rowptr + r + 1); ++e)
                        acc = fma((double)__ldg(p.tb.minv_val + e), (double)psi[__ldg(p.tb.minv_col + e)], acc);
                    o[r] = (float)acc;
                }
            }
        }
        __syncwarp();  // the next row overwrites xs, H and psi
    }
}

// launch over `rows` rows when the per-warp slice fits (returns cudaErrorInvalidConfiguration if not)
inline cudaError_t launch_logsig_rows(const LogsigParams& p, cudaStream_t st) {
    const bool br = p.mode == 1;
    const size_t wf = logsig_rows_warp_floats(p.d, p.tb.w, br);
    const size_t smem = wf * sizeof(float) * (LOGSIG_ROWS_THREADS / 32);
    if (smem > 200 * 1024 || p.d.C < 1 || p.d.C > 8) return cudaErrorInvalidConfiguration;
    const void* fn = nullptr;
    switch (p.d.C) {
        case 1: fn = (const void*)logsig_rows_kernel<1>; break;
        case 2: fn = (const void*)logsig_rows_kernel<2>; break;
        case 3: fn = (const void*)logsig_rows_kernel<3>; break;
        case 4: fn = (const void*)logsig_rows_kernel<4>; break;
        case 5: fn = (const void*)logsig_rows_kernel<5>; break;
        case 6: fn = (const void*)logsig_rows_kernel<6>; break;
        case 7: fn = (const void*)logsig_rows_kernel<7>; break;
        default: fn = (const void*)logsig_rows_kernel<8>; break;
    }
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, LOGSIG_ROWS_THREADS, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    int64_t grid = (int64_t)per_sm * 148;
    const int64_t need = (p.rows + LOGSIG_ROWS_THREADS / 32 - 1) / (LOGSIG_ROWS_THREADS / 32);  // a warp per row
    if (grid > need) grid = need;
    int wfl = (int)wf;
    void* args[] = {const_cast<LogsigParams*>(&p), &wfl};
    return cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(LOGSIG_ROWS_THREADS), args, smem, st);
}
#endif  // SIG_DEFINE_LOGSIG_KERNELS

}  // namespace sigb200
