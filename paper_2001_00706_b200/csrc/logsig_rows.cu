// logsig_rows.cu -- K4 for many small rows compiled per (C, N): one warp per signature row, every
// level loop unrolled at compile time, every word split a division by a compile-time power of C.
//
// Same computation as logsig_rows_kernel (logsig_rows.cuh) and logsig_fwd_kernel (logsig.cuh): the
// truncated log in Horner form H_N = 1/N, H_n = 1/n - x H_{n+1} on levels 0..N-n, log = x H_1
// (reading R7), float64 inside, then words / brackets / expand (Appendix A.2).
//   (x H)_m[w] = sum_{i=1}^{m} x_i[w / C^(m-i)] H_{m-i}[w mod C^(m-i)]
// The runtime-shape warp-per-row kernel spent ~4k warp instructions per c3 row on level searches
// and digit peeling; here the per-term cost is two shared loads, an integer multiply-high and a
// DFMA.  Instantiated for the shapes whose warp slice fits 48 KB of shared memory.
#include <utility>
#include "logsig_owned.cuh"
#include "logsig_rows.cuh"

namespace sigb200 {

namespace {

template <int C, int N>
struct RT {
    __host__ __device__ static constexpr int pw(int k) { return (int)ipow(C, k); }
    __host__ __device__ static constexpr int off(int k) {  // level k >= 1 in the S layout
        int s = 0;
        for (int j = 1; j < k; ++j) s += pw(j);
        return s;
    }
    __host__ __device__ static constexpr int hoff(int m) {  // level m >= 0 in an H array
        int s = 0;
        for (int j = 0; j < m; ++j) s += pw(j);
        return s;
    }
    static constexpr int S = off(N + 1);
    static constexpr int XS = (S + 1) / 2 * 2;     // floats of one row buffer (8-byte aligned after)
    // H_n (levels 0..N-n) alternates between two buffers: A holds H_N, H_{N-2}, ..., B holds
    // H_{N-1}, H_{N-3}, ... -- each sized for its largest member (the one with the smallest n)
    __host__ __device__ static constexpr int hsize(int parity) {
        int s = 0;
        for (int n = 1; n <= N; ++n)
            if (((N - n) & 1) == parity && hoff(N - n + 1) > s) s = hoff(N - n + 1);
        return s;
    }
    static constexpr int HA = hsize(0), HB = hsize(1);
};

__device__ __forceinline__ void cp_async4(float* sdst, const float* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(K) : "memory"); }

// (x H)_m[w] with H on levels 0..m-1 of buffer Hb; the i = m term is x_m[w] * H_0
template <int C, int N, int M>
__device__ __forceinline__ double xh_t(const float* xs, const double* Hb, int w) {
    using T = RT<C, N>;
    double acc = 0.0;
    static_for<1, M + 1>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        constexpr int D = T::pw(M - i);
        const int u = w / D, v = w - u * D;
        acc = fma((double)xs[T::off(i) + u], Hb[T::hoff(M - i) + v], acc);
    });
    return acc;
}

constexpr int RT_THREADS = 128;  // 4 warps: small CTAs pack the shared memory of the SM densely
// double-buffered rows (the next row streams in while this one is computed) or one buffer and
// more warps per SM
#ifndef SIG_ROWS_DB
#define SIG_ROWS_DB 0
#endif
constexpr int RT_NBUF = SIG_ROWS_DB ? 2 : 1;

template <int C, int N>
__host__ __device__ constexpr int rt_wslice(int mode, int W) {
    return RT_NBUF * RT<C, N>::XS + 2 * (RT<C, N>::HA + RT<C, N>::HB) + (mode == 1 ? (W + 1) / 2 * 2 : 0);
}

// ops over a warp's outputs w = lane, lane + 32, ...: two per iteration, so that two independent
// dependent chains (loads, DFMAs) are in flight per lane
template <class F>
__device__ __forceinline__ void lanes2(int lo, int hi, int lane, F&& f) {
    int j = lo + lane;
    for (; j + 32 < hi; j += 64) {
        f(j);
        f(j + 32);
    }
    if (j < hi) f(j);
}

template <int C, int N>
__global__ void __launch_bounds__(RT_THREADS) logsig_rows_t_kernel(const LogsigParams p) {
    using T = RT<C, N>;
    extern __shared__ __align__(16) float lrt[];
    __shared__ int js[N + 2];  // Lyndon words of level k: j in [js[k], js[k+1])
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int W = p.tb.w;
    const int wslice = rt_wslice<C, N>(p.mode, W);
    int* lyn = reinterpret_cast<int*>(lrt + (size_t)(RT_THREADS / 32) * wslice);  // [W] word -> flat index
    if (p.mode != 0) {
        if (threadIdx.x <= N + 1) js[threadIdx.x] = 0;
        __syncthreads();
        // Lyndon words are ordered by length (R5): count those below each level's start
        for (int j = threadIdx.x; j < W; j += blockDim.x) {
            const int f = (int)p.tb.lyn_idx[j];
            lyn[j] = f;
            static_for<2, N + 1>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                if (f < T::off(k)) atomicAdd(&js[k], 1);
            });
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            js[1] = 0;
            js[N + 1] = W;
        }
        __syncthreads();
    }
    float* xbuf = lrt + (size_t)wib * wslice;
    double* Ha = reinterpret_cast<double*>(xbuf + RT_NBUF * T::XS);
    double* Hb = Ha + T::HA;
    float* psi = reinterpret_cast<float*>(Hb + T::HB);
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    // every copy of a row is issued before any is waited for (cp.async): one memory latency per row
    // (a load-then-store loop waited ~12 times per c3 row)
    auto prefetch = [&](int64_t r, float* dst) {
        const float* src = p.sig + r * T::S;
        for (int f = lane; f < T::S; f += 32) cp_async4(dst + f, src + f);
        cp_async_commit();
    };
    int cur = 0;
    if (RT_NBUF == 2 && gw < p.rows) prefetch(gw, xbuf);
    for (int64_t row = gw; row < p.rows; row += nw) {
        if constexpr (RT_NBUF == 2) {
            const bool more = row + nw < p.rows;
            if (more) prefetch(row + nw, xbuf + (size_t)(cur ^ 1) * T::XS);
            if (more) cp_async_wait<1>();
            else cp_async_wait<0>();
        } else {
            prefetch(row, xbuf);
            cp_async_wait<0>();
        }
        __syncwarp();
        const float* xs = xbuf + (size_t)cur * T::XS;
        if (lane == 0) Ha[0] = 1.0 / (double)N;  // H_N
        __syncwarp();
        // H_n, n = N-1 .. 1: into Hb when N - n is odd, else Ha
        static_for<1, N>([&](auto nc) {
            constexpr int n = N - decltype(nc)::value;
            const double* Hc = ((N - n - 1) & 1) ? Hb : Ha;
            double* Hn = ((N - n) & 1) ? Hb : Ha;
            if (lane == 0) Hn[0] = 1.0 / (double)n;
            static_for<1, N - n + 1>([&](auto mc) {
                constexpr int m = decltype(mc)::value;
                lanes2(0, T::pw(m), lane, [&](int w) { Hn[T::hoff(m) + w] = -xh_t<C, N, m>(xs, Hc, w); });
            });
            __syncwarp();
        });
        const double* H1 = ((N - 1) & 1) ? Hb : Ha;
        if (p.mode == 0) {
            float* o = p.out + row * T::S;
            static_for<1, N + 1>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                lanes2(0, T::pw(k), lane, [&](int w) { o[T::off(k) + w] = (float)xh_t<C, N, k>(xs, H1, w); });
            });
        } else {
            float* o = p.out + row * W;
            static_for<1, N + 1>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                lanes2(js[k], js[k + 1], lane, [&](int j) {
                    const double v = xh_t<C, N, k>(xs, H1, lyn[j] - T::off(k));
                    if (p.mode == 2) o[j] = (float)v;
                    else psi[j] = (float)v;
                });
            });
            if (p.mode == 1) {
                __syncwarp();
                for (int r = lane; r < W; r += 32) {  // exact integer coefficients of (psi o phi)^{-1}
                    double acc = 0.0;
                    for (int e = __ldg(p.tb.minv_rowptr + r); e < __ldg(p.tb.minv_rowptr + r + 1); ++e)
                        acc = fma((double)__ldg(p.tb.minv_val + e), (double)psi[__ldg(p.tb.minv_col + e)], acc);
                    o[r] = (float)acc;
                }
            }
        }
        __syncwarp();  // the next row's copies overwrite a row buffer; H and psi are rewritten
        if (RT_NBUF == 2) cur ^= 1;
    }
}

template <int C, int N>
cudaError_t launch_rows_t(const LogsigParams& p, cudaStream_t st) {
    const size_t smem = ((size_t)rt_wslice<C, N>(p.mode, p.tb.w) * (RT_THREADS / 32) + (p.mode != 0 ? (size_t)p.tb.w : 0)) *
                        sizeof(float);
    if (smem > 200 * 1024) return cudaErrorInvalidConfiguration;
    auto fn = logsig_rows_t_kernel<C, N>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, RT_THREADS, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    int64_t grid = (int64_t)per_sm * 148;
    const int64_t need = (p.rows + RT_THREADS / 32 - 1) / (RT_THREADS / 32);  // a warp per row
    if (grid > need) grid = need;
    fn<<<(unsigned)grid, RT_THREADS, smem, st>>>(p);
    return cudaGetLastError();
}

template <int C, int N>
constexpr LogsigRowsLaunch rentry() {
    if constexpr ((size_t)rt_wslice<C, N>(0, 0) * sizeof(float) <= 48 * 1024) return &launch_rows_t<C, N>;
    else return nullptr;
}

template <int C, int... Ns>
LogsigRowsLaunch rpick(int N, std::integer_sequence<int, Ns...>) {
    LogsigRowsLaunch r = nullptr;
    ((N == Ns + 2 ? (r = rentry<C, Ns + 2>(), 0) : 0), ...);
    return r;
}

}  // namespace

// compiled warp-per-row K4 for (C, N), 2 <= N, warp slice <= 48 KB; nullptr otherwise
LogsigRowsLaunch find_logsig_rows_t(int C, int N) {
    switch (C) {
        case 2: return rpick<2>(N, std::make_integer_sequence<int, 11>{});  // N = 2..12
        case 3: return rpick<3>(N, std::make_integer_sequence<int, 7>{});   // N = 2..8
        case 4: return rpick<4>(N, std::make_integer_sequence<int, 5>{});
        case 5: return rpick<5>(N, std::make_integer_sequence<int, 4>{});
        case 6: return rpick<6>(N, std::make_integer_sequence<int, 4>{});
        case 7: return rpick<7>(N, std::make_integer_sequence<int, 3>{});
        case 8: return rpick<8>(N, std::make_integer_sequence<int, 3>{});
        default: return nullptr;
    }
}

}  // namespace sigb200
