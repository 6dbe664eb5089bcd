// logsig_owned.cuh -- K5 (logsignature backward), owned-prefix form compiled per (C, N) for
// power-of-two C.
//
// Same algorithm as logsig_bwd_owned_kernel in logsig.cuh (see the comment there): the Horner
// VJP of log = x H_1, H_n = 1/n - x H_{n+1} (reading R7) as N passes of two
// contractions of a source tensor s on levels 1..TOP,
//   GX: gx_i[u] (+)= sgn * sum_{m} sum_v s_{i+m}[u v] H_m[v]      split by word prefix,
//   GH: gH_m[v]   = sgn * sum_{i} sum_u x_i[u] s_{i+m}[u v]      split by word suffix,
// but with C and N compile-time: every level loop unrolls, and every shared-memory address is a
// per-thread base plus an immediate.  For that, each level of each shared array carries its own
// padding (one float per 32, counted from the level start): a thread's block of B = C^j floats
// starts at a multiple of B, so with B a power of two its padded offsets are constants.
#pragma once
#include "logsig.cuh"
#include <type_traits>
#include "sig_common.cuh"

namespace sigb200 {

template <int C_, int N_>
struct LT {
    static constexpr int C = C_, N = N_;
    static_assert((C & (C - 1)) == 0, "power-of-two C only");
    static constexpr int LC = ilog2(C);
    __host__ __device__ static constexpr int pw(int k) { return (int)ipow(C, k); }
    // S layout (levels 1..N), 1-based level k starts at off(k)
    __host__ __device__ static constexpr int off(int k) {
        int s = 0;
        for (int j = 1; j < k; ++j) s += pw(j);
        return s;
    }
    __host__ __device__ static constexpr int lsz(int k) { return lpad(pw(k)) + 1; }  // padded level
    __host__ __device__ static constexpr int gls(int k) {  // padded dL/dlog: level k >= 1
        int s = 0;
        for (int j = 1; j < k; ++j) s += lsz(j);
        return s;
    }
    __host__ __device__ static constexpr int ghs(int m) {  // padded H / dL/dH arrays: level m >= 0
        int s = 0;
        for (int j = 0; j < m; ++j) s += lsz(j);
        return s;
    }
    __host__ __device__ static constexpr int hb(int n) {  // H_n (levels 0..N-n) in Hall; H_N first
        int s = 0;
        for (int q = N; q > n; --q) s += ghs(N - q + 1);
        return s;
    }
    __host__ __device__ static constexpr int choose_p() {
        int P = 1;
        while (P < N && ipow(C, P + 1) <= LOGSIG_THREADS) ++P;
        return P;
    }
    static constexpr int P = choose_p();
    static constexpr int S = off(N + 1);
    static constexpr int HALL = hb(0);
    static constexpr int GHN = ghs(N);
    static constexpr int GLN = gls(N + 1);
    static constexpr int XS = off(N);  // x on levels 1..N-1
    static constexpr int SCR = lpad((P > 1 ? P - 1 : 1) * pw(P)) + 1;
    static constexpr int O_GHA = HALL, O_GHB = O_GHA + GHN, O_XS = O_GHB + GHN, O_GL = O_XS + XS,
                         O_SCR = O_GL + GLN, TOTAL = O_SCR + SCR;
    // padded offset c inside a block of B floats that starts at a multiple of B
    __host__ __device__ static constexpr int boff(int B, int c) { return B <= 32 ? c : lpad(c); }
};

// sum aligned blocks of a partial row (see owned_block_reduce), compile-time shapes, plus the
// output's extra terms extra(l_c, o, g, G) (lane g of G)
template <class T, int LP, class Extra, class Emit>
__device__ __forceinline__ void owned_block_reduce_t(const float* scr, Extra&& extra, Emit&& emit) {
    constexpr int NP = T::pw(LP);
    static_for<1, LP>([&](auto lc) {
        constexpr int l = decltype(lc)::value;
        constexpr int NOUT = T::pw(l), BS = T::pw(LP - l);
        constexpr int G = BS < 32 ? BS : 32;
        constexpr int SH = ilog2(G);
        constexpr int ITEMS = ((NOUT << SH) + 31) & ~31;
        for (int idx = threadIdx.x; idx < ITEMS; idx += blockDim.x) {
            const int o = idx >> SH, g = idx & (G - 1);
            float sum = 0.0f;
            if (o < NOUT) {
                const int base = (l - 1) * NP + o * BS;
#pragma unroll 4
                for (int e = g; e < BS; e += G) sum += scr[lpad(base + e)];
                sum += extra(lc, o, g, std::integral_constant<int, G>{});
            }
#pragma unroll
            for (int q = G >> 1; q >= 1; q >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, q);
            if (g == 0 && o < NOUT) emit(l, o, sum);
        }
    });
}

// one pass on source levels 1..TOP; A: the source is dL/dlog (step A, gx initialised), else dL/dH_n
// with n = N - TOP.  The pass reads H_{N-TOP+1}.
template <class T, int TOP, bool A>
__device__ __forceinline__ void owned_pass_t(const float* __restrict__ src, const float* __restrict__ Hall,
                                             const float* __restrict__ xs, float* __restrict__ scr, float* gx,
                                             float* __restrict__ gHo) {
    constexpr float sgn = A ? 1.0f : -1.0f;
    constexpr int HB = T::hb(T::N - TOP + 1);
    const int tid = threadIdx.x;
    auto SL = [](int k) constexpr { return A ? T::gls(k) : T::ghs(k); };
    // ---------------- GX, by prefix
    constexpr int Pg = T::P < TOP ? T::P : TOP;
    constexpr int NP = T::pw(Pg);
    if (tid < NP) {
        const int pf = tid;
        static_for<Pg, TOP + 1>([&](auto ic) {  // owned outputs u = pf u'
            constexpr int i = decltype(ic)::value;
            constexpr int NU = T::pw(i - Pg);
#pragma unroll
            for (int up = 0; up < NU; ++up) {
                float acc = 0.0f;
                static_for<0, TOP - i + 1>([&](auto mc) {
                    constexpr int m = decltype(mc)::value;
                    constexpr int B = T::pw(i + m - Pg), NV = T::pw(m);
                    const float* s = src + SL(i + m) + lpad(pf * B);
                    const float* h = Hall + HB + T::ghs(m);
#pragma unroll
                    for (int v = 0; v < NV; ++v) acc = fmaf(s[T::boff(B, up * NV + v)], h[lpad(v)], acc);
                });
                float* dst = gx + T::off(i) + pf * NU + up;
                *dst = A ? acc : fmaf(sgn, acc, *dst);
            }
        });
        static_for<1, Pg>([&](auto ic) {  // partial of gx_i[p[:i]] over the owned words
            constexpr int i = decltype(ic)::value;
            const int ps = pf & (T::pw(Pg - i) - 1);  // p[i:]
            float acc = 0.0f;
            static_for<Pg, TOP + 1>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                constexpr int B = T::pw(k - Pg);
                const float* s = src + SL(k) + lpad(pf * B);
                const float* h = Hall + HB + T::ghs(k - i) + lpad(ps * B);
#pragma unroll
                for (int v = 0; v < B; ++v) acc = fmaf(s[T::boff(B, v)], h[T::boff(B, v)], acc);
            });
            scr[lpad((i - 1) * NP + pf)] = acc;
        });
    }
    __syncthreads();
    // extra terms of gx_i[u]: the short source words w = u w' (|w| = k, i <= k < P')
    auto gx_short = [&](auto ic, int u, int g, auto Gc) -> float {
        constexpr int i = decltype(ic)::value, G = decltype(Gc)::value;
        float t = 0.0f;
        static_for<i, Pg>([&](auto kc) {
            constexpr int k = decltype(kc)::value;
            constexpr int NW = T::pw(k - i);
            const float* s = src + SL(k);
            const float* h = Hall + HB + T::ghs(k - i);
            for (int w = g; w < NW; w += G) t = fmaf(s[lpad(u * NW + w)], h[lpad(w)], t);
        });
        return t;
    };
    owned_block_reduce_t<T, Pg>(scr, gx_short, [&](int i, int u, float sum) {
        float* dst = gx + T::off(i) + u;
        *dst = A ? sum : fmaf(sgn, sum, *dst);
    });
    // ---------------- GH, by suffix
    if constexpr (TOP >= 2) {
        __syncthreads();  // scratch reuse
        constexpr int Ph = T::P < TOP - 1 ? T::P : TOP - 1;
        constexpr int NS = T::pw(Ph);
        if (tid < NS) {
            const int sf = tid;
            const int lsf = lpad(sf);
            // padded offset, inside a level, of element c * NS + sf
            auto pidx = [&](int c) -> int {
                if constexpr (NS >= 32) return lpad(c * NS) + lsf;
                else return lpad(c * NS + sf);
            };
            static_for<Ph, TOP>([&](auto mc) {  // owned outputs v = v'' s, m >= Ph
                constexpr int m = decltype(mc)::value;
                constexpr int NVV = T::pw(m - Ph), R = T::pw(m - Ph);
#pragma unroll
                for (int vv = 0; vv < NVV; ++vv) {
                    float acc = 0.0f;
                    static_for<1, TOP - m + 1>([&](auto icc) {
                        constexpr int i = decltype(icc)::value;
                        const float* s = src + SL(i + m);
#pragma unroll
                        for (int u = 0; u < T::pw(i); ++u) acc = fmaf(xs[T::off(i) + u], s[pidx(u * R + vv)], acc);
                    });
                    gHo[T::ghs(m) + pidx(vv)] = sgn * acc;
                }
            });
            static_for<1, Ph>([&](auto mc) {  // partial of gH_m[s[Ph-m:]] over the owned words
                constexpr int m = decltype(mc)::value;
                constexpr int CM = T::pw(m), CQ = T::pw(Ph - m);
                const int sq = sf >> (T::LC * m);
                float acc = 0.0f;
                static_for<Ph, TOP + 1>([&](auto kc) {  // words y s, split u = (y s)[:k-m]
                    constexpr int k = decltype(kc)::value;
                    const float* s = src + SL(k);
                    const float* x = xs + T::off(k - m) + sq;
#pragma unroll
                    for (int y = 0; y < T::pw(k - Ph); ++y) acc = fmaf(x[y * CQ], s[pidx(y)], acc);
                });
                scr[lpad((m - 1) * NS + (sf & (CM - 1)) * CQ + sq)] = acc;  // grouped by output
            });
        }
        __syncthreads();
        // extra terms of gH_m[v]: the short source words w = u v (|w| = k, m < k < P'')
        auto gh_short = [&](auto mc, int v, int g, auto Gc) -> float {
            constexpr int m = decltype(mc)::value, G = decltype(Gc)::value;
            float t = 0.0f;
            static_for<m + 1, Ph>([&](auto kc) {
                constexpr int k = decltype(kc)::value;
                constexpr int NU = T::pw(k - m);
                const float* s = src + SL(k);
                const float* x = xs + T::off(k - m);
                for (int u = g; u < NU; u += G) t = fmaf(x[u], s[lpad(u * T::pw(m) + v)], t);
            });
            return t;
        };
        owned_block_reduce_t<T, Ph>(scr, gh_short, [&](int m, int v, float sum) {
            gHo[T::ghs(m) + lpad(v)] = sgn * sum;
        });
    }
}

template <int C, int N>
__global__ void __launch_bounds__(LOGSIG_THREADS, 1) logsig_bwd_owned_t_kernel(const LogsigParams p) {
    using T = LT<C, N>;
    const int64_t row = blockIdx.x;
    extern __shared__ __align__(16) float lsf[];
    float* Hall = lsf;
    float* gHa = lsf + T::O_GHA;
    float* gHb = lsf + T::O_GHB;
    float* xs = lsf + T::O_XS;
    float* gl = lsf + T::O_GL;
    float* scr = lsf + T::O_SCR;
    const int tid = threadIdx.x, nth = blockDim.x;
    const float* sg = p.sig + row * T::S;
    for (int f = tid; f < T::XS; f += nth) xs[f] = sg[f];
    if (tid == 0) Hall[T::hb(N)] = 1.0f / (float)N;
    if (p.mode == 0) {
        const float* go = p.gout + row * T::S;
        static_for<1, N + 1>([&](auto kc) {
            constexpr int k = decltype(kc)::value;
            for (int e = tid; e < T::pw(k); e += nth) gl[T::gls(k) + lpad(e)] = go[T::off(k) + e];
        });
    } else {
        for (int f = tid; f < T::GLN; f += nth) gl[f] = 0.0f;
        __syncthreads();
        const float* go = p.gout + row * p.tb.w;
        for (int j = tid; j < p.tb.w; j += nth) {
            double v;
            if (p.mode == 2) {
                v = go[j];
            } else {
                v = 0.0;
                for (int e = p.tb.minvT_rowptr[j]; e < p.tb.minvT_rowptr[j + 1]; ++e)
                    v = fma((double)p.tb.minvT_val[e], (double)go[p.tb.minvT_col[e]], v);
            }
            // level of f and its padded slot from compile-time tables (a runtime T::off / T::gls
            // would loop over powers of C for every word: a quarter of the kernel's instructions)
            const int f = (int)p.tb.lyn_idx[j];
            int base = T::gls(1), offk = 0;
            static_for<2, N + 1>([&](auto kc) {
                constexpr int kk = decltype(kc)::value;
                if (f >= T::off(kk)) {
                    base = T::gls(kk);
                    offk = T::off(kk);
                }
            });
            gl[base + lpad(f - offk)] = (float)v;
        }
    }
    __syncthreads();
    // H_{N-1} .. H_1: H_n[w] = 1/n (level 0), else -sum_{i=1}^{m} x_i[w[:i]] H_{n+1}[w[i:]]
    static_for<1, N>([&](auto nc) {
        constexpr int n = N - decltype(nc)::value;  // N-1 .. 1
        constexpr int TOP = N - n;
        static_for<0, TOP + 1>([&](auto mc) {
            constexpr int m = decltype(mc)::value;
            for (int w = tid; w < T::pw(m); w += nth) {
                float val = 1.0f / (float)n;
                if constexpr (m > 0) {
                    float acc = 0.0f;
                    static_for<1, m + 1>([&](auto ic) {
                        constexpr int i = decltype(ic)::value;
                        const int u = w >> (T::LC * (m - i)), v = w & (T::pw(m - i) - 1);
                        acc = fmaf(xs[T::off(i) + u], Hall[T::hb(n + 1) + T::ghs(m - i) + lpad(v)], acc);
                    });
                    val = -acc;
                }
                Hall[T::hb(n) + T::ghs(m) + lpad(w)] = val;
            }
        });
        __syncthreads();
    });
    float* gx = p.gsig + row * T::S;
    owned_pass_t<T, N, true>(gl, Hall, xs, scr, gx, gHa);
    __syncthreads();
    static_for<1, N>([&](auto nc) {  // H_n = 1/n - x H_{n+1}; the source is dL/dH_n on levels 1..N-n
        constexpr int n = decltype(nc)::value;
        float* gc = (n & 1) ? gHa : gHb;
        float* gn = (n & 1) ? gHb : gHa;
        owned_pass_t<T, N - n, false>(gc, Hall, xs, scr, gx, gn);
        __syncthreads();
    });
}

template <int C, int N>
cudaError_t launch_logsig_bwd_owned_t(const LogsigParams& p, cudaStream_t st) {
    constexpr size_t smem = (size_t)LT<C, N>::TOTAL * sizeof(float);
    if (smem > 48 * 1024) {
        cudaError_t e =
            cudaFuncSetAttribute(logsig_bwd_owned_t_kernel<C, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    logsig_bwd_owned_t_kernel<C, N><<<(unsigned)p.rows, LOGSIG_THREADS, smem, st>>>(p);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// K4 (logsignature forward) compiled per (C, N), power-of-two C: the same Horner recursion as
// logsig_fwd_kernel (H_N = 1/N, H_n = 1/n - x H_{n+1} on levels 0..N-n, log = x H_1; reading R7),
// float64 accumulation of float32 inputs, but every level loop unrolled and every index a shift or
// mask: (x H)_m[w] = sum_{i=1}^{m} x_i[w >> (m-i) log2 C] * H_{m-i}[w & (C^(m-i) - 1)].
// H_n lives in one of two float64 buffers (levels 0..N-1); x on levels 1..N-1 in shared memory
// (the top level is read once from global by the output stage).
// ---------------------------------------------------------------------------------------------
template <class T>
__host__ __device__ constexpr int hofs(int m) {  // offset of level m in an H buffer
    int s = 0;
    for (int j = 0; j < m; ++j) s += T::pw(j);
    return s;
}

template <class T, int K>
__device__ __forceinline__ double log_coef_t(const float* xs, const float* srcN, const double* H1, int w) {
    double acc = 0.0;
    static_for<1, K + 1>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        float xv;
        if constexpr (i == T::N) xv = __ldg(srcN + w);
        else xv = xs[T::off(i) + (w >> (T::LC * (K - i)))];
        acc = fma((double)xv, H1[hofs<T>(K - i) + (w & (T::pw(K - i) - 1))], acc);
    });
    return acc;
}

template <int C, int N>
struct LogFwdT {
    using T = LT<C, N>;
    static constexpr int HS = hofs<T>(N);              // levels 0..N-1
    static constexpr int XSP = (T::XS + 3) / 4 * 4;      // x on levels 1..N-1, padded
    static size_t smem(int w, bool brackets) {
        return 2 * (size_t)HS * sizeof(double) + (size_t)XSP * sizeof(float) + (brackets ? (size_t)w * sizeof(float) : 0);
    }
};

#ifndef SIG_LOGFWD_THREADS
#define SIG_LOGFWD_THREADS 512
#endif
template <int C, int N>
__global__ void __launch_bounds__(SIG_LOGFWD_THREADS, 1024 / SIG_LOGFWD_THREADS) logsig_fwd_t_kernel(const LogsigParams p) {
    using T = LT<C, N>;
    using F = LogFwdT<C, N>;
    const int64_t row = blockIdx.x;
    extern __shared__ __align__(16) double lsd[];
    double* Hbuf[2] = {lsd, lsd + F::HS};
    float* xs = reinterpret_cast<float*>(lsd + 2 * F::HS);
    float* psi = xs + F::XSP;
    const int tid = threadIdx.x, nth = blockDim.x;
    const float* src = p.sig + row * T::S;
    for (int f = tid; f < T::XS; f += nth) xs[f] = src[f];
    if (tid == 0) Hbuf[0][0] = 1.0 / (double)N;  // H_N (level 0 only)
    __syncthreads();
    // H_n, n = N-1 .. 1, into buffer (N - n) & 1
    static_for<1, N>([&](auto nc) {
        constexpr int n = N - decltype(nc)::value;
        const double* Hc = Hbuf[(N - n - 1) & 1];
        double* Hn = Hbuf[(N - n) & 1];
        static_for<0, N - n + 1>([&](auto mc) {
            constexpr int m = decltype(mc)::value;
            for (int w = tid; w < T::pw(m); w += nth) {
                double val = 1.0 / (double)n;
                if constexpr (m > 0) {
                    double acc = 0.0;
                    static_for<1, m + 1>([&](auto ic) {
                        constexpr int i = decltype(ic)::value;
                        acc = fma((double)xs[T::off(i) + (w >> (T::LC * (m - i)))],
                                  Hc[hofs<T>(m - i) + (w & (T::pw(m - i) - 1))], acc);
                    });
                    val = -acc;
                }
                Hn[hofs<T>(m) + w] = val;
            }
        });
        __syncthreads();
    });
    const double* H1 = Hbuf[(N - 1) & 1];
    const float* srcN = src + T::off(N);
    if (p.mode == 0) {
        float* o = p.out + row * T::S;
        static_for<1, N + 1>([&](auto kc) {
            constexpr int k = decltype(kc)::value;
            for (int w = tid; w < T::pw(k); w += nth) o[T::off(k) + w] = (float)log_coef_t<T, k>(xs, srcN, H1, w);
        });
        return;
    }
    float* o = p.out + row * p.tb.w;
    for (int j = tid; j < p.tb.w; j += nth) {
        const int f = (int)p.tb.lyn_idx[j];
        double v = 0.0;
        static_for<1, N + 1>([&](auto kc) {
            constexpr int k = decltype(kc)::value;
            if (f >= T::off(k) && f < T::off(k + 1)) v = log_coef_t<T, k>(xs, srcN, H1, f - T::off(k));
        });
        if (p.mode == 2) o[j] = (float)v;
        else psi[j] = (float)v;
    }
    if (p.mode == 1) {
        __syncthreads();
        // exact integer coefficients of (psi o phi)^{-1}
        for (int r = tid; r < p.tb.w; r += nth) {
            double acc = 0.0;
            for (int e = p.tb.minv_rowptr[r]; e < p.tb.minv_rowptr[r + 1]; ++e)
                acc = fma((double)p.tb.minv_val[e], (double)psi[p.tb.minv_col[e]], acc);
            o[r] = (float)acc;
        }
    }
}

template <int C, int N>
cudaError_t launch_logsig_fwd_t(const LogsigParams& p, cudaStream_t st) {
    const size_t smem = LogFwdT<C, N>::smem(p.tb.w, p.mode == 1);
    if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    if (smem > 48 * 1024) {
        cudaError_t e =
            cudaFuncSetAttribute(logsig_fwd_t_kernel<C, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    logsig_fwd_t_kernel<C, N><<<(unsigned)p.rows, SIG_LOGFWD_THREADS, smem, st>>>(p);
    return cudaGetLastError();
}

using LogsigFwdLaunch = cudaError_t (*)(const LogsigParams&, cudaStream_t);
// nullptr when (C, N) has no compiled instance
LogsigFwdLaunch find_logsig_fwd_t(int C, int N);
// dynamic shared memory of the compiled K4 for one row (0 when there is no compiled instance)
size_t logsig_fwd_t_smem(int C, int N, int w, bool brackets);

using LogsigBwdLaunch = cudaError_t (*)(const LogsigParams&, cudaStream_t);
// nullptr when (C, N) has no compiled instance (non power-of-two C, or too large for one CTA)
LogsigBwdLaunch find_logsig_bwd_owned(int C, int N);

}  // namespace sigb200
