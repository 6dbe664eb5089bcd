// sig_common.cuh -- compile-time shapes and small device helpers shared by the sm_100a kernels.
//
// Truncated tensor layout: levels k = 1..N are
// stored back to back; inside level k the word (j_1..j_k) (0-based letters) is at offset
// sum_m j_m C^(k-m).  The scalar level 0 is implicit.
//
// Work decomposition: a thread owns one word prefix p = (p_0..p_{P-1}) of length
// P.  It holds in registers every coefficient whose word starts with p, i.e. the contiguous block
// of C^(k-P) floats at level k for every k >= max(P,1), plus one replicated copy of the prefix
// coefficients A_i[p_0..p_{i-1}] for i < P.  The fused multiply-exponentiate (eq-fusedterm,
// P:L164-167) for level k needs A_i only along the thread's own prefix below level P, so a thread
// can advance its block with no communication at all.
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace sigb200 {

#ifndef SIG_ZSWZ
#define SIG_ZSWZ 0
#endif
// Increments are staged in shared memory with adjacent channels swapped (c <-> c^1 when C is
// even), so that a vector LDS.128 of a staged row puts z_c in a register whose parity differs from
// that of the state coefficients ending in letter c (which vector LDG/STG keep in natural order).
// The FFMA z_c * b + A[..c] then reads its two non-reused operands from different register banks
// (two same-parity register sources halve the FFMA issue rate; K1).
__host__ __device__ constexpr int zswz(int C, int c) { return (SIG_ZSWZ && C % 2 == 0) ? (c ^ 1) : c; }

__host__ __device__ __forceinline__ constexpr int64_t ipow(int64_t C, int k) {
    int64_t r = 1;
    for (int i = 0; i < k; ++i) r *= C;
    return r;
}

template <int C_, int N_, int P_>
struct Shape {
    static constexpr int C = C_;
    static constexpr int N = N_;
    static constexpr int P = P_;
    static constexpr int K0 = P_ > 1 ? P_ : 1;           // lowest owned level
    static constexpr int CP = (int)ipow(C_, P_);         // threads per unit (one per prefix)
    // number of owned coefficients at level k (k >= K0)
    __host__ __device__ static constexpr int own(int k) { return (int)ipow(C_, k - P_); }
    // register offset of level k inside the owned array
    __host__ __device__ static constexpr int own_off(int k) {
        int s = 0;
        for (int j = K0; j < k; ++j) s += own(j);
        return s;
    }
    static constexpr int OWN = own_off(N_ + 1);           // owned levels K0..N
    static constexpr int OWN_BELOW_TOP = own_off(N_);     // owned levels K0..N-1
    // flat offset of level k (1-based) in the S-wide layout
    __host__ __device__ static constexpr int64_t lvl_off(int k) {
        int64_t s = 0;
        for (int j = 1; j < k; ++j) s += ipow(C_, j);
        return s;
    }
    static constexpr int64_t S = lvl_off(N_ + 1);
    static constexpr int NLOW = P_ > 1 ? P_ - 1 : 0;     // replicated prefix levels 1..P-1
    // scratch for the Horner intermediates B_i, i = P+1..N-1 (C^(i-P) floats each)
    __host__ __device__ static constexpr int tmp_off(int i) {
        int s = 0;
        for (int j = P_ + 1; j < i; ++j) s += own(j);
        return s;
    }
    static constexpr int TMP = tmp_off(N_) > 0 ? tmp_off(N_) : 1;
    static constexpr int LOWA = NLOW + 1;                 // low[1..P-1] (index 0 unused)
    static constexpr int PD = P_ > 0 ? P_ : 1;            // digits array size
    static constexpr int PL1 = P_ + 1;                    // arrays indexed 0..P
    static constexpr int OWNA = OWN_BELOW_TOP > 0 ? OWN_BELOW_TOP : 1;
};

__host__ __device__ constexpr int ilog2(int v) {
    int r = 0;
    while ((1 << (r + 1)) <= v) ++r;
    return r;
}

// compile-time loop: f(std::integral_constant<int, I>) for I in [B, E)
template <int B, int E, class F>
__device__ __forceinline__ void static_for(F&& f) {
    if constexpr (B < E) {
        f(std::integral_constant<int, B>{});
        static_for<B + 1, E>(f);
    }
}

template <class SH>
__device__ __forceinline__ void prefix_digits(int prefix, int (&p)[SH::PD]) {
    int r = prefix;
#pragma unroll
    for (int j = SH::P - 1; j >= 0; --j) {
        p[j] = r % SH::C;
        r /= SH::C;
    }
}

// Store src[OFF .. OFF+n) (a register array: indices must stay compile-time constants so it is
// never demoted to local memory) to dst, vectorised by the runtime alignment of dst.
template <int n, int OFF, bool STREAMING, int SZ>
__device__ __forceinline__ void store_run(float* dst, const float (&src)[SZ]) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(dst);
    if constexpr (n % 4 == 0) {
        if ((a & 15) == 0) {
#pragma unroll
            for (int i = 0; i < n; i += 4) {
                float4 v = make_float4(src[OFF + i], src[OFF + i + 1], src[OFF + i + 2], src[OFF + i + 3]);
                if (STREAMING) __stcs(reinterpret_cast<float4*>(dst + i), v);
                else *reinterpret_cast<float4*>(dst + i) = v;
            }
            return;
        }
    }
    if constexpr (n % 2 == 0) {
        if ((a & 7) == 0) {
#pragma unroll
            for (int i = 0; i < n; i += 2) {
                float2 v = make_float2(src[OFF + i], src[OFF + i + 1]);
                if (STREAMING) __stcs(reinterpret_cast<float2*>(dst + i), v);
                else *reinterpret_cast<float2*>(dst + i) = v;
            }
            return;
        }
    }
#pragma unroll
    for (int i = 0; i < n; ++i) {
        if (STREAMING) __stcs(dst + i, src[OFF + i]);
        else dst[i] = src[OFF + i];
    }
}

// Load n floats from src into dst[OFF .. OFF+n) (register array), vectorised by alignment.
template <int n, int OFF, int SZ>
__device__ __forceinline__ void load_run(float (&dst)[SZ], const float* src) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(src);
    if constexpr (n % 4 == 0) {
        if ((a & 15) == 0) {
#pragma unroll
            for (int i = 0; i < n; i += 4) {
                float4 v = __ldg(reinterpret_cast<const float4*>(src + i));
                dst[OFF + i] = v.x; dst[OFF + i + 1] = v.y; dst[OFF + i + 2] = v.z; dst[OFF + i + 3] = v.w;
            }
            return;
        }
    }
    if constexpr (n % 2 == 0) {
        if ((a & 7) == 0) {
#pragma unroll
            for (int i = 0; i < n; i += 2) {
                float2 v = __ldg(reinterpret_cast<const float2*>(src + i));
                dst[OFF + i] = v.x; dst[OFF + i + 1] = v.y;
            }
            return;
        }
    }
#pragma unroll
    for (int i = 0; i < n; ++i) dst[OFF + i] = __ldg(src + i);
}

// Load n floats from SHARED memory src into dst[OFF .. OFF+n) (plain vector loads by alignment).
template <int n, int OFF, int SZ>
__device__ __forceinline__ void load_run_s(float (&dst)[SZ], const float* src) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(src);
    if constexpr (n % 4 == 0) {
        if ((a & 15) == 0) {
#pragma unroll
            for (int i = 0; i < n; i += 4) {
                const float4 v = *reinterpret_cast<const float4*>(src + i);
                dst[OFF + i] = v.x; dst[OFF + i + 1] = v.y; dst[OFF + i + 2] = v.z; dst[OFF + i + 3] = v.w;
            }
            return;
        }
    }
#pragma unroll
    for (int i = 0; i < n; ++i) dst[OFF + i] = src[i];
}

// dst[OFF .. OFF+n) += src[0 .. n), vectorised by the alignment of src (no staging array).
template <int n, int OFF, int SZ>
__device__ __forceinline__ void add_run(float (&dst)[SZ], const float* src) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(src);
    if constexpr (n % 4 == 0) {
        if ((a & 15) == 0) {
#pragma unroll
            for (int i = 0; i < n; i += 4) {
                float4 v = __ldg(reinterpret_cast<const float4*>(src + i));
                dst[OFF + i] += v.x; dst[OFF + i + 1] += v.y; dst[OFF + i + 2] += v.z; dst[OFF + i + 3] += v.w;
            }
            return;
        }
    }
#pragma unroll
    for (int i = 0; i < n; ++i) dst[OFF + i] += __ldg(src + i);
}

// Copy n floats global -> shared by the whole CTA with several loads in flight per thread (a plain
// load-then-store loop serialises one global latency per element: the fold/scan kernels spent most
// of their time there).  float4 when both sides are 16-byte aligned.
__device__ __forceinline__ void stage_to_smem(float* __restrict__ dst, const float* __restrict__ src, int n) {
    const int tid = threadIdx.x, nt = blockDim.x;
    if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
        const int n4 = n >> 2;
        const float4* s4 = reinterpret_cast<const float4*>(src);
        float4* d4 = reinterpret_cast<float4*>(dst);
        int e = tid;
        for (; e + 3 * nt < n4; e += 4 * nt) {
            const float4 a = __ldg(s4 + e), b = __ldg(s4 + e + nt), c = __ldg(s4 + e + 2 * nt), d = __ldg(s4 + e + 3 * nt);
            d4[e] = a;
            d4[e + nt] = b;
            d4[e + 2 * nt] = c;
            d4[e + 3 * nt] = d;
        }
        for (; e < n4; e += nt) d4[e] = __ldg(s4 + e);
        for (int f = (n4 << 2) + tid; f < n; f += nt) dst[f] = __ldg(src + f);
        return;
    }
    int e = tid;
    for (; e + 3 * nt < n; e += 4 * nt) {
        const float a = __ldg(src + e), b = __ldg(src + e + nt), c = __ldg(src + e + 2 * nt), d = __ldg(src + e + 3 * nt);
        dst[e] = a;
        dst[e + nt] = b;
        dst[e + 2 * nt] = c;
        dst[e + 3 * nt] = d;
    }
    for (; e < n; e += nt) dst[e] = __ldg(src + e);
}

// reciprocals 1/s, s = 1..16 (exact float roundings of the rationals)
__device__ __forceinline__ constexpr float inv_int(int s) {
    return s == 1 ? 1.0f : 1.0f / (float)s;
}

// shared-memory address of a generic pointer into shared memory (PTX operands of the async copies)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- TMA bulk copies global -> shared completed on an mbarrier (1-D cp.async.bulk; sizes and
// addresses multiples of 16 bytes)
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}"
        ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}
// order this thread's earlier generic-proxy accesses of shared memory before later async-proxy ones
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// bulk copy of any multiple of 16 bytes, in pieces of at most `piece` bytes (4 KB vs 64 KB pieces
// measured the same for c5's 68 KB per CTA)
__device__ __forceinline__ void bulk_g2s_big(void* sdst, const void* gsrc, size_t bytes, uint64_t* bar,
                                             unsigned piece = 65536) {
    char* d = static_cast<char*>(sdst);
    const char* g = static_cast<const char*>(gsrc);
    while (bytes > 0) {
        const unsigned n = bytes > piece ? piece : (unsigned)bytes;
        bulk_g2s(d, g, n, bar);
        d += n;
        g += n;
        bytes -= n;
    }
}

}  // namespace sigb200
