// tmem_probe.cu -- dev prototype: K2's constant-G_N contraction (a) on tcgen05 tensor cores with the
// result read back from TMEM, timed against the FFMA2 top loop of sig_bwd2p_kernel (c2: C=8, N=5, P=3).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/bin/tmem_probe scripts/tmem_probe.cu
//
// Contraction (a): G_N is constant over the reversal, so
//   G_{N-1,t}[W] = Gbar_{N-1}[W] + sum_c G_N[W c] X_t[c],   X_t = x_end - x_{t+1}  (cumulative increments)
// i.e. per path and tile of T steps one GEMM D[4096 x T] = G_N[4096 x 8] . X[8 x T] (M = 4096 (prefix,
// channel) rows, K = C = 8, N = T).  Here it is issued as 32 M-blocks of tcgen05.mma.cta_group::1.kind::tf32
// 128 x 8 x 8 (T = 8 steps per tile, two TMEM buffers of 32 x 8 columns), 3xTF32 (hi.hi + hi.lo + lo.hi),
// A = G_N from shared memory (K-major, no swizzle), accumulators in TMEM.  Each thread then reads its
// 16 values of G_{N-1,t} per step with tcgen05.ld (lane = its row inside the M-block, one column per
// M-block) instead of computing them with 64 FFMA2.
//
// Variants (256 threads = 8 warps, one CTA per SM, two warps per SM sub-partition, as sig_bwd2p_kernel):
//   FFMA : per step 64 FFMA2 (gz += B G_N) + 64 FFMA2 (beta += G_N z)        -- the current top loop
//   TMEM : per step 64 FFMA2 (gz) + 16 tcgen05.ld.32x32b.x1 (G_{N-1,t}); per 8 steps one thread issues
//          96 MMAs (32 blocks x 3 products) into the other TMEM buffer (mbarrier-tracked)
//   TMEM2: as TMEM with 8 tcgen05.ld.32x32b.x2 per two steps' worth of columns (loads every other step)
//   LDONLY: TMEM's per-step loads and FFMA2 without the MMAs and the per-tile sync (the load cost alone)
//   GZONLY: the 64 FFMA2 of gz alone (the floor any offload of G_{N-1} could reach)
// Capacity note: G_N as tf32 hi + lo is 2 x 128 KB per path; the timing kernels point hi and lo at the
// same 128 KB copy (same instruction stream and bandwidth).  The accuracy mode uses 16 M-blocks (2048
// rows) with distinct hi and lo copies and compares D against float64.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cstring>
#include <cuda_runtime.h>

constexpr int STEPS = 1024;  // steps per CTA in the timing runs (multiple of 8)
constexpr int NBLK = 32;     // M-blocks of 128 rows = 4096 rows

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, no swizzle: core matrix = 8 rows x 16 B; element (m, k) of a [rows x 8] tf32 block at
// (m/8)*256 + (k/4)*128 + (m%8)*16 + (k%4)*4 bytes  -> LBO (K-adjacent core matrices) = 128 B,
// SBO (8-row groups) = 256 B.
__host__ __device__ inline uint32_t kmaj_off(int m, int k) { return (m / 8) * 256 + (k / 4) * 128 + (m % 8) * 16 + (k % 4) * 4; }

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((128 >> 4) & 0x3FFF) << 16;  // LBO
    d |= (uint64_t)((256 >> 4) & 0x3FFF) << 32;  // SBO
    d |= (uint64_t)1 << 46;                      // version (sm_100)
    // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
    return d;
}
// kind::tf32, D f32, A/B tf32 K-major, M = 128, N = 8
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((8u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(IDESC), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
        "r"(phase));
}
__device__ __forceinline__ uint32_t ldtm1(uint32_t taddr) {
    uint32_t r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr));
    return r;
}
__device__ __forceinline__ void ldtm2(uint32_t taddr, uint32_t& a, uint32_t& b) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(a), "=r"(b) : "r"(taddr));
}
__device__ __forceinline__ void ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// shared memory: [A hi: nblk*128 rows x 8 tf32] [A lo] [B hi: 8 x 8] [B lo] [2 mbarriers] [tmem addr]
struct Smem {
    __host__ __device__ static constexpr size_t a_bytes(int nblk) { return (size_t)nblk * 128 * 8 * 4; }
};

// Issue the 3xTF32 products of one tile into TMEM columns col0 + blk*8 (blocks 0..nblk-1).
__device__ __forceinline__ void issue_tile(uint32_t tmem, int col0, int nblk, uint32_t a_hi, uint32_t a_lo, uint32_t b_hi,
                                           uint32_t b_lo) {
    for (int blk = 0; blk < nblk; ++blk) {
        const uint32_t d = tmem + col0 + blk * 8;
        const uint32_t ab = blk * 128 * 8 * 4;
        mma_tf32(d, sdesc(a_hi + ab), sdesc(b_hi), 0);
        mma_tf32(d, sdesc(a_hi + ab), sdesc(b_lo), 1);
        mma_tf32(d, sdesc(a_lo + ab), sdesc(b_hi), 1);
    }
}

// V: 0 FFMA, 1 TMEM (x1 loads), 2 TMEM2 (x2 loads), 3 accuracy (writes D of tile 0 to out)
template <int V>
__global__ void __launch_bounds__(256, 1) probe(float* out, const float* in, const float* ahl, const float* bhl, int steps,
                                                int nblk, int lo_same) {
    extern __shared__ __align__(1024) unsigned char sm[];
    const size_t ab = Smem::a_bytes(nblk);
    float* a_hi = reinterpret_cast<float*>(sm);
    float* a_lo = lo_same ? a_hi : reinterpret_cast<float*>(sm + ab);
    float* b_hi = reinterpret_cast<float*>(sm + (lo_same ? ab : 2 * ab));
    float* b_lo = b_hi + 64;
    uint64_t* bar = reinterpret_cast<uint64_t*>(b_lo + 64);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
    const int tid = threadIdx.x, warp = tid >> 5;

    float g[128];  // G_N of the two prefixes, prefix-pair layout (as sig_bwd2p_kernel)
#pragma unroll
    for (int i = 0; i < 128; ++i) g[i] = in[i] + tid * 1e-3f;
    float beta[16], gz[16], B[16], z[8];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        beta[i] = 0.f;
        gz[i] = 0.f;
        B[i] = in[128 + i];
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) z[i] = in[144 + i];

    if constexpr (V == 0 || V == 5) {
        for (int s = 0; s < steps; ++s) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    float2 r = __ffma2_rn(make_float2(B[2 * k], B[2 * k + 1]), make_float2(g[(k * 8 + q) * 2], g[(k * 8 + q) * 2 + 1]),
                                          make_float2(gz[2 * q], gz[2 * q + 1]));
                    gz[2 * q] = r.x;
                    gz[2 * q + 1] = r.y;
                }
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    if constexpr (V == 5) break;
                    float2 r = __ffma2_rn(make_float2(g[(c * 8 + k) * 2], g[(c * 8 + k) * 2 + 1]), make_float2(z[k], z[k]),
                                          make_float2(beta[2 * c], beta[2 * c + 1]));
                    beta[2 * c] = r.x;
                    beta[2 * c + 1] = r.y;
                }
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                B[i] = B[i] * 0.999f + 1e-7f * gz[i];
                B[i + 8] = B[i + 8] * 0.999f + 1e-7f * beta[i];
                z[i] = z[i] * 0.999f + 1e-6f;
            }
        }
    } else {
        // stage G_N (hi, lo) and X (hi, lo) into the K-major no-swizzle layout
        const int rows = nblk * 128;
        for (int e = tid; e < rows * 8; e += blockDim.x) {
            const int m = e / 8, k = e % 8;
            *reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(a_hi) + kmaj_off(m, k)) = ahl[e];
            if (!lo_same) *reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(a_lo) + kmaj_off(m, k)) = ahl[rows * 8 + e];
        }
        for (int e = tid; e < 64; e += blockDim.x) {
            const int n = e / 8, k = e % 8;  // B is N x K (K-major): n = step, k = channel
            *reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(b_hi) + kmaj_off(n, k)) = bhl[e];
            *reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(b_lo) + kmaj_off(n, k)) = bhl[64 + e];
        }
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "r"(512));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
        if (tid == 0) {
            mbar_init(&bar[0], 1);
            mbar_init(&bar[1], 1);
            asm volatile("fence.mbarrier_init.release.cluster;");
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy smem writes -> tensor core
        fence_before();
        __syncthreads();
        fence_after();
        const uint32_t tmem = *tslot;
        const uint32_t sa_hi = smem_u32(a_hi), sa_lo = smem_u32(a_lo), sb_hi = smem_u32(b_hi), sb_lo = smem_u32(b_lo);
        if (tid == 0) {
            issue_tile(tmem, 0, nblk, sa_hi, sa_lo, sb_hi, sb_lo);
            mma_commit(&bar[0]);
        }
        const uint32_t lane_base = (uint32_t)(32 * (warp % 4)) << 16;
        const int half = warp / 4;  // M-blocks half*16 .. half*16+15
        uint32_t ph[2] = {0u, 0u};
        const int tiles = steps / 8;
        for (int tl = 0; tl < tiles; ++tl) {
            const int buf = tl & 1;
            if (tl > 0 && V != 4) {
                fence_before();
                __syncthreads();  // every thread finished reading buffer buf^1 (tile tl-1)
                fence_after();
            }
            if (V != 4 && tid == 0 && tl + 1 < tiles) {
                issue_tile(tmem, (buf ^ 1) * 256, nblk, sa_hi, sa_lo, sb_hi, sb_lo);
                mma_commit(&bar[buf ^ 1]);
            }
            if (V != 4 || tl == 0) {
                mbar_wait(&bar[buf], ph[buf]);
                ph[buf] ^= 1u;
            }
            fence_after();
            if constexpr (V == 3) {
                if (tl == 0) {  // D of tile 0: rows blk*128 + lane, columns blk*8 + s
                    for (int i = 0; i < 16; ++i) {
                        const int blk = half * 16 + i;
                        if (blk >= nblk) break;
                        for (int s = 0; s < 8; ++s) {
                            const uint32_t v = ldtm1(tmem + lane_base + buf * 256 + blk * 8 + s);
                            ld_wait();
                            out[(size_t)(blk * 128 + 32 * (warp % 4) + (tid & 31)) * 8 + s] = __uint_as_float(v);
                        }
                    }
                }
                continue;
            }
#pragma unroll 1
            for (int s = 0; s < 8; ++s) {
                if constexpr (V == 1 || V == 4) {
                    uint32_t r[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) r[i] = ldtm1(tmem + lane_base + buf * 256 + (half * 16 + i) * 8 + s);
                    ld_wait();
#pragma unroll
                    for (int i = 0; i < 16; ++i) beta[i] += __uint_as_float(r[i]);
                } else if (V == 2 && (s & 1) == 0) {  // V == 2: two steps' columns per load
                    uint32_t r[32];
#pragma unroll
                    for (int i = 0; i < 16; ++i) ldtm2(tmem + lane_base + buf * 256 + (half * 16 + i) * 8 + s, r[2 * i], r[2 * i + 1]);
                    ld_wait();
#pragma unroll
                    for (int i = 0; i < 16; ++i) beta[i] += __uint_as_float(r[2 * i]) - __uint_as_float(r[2 * i + 1]);
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) {
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        float2 r2 = __ffma2_rn(make_float2(B[2 * k], B[2 * k + 1]),
                                               make_float2(g[(k * 8 + q) * 2], g[(k * 8 + q) * 2 + 1]), make_float2(gz[2 * q], gz[2 * q + 1]));
                        gz[2 * q] = r2.x;
                        gz[2 * q + 1] = r2.y;
                    }
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    B[i] = B[i] * 0.999f + 1e-7f * gz[i];
                    B[i + 8] = B[i + 8] * 0.999f + 1e-7f * beta[i];
                }
            }
        }
        fence_before();
        __syncthreads();
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
    if constexpr (V != 3) {
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i) s += gz[i] + beta[i];
        out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    }
}

static uint32_t tf32_rn(float x) {  // round to nearest (ties away) to 10 mantissa bits, as cvt.rna.tf32
    uint32_t u;
    memcpy(&u, &x, 4);
    u = (u + 0x1000u) & 0xFFFFE000u;
    return u;
}
static float f_of(uint32_t u) {
    float f;
    memcpy(&f, &u, 4);
    return f;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    // ---- accuracy: 16 blocks = 2048 rows, distinct hi/lo ----
    const int nb_acc = 16, rows = nb_acc * 128;
    std::vector<float> A((size_t)rows * 8), X(64);
    uint64_t st = 0x9E3779B97F4A7C15ull;
    auto rnd = [&]() {
        st = st * 6364136223846793005ull + 1442695040888963407ull;
        return ((st >> 40) * (1.0 / 16777216.0)) * 2.0 - 1.0;
    };
    for (auto& v : A) v = (float)rnd();
    for (auto& v : X) v = (float)(0.3 * rnd());
    std::vector<float> ahl((size_t)rows * 16), bhl(128);
    for (int e = 0; e < rows * 8; ++e) {
        const float hi = f_of(tf32_rn(A[e]));
        ahl[e] = hi;
        ahl[(size_t)rows * 8 + e] = f_of(tf32_rn(A[e] - hi));
    }
    for (int e = 0; e < 64; ++e) {
        const float hi = f_of(tf32_rn(X[e]));
        bhl[e] = hi;
        bhl[64 + e] = f_of(tf32_rn(X[e] - hi));
    }
    float *d_out, *d_in, *d_a, *d_b;
    cudaMalloc(&d_out, sizeof(float) * (size_t)256 * sms * 8 + sizeof(float) * rows * 8);
    cudaMalloc(&d_in, sizeof(float) * 256);
    cudaMalloc(&d_a, sizeof(float) * ahl.size());
    cudaMalloc(&d_b, sizeof(float) * bhl.size());
    cudaMemcpy(d_a, ahl.data(), sizeof(float) * ahl.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(d_b, bhl.data(), sizeof(float) * bhl.size(), cudaMemcpyHostToDevice);
    float h[256];
    for (int i = 0; i < 256; ++i) h[i] = 0.001f * (i % 97) - 0.03f;
    cudaMemcpy(d_in, h, sizeof(h), cudaMemcpyHostToDevice);
    const size_t smem_acc = 2 * Smem::a_bytes(nb_acc) + 512 + 64;
    const size_t smem_t = Smem::a_bytes(NBLK) + 512 + 64;
    cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_t);
    cudaFuncSetAttribute(probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_t);
    cudaFuncSetAttribute(probe<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_t);
    cudaFuncSetAttribute(probe<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_acc);
    probe<3><<<1, 256, smem_acc>>>(d_out, d_in, d_a, d_b, 8, nb_acc, 0);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("{\"error\": \"accuracy kernel: %s\"}\n", cudaGetErrorString(e));
        return 1;
    }
    std::vector<float> D((size_t)rows * 8);
    cudaMemcpy(D.data(), d_out, sizeof(float) * D.size(), cudaMemcpyDeviceToHost);
    double max_rel = 0, max_rel_1 = 0, max_abs_ref = 0;
    for (int m = 0; m < rows; ++m)
        for (int s = 0; s < 8; ++s) {
            double ref = 0, one = 0;
            for (int k = 0; k < 8; ++k) {
                ref += (double)A[(size_t)m * 8 + k] * X[s * 8 + k];
                one += (double)ahl[(size_t)m * 8 + k] * bhl[s * 8 + k];  // single TF32 product (hi.hi)
            }
            max_abs_ref = fmax(max_abs_ref, fabs(ref));
            max_rel = fmax(max_rel, fabs(D[(size_t)m * 8 + s] - ref));
            max_rel_1 = fmax(max_rel_1, fabs(one - ref));
        }
    printf("{\"accuracy\": {\"rows\": %d, \"max_abs_err_3xtf32\": %.3e, \"max_abs_err_1xtf32\": %.3e, \"max_abs_ref\": %.3e, "
           "\"rel_3xtf32\": %.3e, \"rel_1xtf32\": %.3e}}\n",
           rows, max_rel, max_rel_1, max_abs_ref, max_rel / max_abs_ref, max_rel_1 / max_abs_ref);

    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, auto kern, size_t smem) {
        const int blocks = sms * 4, threads = 256;
        for (int w = 0; w < 2; ++w) kern<<<blocks, threads, smem>>>(d_out, d_in, d_a, d_b, STEPS, NBLK, 1);
        cudaEventRecord(e0);
        kern<<<blocks, threads, smem>>>(d_out, d_in, d_a, d_b, STEPS, NBLK, 1);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaError_t er = cudaGetLastError();
        // per step and CTA: 256 threads x 256 FMA of the top level (G_{N-1} update + gz), whichever unit does them
        const double flop = 2.0 * 256.0 * STEPS * (double)threads * blocks;
        const double ns_step = ms * 1e6 / (STEPS * (double)blocks / sms);
        printf("{\"variant\": \"%s\", \"ms\": %.3f, \"ns_per_step_per_SM\": %.1f, \"equiv_fp32_tflops\": %.2f, \"err\": \"%s\"}\n", name,
               ms, ns_step, flop / (ms * 1e-3) / 1e12, cudaGetErrorString(er));
    };
    run("FFMA  (64 FFMA2 gz + 64 FFMA2 G_{N-1} per step)", probe<0>, 0);
    run("TMEM  (64 FFMA2 gz + 16 tcgen05.ld x1 + 96 MMA / 8 steps)", probe<1>, smem_t);
    run("TMEM2 (64 FFMA2 gz + 16 tcgen05.ld x2 every 2 steps + MMA)", probe<2>, smem_t);
    run("LDONLY(64 FFMA2 gz + 16 tcgen05.ld x1, no MMA / sync: the load cost alone)", probe<4>, smem_t);
    run("GZONLY(64 FFMA2 gz: lower bound of any offload)", probe<5>, 0);
    return 0;
}
