// top_loop_bench.cu -- dev microbenchmark of K2's top-level loop (the constant-G_N contractions).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/bin/top_loop_bench scripts/top_loop_bench.cu
//
// Per "step" each thread holds G_N for two sibling prefixes (2 x 64 floats) and does, per prefix,
//   beta[c] += sum_q G[c][q] z_q      (dot products, 64 FMA)
//   gz[q]   += sum_c B[c] G[c][q]      (rank-1 update, 64 FMA)
// i.e. 256 FMA per step, as in sig_bwd2p_kernel's top level, with 256 threads per CTA and one CTA per
// SM (two warps per SM sub-partition).  Variants differ only in register layout / instruction form:
//   PP   : prefix-pair float2 (G[c][q] of a and b in one pair): beta = FFMA2(G, z bcast, beta);
//          gz = FFMA2(B pair, G pair, gz pair)                        -- the current kernel
//   NAT  : natural layout (q pairs per prefix): gz = FFMA2(B bcast, G pair, gz pair);
//          beta = FFMA2(G pair, z pair, acc pair) + horizontal add     -- the round-1 kernel
//   NATS : natural layout, gz as NAT, beta as scalar FFMA chains
//   PPS  : prefix-pair layout, beta as PP, gz as scalar FFMA (B_a G_a, B_b G_b)
#include <cstdio>
#include <cuda_runtime.h>

constexpr int STEPS = 1024;

template <int V>
__global__ void __launch_bounds__(256, 1) top_loop(float* out, const float* in, int steps) {
    float g[128];  // G_N of the two prefixes (layout per variant)
#pragma unroll
    for (int i = 0; i < 128; ++i) g[i] = in[i] + threadIdx.x * 1e-3f;
    float beta[16], gz[16], B[16], z[8];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        beta[i] = 0.f;
        gz[i] = 0.f;
        B[i] = in[128 + i];
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) z[i] = in[144 + i];
    for (int s = 0; s < steps; ++s) {
        if constexpr (V == 0) {  // PP: g[(c*8+q)*2 + prefix]
#pragma unroll
            for (int k = 0; k < 8; ++k) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    float2 r = __ffma2_rn(make_float2(B[2 * k], B[2 * k + 1]), make_float2(g[(k * 8 + q) * 2], g[(k * 8 + q) * 2 + 1]),
                                          make_float2(gz[2 * q], gz[2 * q + 1]));
                    gz[2 * q] = r.x; gz[2 * q + 1] = r.y;
                }
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    float2 r = __ffma2_rn(make_float2(g[(c * 8 + k) * 2], g[(c * 8 + k) * 2 + 1]), make_float2(z[k], z[k]),
                                          make_float2(beta[2 * c], beta[2 * c + 1]));
                    beta[2 * c] = r.x; beta[2 * c + 1] = r.y;
                }
            }
        } else if constexpr (V == 1 || V == 2) {  // NAT: g[p*64 + c*8 + q]
#pragma unroll
            for (int p = 0; p < 2; ++p)
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const float b = B[p * 8 + c];
                    float2 acc = make_float2(0.f, 0.f);
                    float sacc = beta[p * 8 + c];
#pragma unroll
                    for (int q = 0; q < 8; q += 2) {
                        const float2 gg = make_float2(g[p * 64 + c * 8 + q], g[p * 64 + c * 8 + q + 1]);
                        float2 r = __ffma2_rn(make_float2(b, b), gg, make_float2(gz[q], gz[q + 1]));
                        gz[q] = r.x; gz[q + 1] = r.y;
                        if constexpr (V == 1) acc = __ffma2_rn(gg, make_float2(z[q], z[q + 1]), acc);
                        else sacc = fmaf(gg.y, z[q + 1], fmaf(gg.x, z[q], sacc));
                    }
                    if constexpr (V == 1) beta[p * 8 + c] += acc.x + acc.y;
                    else beta[p * 8 + c] = sacc;
                }
        } else {  // PPS
#pragma unroll
            for (int k = 0; k < 8; ++k) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    gz[2 * q] = fmaf(B[2 * k], g[(k * 8 + q) * 2], gz[2 * q]);
                    gz[2 * q + 1] = fmaf(B[2 * k + 1], g[(k * 8 + q) * 2 + 1], gz[2 * q + 1]);
                }
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    float2 r = __ffma2_rn(make_float2(g[(c * 8 + k) * 2], g[(c * 8 + k) * 2 + 1]), make_float2(z[k], z[k]),
                                          make_float2(beta[2 * c], beta[2 * c + 1]));
                    beta[2 * c] = r.x; beta[2 * c + 1] = r.y;
                }
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {  // step-dependent chain values and increments
            B[i] = B[i] * 0.999f + 1e-7f * gz[i];
            B[i + 8] = B[i + 8] * 0.999f + 1e-7f * beta[i];
            z[i] = z[i] * 0.999f + 1e-6f;
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += gz[i] + beta[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out, *in;
    cudaMalloc(&out, sizeof(float) * 256 * sms * 8);
    cudaMalloc(&in, sizeof(float) * 256);
    float h[256];
    for (int i = 0; i < 256; ++i) h[i] = 0.001f * (i % 97) - 0.03f;
    cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, auto kern) {
        const int blocks = sms * 4, threads = 256;
        for (int w = 0; w < 2; ++w) kern<<<blocks, threads>>>(out, in, STEPS);
        cudaEventRecord(e0);
        kern<<<blocks, threads>>>(out, in, STEPS);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flop = 2.0 * 256.0 * STEPS * (double)threads * blocks;  // 256 FMA per step
        printf("{\"variant\": \"%s\", \"fp32_tflops\": %.2f, \"ms\": %.3f}\n", name, flop / (ms * 1e-3) / 1e12, ms);
    };
    run("PP   (pair x pair gz, bcast beta)", top_loop<0>);
    run("NAT  (bcast gz, pair-z beta + hadd)", top_loop<1>);
    run("NATS (bcast gz, scalar beta)", top_loop<2>);
    run("PPS  (scalar gz, bcast beta)", top_loop<3>);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
