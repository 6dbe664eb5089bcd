// top_loop_bench.cu -- dev microbenchmark of the K2 top-level loop shape (prefix-pair layout).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tlb scripts/top_loop_bench.cu && /tmp/tlb
//
// Per "step" every thread runs, for c, q in [0, 8)^2 on float2 pairs:
//   gz[q] = fma2(B[c], G[c*8+q], gz[q])        (rank-1 gz update, B reused over q)
//   H[c]  = fma2(G[c*8+q], z[q] (bcast), H[c]) (dot product into the level-(N-1) gradient)
// i.e. 128 FFMA2 per step with 64 float2 of G (128 registers), as in sig_bwd2p_kernel's top level.
// Variants: which half of the loop runs, threads per CTA (1 CTA per SM), loop order.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int STEPS = 2048;

template <int MODE, int ORDER, int NT = 256>
__global__ void __launch_bounds__(NT, 1) top_loop(float* out, const float* in, int steps) {
    float2 G[64], gz[8], H[8], B[8];
    float z[8];
#pragma unroll
    for (int i = 0; i < 64; ++i) G[i] = make_float2(in[i & 31] + threadIdx.x, in[(i + 7) & 31]);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        gz[i] = make_float2(0.f, 0.f);
        H[i] = make_float2(in[i], in[i + 8]);
        B[i] = make_float2(in[i + 16], in[i + 3]);
        z[i] = in[i + 20] * 1e-3f;
    }
    for (int s = 0; s < steps; ++s) {
        if (ORDER == 0) {
#pragma unroll
            for (int c = 0; c < 8; ++c)
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (MODE & 1) gz[q] = __ffma2_rn(B[c], G[c * 8 + q], gz[q]);
                    if (MODE & 2) H[c] = __ffma2_rn(G[c * 8 + q], make_float2(z[q], z[q]), H[c]);
                }
        } else {
#pragma unroll
            for (int q = 0; q < 8; ++q)
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    if (MODE & 1) gz[q] = __ffma2_rn(B[c], G[c * 8 + q], gz[q]);
                    if (MODE & 2) H[c] = __ffma2_rn(G[c * 8 + q], make_float2(z[q], z[q]), H[c]);
                }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {  // keep B and z step-dependent (like the chain values)
            B[i].x += 1e-7f * gz[i].y;
            z[i] = z[i] * 0.999f + 1e-6f;
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += gz[i].x + gz[i].y + H[i].x + H[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out, *in;
    cudaMalloc(&out, sizeof(float) * 256 * sms * 8);
    cudaMalloc(&in, sizeof(float) * 64);
    cudaMemset(in, 0, sizeof(float) * 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, auto kern, double ffma2_per_step, int threads) {
        const int blocks = sms * 4;
        for (int w = 0; w < 2; ++w) kern<<<blocks, threads>>>(out, in, STEPS);
        cudaEventRecord(e0);
        kern<<<blocks, threads>>>(out, in, STEPS);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double fma = 2.0 * ffma2_per_step * STEPS * (double)threads * blocks;
        printf("{\"variant\": \"%s\", \"threads\": %d, \"fp32_tflops\": %.2f, \"ms\": %.3f}\n", name, threads,
               2.0 * fma / (ms * 1e-3) / 1e12, ms);
    };
    run("gz+H c-outer", top_loop<3, 0>, 128, 256);
    run("gz+H q-outer", top_loop<3, 1>, 128, 256);
    run("gz only", top_loop<1, 0>, 64, 256);
    run("H only", top_loop<2, 0>, 64, 256);
    run("gz+H c-outer 4 warps/SMSP", top_loop<3, 0, 512>, 128, 512);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
