// fma_peak.cu -- FP32 FMA throughput microbenchmark for the roofline denominator (B200, sm_100a).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fma_peak scripts/fma_peak.cu && ./fma_peak
//
// Variants (all: 8 warps/SMSP, 16 independent accumulator chains per thread, long unrolled loops):
//   ffma_reuse : acc_i = fma(acc_i, a, b)          -- a, b loop-invariant (reuse cache / 2 banks)
//   ffma_2par  : acc_i = fma(x_i, y_i, acc_i) with x_i, y_i of equal register parity (bank conflicts)
//   ffma2      : packed f32x2 acc_i = fma2(acc_i, a2, b2)
// Reports TFLOP/s (2 FLOP per FMA) and the SM clock.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void ffma_reuse(float* out, float a, float b) {
    float acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fmaf(acc[i], a, b);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ffma_vary(float* out, const float* in) {
    // acc_i += x_i * y_i with 16 distinct x and y per thread (3 distinct register sources)
    float x[16], y[16], acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        x[i] = in[i] + threadIdx.x;
        y[i] = in[16 + i] - threadIdx.x;
        acc[i] = 0.f;
    }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fmaf(x[i], y[i], acc[i]);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ffma2_reuse(float* out, float a, float b) {
    float2 acc[8];
    const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = __ffma2_rn(acc[i], a2, b2);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i].x + acc[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ffma2_vary(float* out, const float* in) {
    float2 x[8], y[8], acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        x[i] = make_float2(in[2 * i] + threadIdx.x, in[2 * i + 1]);
        y[i] = make_float2(in[16 + 2 * i], in[17 + 2 * i] - threadIdx.x);
        acc[i] = make_float2(0.f, 0.f);
    }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = __ffma2_rn(x[i], y[i], acc[i]);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i].x + acc[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const int threads = 1024, blocks = sms * 2;
    float *out, *in;
    cudaMalloc(&out, sizeof(float) * threads * blocks);
    cudaMalloc(&in, sizeof(float) * 64);
    cudaMemset(in, 0, sizeof(float) * 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, auto launch, double fmas_per_thread) {
        for (int w = 0; w < 3; ++w) launch();
        cudaEventRecord(e0);
        const int reps = 5;
        for (int r = 0; r < reps; ++r) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flop = 2.0 * fmas_per_thread * threads * blocks * reps;
        printf("{\"kernel\": \"%s\", \"tflops\": %.2f, \"ms\": %.3f}\n", name, flop / (ms * 1e-3) / 1e12, ms / reps);
    };
    run("ffma_reuse", [&] { ffma_reuse<<<blocks, threads>>>(out, 1.0001f, 1e-7f); }, 16.0 * ITERS);
    run("ffma_vary", [&] { ffma_vary<<<blocks, threads>>>(out, in); }, 16.0 * ITERS);
    run("ffma2_reuse", [&] { ffma2_reuse<<<blocks, threads>>>(out, 1.0001f, 1e-7f); }, 16.0 * ITERS);
    run("ffma2_vary", [&] { ffma2_vary<<<blocks, threads>>>(out, in); }, 16.0 * ITERS);
    printf("{\"sms\": %d, \"clock_khz_attr\": %d}\n", sms, clk);
    return 0;
}
