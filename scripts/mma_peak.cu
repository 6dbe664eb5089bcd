// mma_peak.cu -- dev microbenchmark: throughput of the warp-level (legacy) mma.sync tensor-core
// path on sm_100a, TF32 m16n8k8 and BF16 m16n8k16, fp32 accumulate, 8 independent accumulators
// per warp, 8 warps per SM sub-partition.  Informs whether the constant-G_N top-level
// contractions of the backward could move to tensor cores without tcgen05.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_peak scripts/mma_peak.cu && ./mma_peak
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void mma_tf32(float* out) {
    unsigned a[4] = {threadIdx.x, threadIdx.x + 1, threadIdx.x + 2, threadIdx.x + 3};
    unsigned b[2] = {threadIdx.x * 3, threadIdx.x * 5};
    float d[8][4] = {};
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile(
                "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};"
                : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
                : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void mma_bf16(float* out) {
    unsigned a[4] = {threadIdx.x, threadIdx.x + 1, threadIdx.x + 2, threadIdx.x + 3};
    unsigned b[2] = {threadIdx.x * 3, threadIdx.x * 5};
    float d[8][4] = {};
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};"
                : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
                : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    cudaMalloc(&out, sizeof(float) * 1024 * sms * 2);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, auto kern, double flop_per_mma) {
        const int threads = 1024;
        for (int w = 0; w < 2; ++w) kern<<<sms, threads>>>(out);
        cudaEventRecord(e0);
        const int reps = 5;
        for (int r = 0; r < reps; ++r) kern<<<sms, threads>>>(out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flop = flop_per_mma * 8.0 * ITERS * (threads / 32) * (double)sms * reps;
        printf("{\"kernel\": \"%s\", \"tflops\": %.1f}\n", name, flop / (ms * 1e-3) / 1e12);
    };
    run("mma.sync m16n8k8 tf32", mma_tf32, 2.0 * 16 * 8 * 8);
    run("mma.sync m16n8k16 bf16", mma_bf16, 2.0 * 16 * 8 * 16);
    return 0;
}
