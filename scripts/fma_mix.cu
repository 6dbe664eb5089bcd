// fma_mix.cu -- dev microbenchmark: FP32 pipe throughput of FFMA2 / FFMA mixes at low occupancy.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fma_mix scripts/fma_mix.cu && ./fma_mix
// Each kernel: NCH independent float2 chains (FFMA2) plus NS independent scalar chains (FFMA) per
// iteration; launched with W warps per SM sub-partition (one CTA per SM, 4*W warps).
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;

template <int NCH, int NS>
__global__ void mix(float* out, float a, float b) {
    float2 acc[NCH > 0 ? NCH : 1];
    float s[NS > 0 ? NS : 1];
    const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
#pragma unroll
    for (int i = 0; i < NCH; ++i) acc[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
#pragma unroll
    for (int i = 0; i < NS; ++i) s[i] = threadIdx.x * 2e-3f + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < NCH; ++i) acc[i] = __ffma2_rn(acc[i], a2, b2);
#pragma unroll
        for (int i = 0; i < NS; ++i) s[i] = fmaf(s[i], a, b);
    }
    float r = 0;
#pragma unroll
    for (int i = 0; i < NCH; ++i) r += acc[i].x + acc[i].y;
#pragma unroll
    for (int i = 0; i < NS; ++i) r += s[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    cudaMalloc(&out, sizeof(float) * 1024 * sms * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, auto kern, int nch, int ns, int wps) {
        const int threads = 128 * wps;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        auto launch = [&] { kern<<<sms, threads, 200 * 1024>>>(out, 1.0001f, 1e-7f); };
        for (int w = 0; w < 2; ++w) launch();
        cudaEventRecord(e0);
        const int reps = 5;
        for (int r = 0; r < reps; ++r) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double fma = (2.0 * nch + ns) * ITERS * threads * (double)sms * reps;
        // pipe-cycles model: FFMA2 = 2 lane-slots, FFMA = 1
        printf("{\"kernel\": \"%s\", \"warps_per_smsp\": %d, \"fma_tflops\": %.2f}\n", name, wps, 2 * fma / (ms * 1e-3) / 1e12);
    };
    for (int w : {2, 4, 8}) {
        run("ffma2x8", mix<8, 0>, 8, 0, w);
        run("ffma2x4", mix<4, 0>, 4, 0, w);
        run("ffmax8", mix<0, 8>, 0, 8, w);
        run("ffma2x6+ffmax2", mix<6, 2>, 6, 2, w);
        run("ffma2x4+ffmax4", mix<4, 4>, 4, 4, w);
        run("ffma2x8+ffmax1", mix<8, 1>, 8, 1, w);
    }
    return 0;
}
