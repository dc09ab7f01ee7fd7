// FP32 FMA throughput with packed fma.rn.f32x2 in the register-tiled SGEMM pattern (8 x 8
// accumulators per thread as 8 x 4 pairs; the row operand duplicated into a pair once per
// step): does FFMA2 raise the attainable FP32 rate over FFMA (microbench_ffma2.cu)?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/microbench_ffma2_tile scripts/microbench_ffma2_tile.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pk(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}

__global__ void ffma2_tile(float* out, float s, int iters) {
    unsigned long long acc[8][4];
    float a[8], b[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        a[i] = s + i * 1e-3f + threadIdx.x * 1e-9f;
        b[i] = s - i * 1e-3f;
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0ull;
    }
    for (int it = 0; it < iters; ++it) {
        unsigned long long bp[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) bp[j] = pk(b[2 * j], b[2 * j + 1]);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const unsigned long long ap = pk(a[i], a[i]);
#pragma unroll
            for (int j = 0; j < 4; ++j) asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[i][j]) : "l"(ap), "l"(bp[j]));
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = __int_as_float(__float_as_int(a[i]) ^ (it & 1));
    }
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) t += __uint_as_float(static_cast<unsigned>(acc[i][j])) + __uint_as_float(static_cast<unsigned>(acc[i][j] >> 32));
    if (t == 12345.f) out[0] = t;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float* d;
    cudaMalloc(&d, 4);
    for (int threads : {128, 256, 512}) {
        const int iters = 40000;
        auto launch = [&] { ffma2_tile<<<sms, threads>>>(d, 1.0001f, iters); };
        launch();
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * 64 * iters * threads * static_cast<double>(sms);
        printf("FFMA2 8x8 tile threads/SM %4d: %.1f TFLOP/s (%.1f FMA/clk/SM at %.0f MHz nominal) %s\n", threads,
               flops / ms / 1e9, flops / 2 / (ms * 1e-3) / sms / (clk * 1e3), clk / 1e3,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
