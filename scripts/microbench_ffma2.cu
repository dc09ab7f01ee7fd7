// FP32 FMA throughput, GEMM-microkernel pattern: each thread keeps an 8 x 8 accumulator
// tile and per step multiplies 8 "row" registers by 8 "column" registers (64 independent
// FFMAs per 16 operand registers, as in a register-tiled SGEMM).  Complements
// microbench_ffma.cu (16 chains on 4+4 shared operands).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/microbench_ffma2 scripts/microbench_ffma2.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ffma_tile(float* out, float s, int iters) {
    float acc[8][8];
    float a[8], b[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        a[i] = s + i * 1e-3f + threadIdx.x * 1e-9f;
        b[i] = s - i * 1e-3f;
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        // perturb operands so the compiler cannot hoist (one cheap op per 8 FMAs)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = __int_as_float(__float_as_int(a[i]) ^ (it & 1));
    }
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) t += acc[i][j];
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
        auto launch = [&] { ffma_tile<<<sms, threads>>>(d, 1.0001f, iters); };
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
        printf("FFMA 8x8 tile  threads/SM %4d: %.1f TFLOP/s (%.1f FMA/clk/SM at %.0f MHz nominal) %.2f ms %s\n", threads,
               flops / ms / 1e9, flops / 2 / (ms * 1e-3) / sms / (clk * 1e3), clk / 1e3, ms,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
