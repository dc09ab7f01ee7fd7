// FP32 FMA throughput of one B200 (all SMs): 3-register FFMA chains and packed FFMA2, with
// 16 independent accumulators per thread; the measured denominator for the SIMT FP32 path.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/microbench_ffma scripts/microbench_ffma.cu
#include <cstdio>
#include <cuda_runtime.h>

template <bool PACKED>
__global__ void ffma_bw(float* out, float a0, float b0, int iters) {
    float acc[16];
    float a[4], b[4];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-7f + i;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        a[i] = a0 + i * 1e-3f;
        b[i] = b0 - i * 1e-3f;
    }
    for (int it = 0; it < iters; ++it) {
        if (PACKED) {
#pragma unroll
            for (int i = 0; i < 16; i += 2) {
                unsigned long long d, x, y;
                asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(acc[i]), "f"(acc[i + 1]));
                asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a[i & 3]), "f"(a[(i + 1) & 3]));
                asm("mov.b64 %0, {%1, %2};" : "=l"(y) : "f"(b[i & 3]), "f"(b[(i + 1) & 3]));
                asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(x), "l"(y));
                asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[i]), "=f"(acc[i + 1]) : "l"(d));
            }
        } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(acc[i]) : "f"(a[i & 3]), "f"(b[i & 3]));
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i];
    if (s == 12345.f) out[0] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* d;
    cudaMalloc(&d, 4);
    for (int packed = 0; packed < 2; ++packed)
        for (int threads : {256, 512, 1024}) {
            const int iters = 20000;
            auto launch = [&] {
                if (packed) ffma_bw<true><<<sms, threads>>>(d, 1.0001f, 0.9999f, iters);
                else ffma_bw<false><<<sms, threads>>>(d, 1.0001f, 0.9999f, iters);
            };
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
            const double flops = 2.0 * 16 * iters * threads * static_cast<double>(sms);
            int clk = 0;
            cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
            printf("%s threads/SM %4d: %.1f TFLOP/s (%.1f FMA/clk/SM at %.0f MHz nominal)  %s\n",
                   packed ? "FFMA2" : "FFMA ", threads, flops / ms / 1e9,
                   flops / 2 / (ms * 1e-3) / sms / (clk * 1e3), clk / 1e3, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
