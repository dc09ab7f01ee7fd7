// tcgen05.mma throughput on a CTA pair (cta_group::2, M=256, kind::f16, operands in smem,
// SW128 K-major): back-to-back MMAs of a given N, and the split kernel's per-kk pattern
// (3 x N=128 with A_hi read twice) against a merged pattern, all on 148 SMs at once.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/microbench_mma scripts/microbench_mma.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2402_15281_b200/csrc/ptx.cuh"

using namespace svn;

__host__ __device__ constexpr uint32_t idesc_f16(int m, int n) {
    return (1u << 4) | (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}

// mode 0: N=256 chain; 1: N=128 chain; 2: split pattern 3 x N=128 (hi.hi, hi.lo, lo.hi)
// mode 3: merged pattern N=256 (hi.[hi;lo]) + N=128 (lo.hi)
// mode 4: M=128 pair (64 rows per CTA, TMEM "2x2" layout) N=256 chain; 5: M=128 split pattern
// 3 x N=256; 6: M=128 N=128 chain
__global__ void __cluster_dims__(2, 1, 1) mma_bw(int mode, int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t done;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        mbar_init(&done, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc_pair(&slot, 512);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (cluster_ctarank() == 0 && threadIdx.x == 0) {
        const uint32_t a_hi = smem_u32(sm), a_lo = a_hi + 16384, b = a_hi + 32768;  // 16 KiB A slabs, 32 KiB B
        constexpr uint32_t i256 = idesc_f16(256, 256), i128 = idesc_f16(256, 128);
        constexpr uint32_t m128n256 = idesc_f16(128, 256), m128n128 = idesc_f16(128, 128);
        const unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const uint64_t ah = sw128_desc(a_hi + kk * 32), al = sw128_desc(a_lo + kk * 32);
                const uint64_t bh = sw128_desc(b + kk * 32), bl = sw128_desc(b + 16384 + kk * 32);
                if (mode == 0) {
                    mma_bf16_pair(tmem, ah, bh, i256, 1u);
                } else if (mode == 1) {
                    mma_bf16_pair(tmem, ah, bh, i128, 1u);
                } else if (mode == 2) {
                    mma_bf16_pair(tmem, ah, bh, i128, 1u);
                    mma_bf16_pair(tmem + 128, ah, bl, i128, 1u);
                    mma_bf16_pair(tmem + 128, al, bh, i128, 1u);
                } else if (mode == 3) {
                    mma_bf16_pair(tmem, ah, bh, i256, 1u);
                    mma_bf16_pair(tmem + 128, al, bh, i128, 1u);
                } else if (mode == 4) {
                    mma_bf16_pair(tmem, ah, bh, m128n256, 1u);
                } else if (mode == 5) {
                    mma_bf16_pair(tmem, ah, bh, m128n256, 1u);
                    mma_bf16_pair(tmem + 128, ah, bl, m128n256, 1u);
                    mma_bf16_pair(tmem + 128, al, bh, m128n256, 1u);
                } else {
                    mma_bf16_pair(tmem, ah, bh, m128n128, 1u);
                }
            }
        }
        mma_commit_pair(&done, 3);
        mbar_wait(&done, 0);
        if (blockIdx.x == 0) out[0] = clock64() - t0;
    } else if (cluster_ctarank() == 1 && threadIdx.x == 0) {
        mbar_wait(&done, 0);
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    if (warp == 0) tmem_dealloc_pair(tmem, 512);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(mma_bw, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const char* names[7] = {"N=256 chain", "N=128 chain", "split 3xN128", "merged N256+N128",
                            "M128 N=256 chain", "M128 split 3xN256", "M128 N=128 chain"};
    const double flop_per_it[7] = {4 * 256.0 * 256 * 16 * 2, 4 * 256.0 * 128 * 16 * 2, 3 * 4 * 256.0 * 128 * 16 * 2,
                                   (4 * 256.0 * 256 * 16 * 2 + 4 * 256.0 * 128 * 16 * 2),
                                   4 * 128.0 * 256 * 16 * 2, 3 * 4 * 128.0 * 256 * 16 * 2, 4 * 128.0 * 128 * 16 * 2};
    for (int mode = 0; mode < 7; ++mode) {
        const int iters = 4000;
        mma_bw<<<sms, 128, 96 * 1024>>>(mode, 10, d);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        mma_bw<<<sms, 128, 96 * 1024>>>(mode, iters, d);
        cudaEventRecord(e1);
        cudaError_t e = cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long cyc = 0;
        cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
        const double flops = flop_per_it[mode] * iters * (sms / 2);
        printf("%-18s %8.1f TFLOP/s  %6.1f cycles per kk-group (pair)  %s\n", names[mode], flops / ms / 1e9,
               static_cast<double>(cyc) / iters / 4, cudaGetErrorString(e));
    }
    return 0;
}
