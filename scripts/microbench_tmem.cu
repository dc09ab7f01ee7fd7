// Microbenchmarks (sm_100a): TMEM load bandwidth per SM, and mbarrier arrive costs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb scripts/microbench_tmem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2402_15281_b200/csrc/ptx.cuh"

using namespace svn;

__global__ void tmem_bw(int iters, int nwarps_active, unsigned long long* out) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc(&slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    float acc = 0.f;
    unsigned long long t0 = clock64();
    if (warp < nwarps_active) {
        const uint32_t quad = warp & 3;
        for (int it = 0; it < iters; ++it) {
            for (int c = 0; c < 512; c += 64) {
                float v[64];
                tmem_ld64(tmem + ((quad * 32u) << 16) + c, v);
#pragma unroll
                for (int i = 0; i < 64; ++i) acc += v[i];
            }
        }
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 12345.f) out[1000] = 1;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

// cost of arrive flavours (single thread, N arrives on a local barrier with large count)
__global__ void __cluster_dims__(2, 1, 1) arrive_cost(int n, unsigned long long* out) {
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1u << 20);
        fence_mbar_init();
    }
    __syncthreads();
    cluster_sync_all();
    const uint32_t rank = cluster_ctarank();
    if (threadIdx.x == 0 && rank == 1) {
        const uint32_t remote = mapa_shared(smem_u32(&bar), 0);
        unsigned long long t0 = clock64();
        for (int i = 0; i < n; ++i) mbar_arrive_cluster(remote);
        unsigned long long t1 = clock64();
        for (int i = 0; i < n; ++i)
            asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
        unsigned long long t2 = clock64();
        for (int i = 0; i < n; ++i) {
            fence_proxy_async_smem();
            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
        }
        unsigned long long t3 = clock64();
        for (int i = 0; i < n; ++i) {
            asm volatile("fence.acq_rel.cluster;" ::: "memory");
            asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
        }
        unsigned long long t4 = clock64();
        out[0] = (t1 - t0) / n;
        out[1] = (t2 - t1) / n;
        out[2] = (t3 - t2) / n;
        out[3] = (t4 - t3) / n;
    }
    cluster_sync_all();
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 2048 * 8);
    unsigned long long h[1024];
    for (int nw : {4, 8, 16}) {
        tmem_bw<<<148, nw * 32>>>(2, nw, d);
        cudaDeviceSynchronize();
        const int iters = 50;
        tmem_bw<<<148, nw * 32>>>(iters, nw, d);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
        double bytes = double(iters) * 512 * 128 * 4 * (nw / 4);  // each quad warp reads 32 lanes x 512 cols
        printf("tmem ld x64: warps %2d  cycles %llu  B/clk/SM %.1f  (%s)\n", nw, h[0], bytes / h[0],
               cudaGetErrorString(e));
    }
    arrive_cost<<<2, 32>>>(1000, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 4 * 8, cudaMemcpyDeviceToHost);
    printf("remote arrive cycles: release.cluster %llu | default %llu | fence.proxy+release.cluster %llu | "
           "fence.acq_rel.cluster+relaxed %llu (%s)\n",
           h[0], h[1], h[2], h[3], cudaGetErrorString(e));
    return 0;
}
