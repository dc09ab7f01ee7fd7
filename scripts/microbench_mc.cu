// Semantics probe for a 4-CTA cluster (two CTA pairs): does a cta_group::2 multicast TMA
// issued by pair 0 deliver into both pairs and signal each destination pair's leader
// barrier, and does a cta_group::2 tcgen05.commit multicast reach all four CTAs?
// All waits are bounded (clock64 timeout), so a wrong guess reports instead of hanging.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/microbench_mc scripts/microbench_mc.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#include "../paper_2402_15281_b200/csrc/ptx.cuh"

using namespace svn;

constexpr int BR = 128;              // rows per CTA half
constexpr uint32_t HALF = BR * 128;  // 16 KiB

__device__ bool wait_bounded(uint64_t* bar, uint32_t parity) {
    const long long t0 = clock64();
    while (!mbar_try_wait(bar, parity))
        if (clock64() - t0 > 300000000LL) return false;
    return true;
}

__device__ __forceinline__ void tma_mc(void* dst, const void* tmap, int32_t c0, int32_t c1, uint32_t bar,
                                       uint16_t mask, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster.L2::cache_hint"
        " [%0], [%1, {%4, %5}], [%2], %3, %6;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar), "h"(mask), "r"(c0), "r"(c1), "l"(pol)
        : "memory");
}

// variant 0: mbar = mapa(full, 0) (pair-0 leader, shared::cluster)
// variant 1: mbar = own shared::cta address with the peer bit cleared (CUTLASS convention)
__global__ void __cluster_dims__(4, 1, 1) probe(const __grid_constant__ CUtensorMap tm, int variant, int4 expect, int* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full, empty;
    const uint32_t cr = cluster_ctarank();
    const uint32_t rank = cr & 1, pc = cr >> 1;
    if (threadIdx.x == 0) {
        mbar_init(&full, 1);
        mbar_init(&empty, 2);
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < HALF / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0xdeadbeefu;
    fence_proxy_async_smem();
    __syncthreads();
    cluster_sync_all();
    if (threadIdx.x == 0) {
        const int ex = cr == 0 ? expect.x : cr == 1 ? expect.y : cr == 2 ? expect.z : expect.w;
        if (ex >= 0) mbar_arrive_expect_tx_local(&full, static_cast<uint32_t>(ex));
        if (pc == 0) {
            const uint32_t bar = variant == 0 ? mapa_shared(smem_u32(&full), 0) : (smem_u32(&full) & 0xFEFFFFFFu);
            const uint16_t mask = static_cast<uint16_t>((1u << rank) | (1u << (2 + rank)));
            tma_mc(sm, &tm, 0, static_cast<int32_t>(rank * BR), bar, mask, policy_evict_last());
        }
        int ok_full = -1;
        if (ex >= 0) ok_full = wait_bounded(&full, 0) ? 1 : 0;
        out[cr] = ok_full;  // per CTA: own full-barrier wait result (-1: not armed)
    }
    cluster_sync_all();
    // data check: CTA with rank r must hold rows r*BR .. r*BR+127 (word = row id)
    int bad = 0;
    for (int i = threadIdx.x; i < HALF / 4; i += blockDim.x) {
        const uint32_t row = i / 32;
        if (reinterpret_cast<uint32_t*>(sm)[i] != rank * BR + row) ++bad;
    }
    atomicAdd(&out[64 + cr], bad);
    // commit multicast from each pair leader to all four CTAs (no MMA pending -> immediate arrive)
    if (threadIdx.x == 0 && rank == 0) {
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&empty)),
            "h"(static_cast<uint16_t>(0xF))
            : "memory");
    }
    if (threadIdx.x == 0) out[72 + cr] = wait_bounded(&empty, 0) ? 1 : 0;
    cluster_sync_all();
}

int main() {
    const int rows = 2 * BR;
    std::vector<uint32_t> h(rows * 32);
    for (int r = 0; r < rows; ++r)
        for (int w = 0; w < 32; ++w) h[r * 32 + w] = r;
    uint32_t* g;
    cudaMalloc(&g, h.size() * 4);
    cudaMemcpy(g, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    CUtensorMap tm;
    cuuint64_t dims[2] = {128, static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {128, BR};
    cuuint32_t es[2] = {1, 1};
    CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    int* d;
    cudaMalloc(&d, 128 * 4);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, HALF);
    const int4 cfgs[4] = {make_int4(2 * HALF, -1, 2 * HALF, -1), make_int4(HALF, HALF, HALF, HALF),
                          make_int4(2 * HALF, -1, -1, -1), make_int4(2 * HALF, -1, HALF, HALF)};
    for (int run = 0; run < 8; ++run) {
        const int variant = run & 1;
        const int4 ex = cfgs[run >> 1];
        cudaMemset(d, 0, 128 * 4);
        printf("expect {%d,%d,%d,%d} ", ex.x, ex.y, ex.z, ex.w);
        probe<<<4, 128, HALF>>>(tm, variant, ex, d);
        cudaError_t e = cudaDeviceSynchronize();
        int o[128];
        cudaMemcpy(o, d, sizeof(o), cudaMemcpyDeviceToHost);
        printf("variant %d (%s): %s | full-wait per cta %d %d %d %d | bad words %d %d %d %d | commit arrivals %d %d %d %d\n",
               variant, variant == 0 ? "mapa leader0" : "cta addr & ~peer", cudaGetErrorString(e),
               o[0], o[1], o[2], o[3], o[64], o[65], o[66], o[67], o[72], o[73], o[74], o[75]);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
