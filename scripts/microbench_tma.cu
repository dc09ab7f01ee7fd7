// Per-SM L2 -> SMEM bulk-copy throughput (cp.async.bulk, 16 KiB chunks, S-stage ring),
// all SMs streaming the same L2-resident buffer, like the weight stream of the fused kernel.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include "../paper_2402_15281_b200/csrc/ptx.cuh"
using namespace svn;

template <int S, int CH>
__global__ void tma_bw(const uint8_t* src, size_t src_bytes, int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full[S];
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const uint64_t pol = policy_evict_last();
    const size_t nch = src_bytes / CH;
    unsigned long long t0 = clock64();
    int64_t issued = 0;
    for (; issued < S && issued < iters; ++issued) {
        mbar_arrive_expect_tx(&full[issued % S], CH);
        bulk_g2s(sm + (issued % S) * CH, src + ((blockIdx.x * 7 + issued) % nch) * CH, CH, &full[issued % S], pol);
    }
    for (int64_t i = 0; i < iters; ++i) {
        const int s = i % S;
        mbar_wait(&full[s], (i / S) & 1);
        if (issued < iters) {
            mbar_arrive_expect_tx(&full[s], CH);
            bulk_g2s(sm + s * CH, src + ((blockIdx.x * 7 + issued) % nch) * CH, CH, &full[s], pol);
            ++issued;
        }
    }
    unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
}

// 2-D tensor TMA version: tensor [rows][128 B], box [box_rows][128 B]
template <int S>
__global__ void tma2d_bw(const __grid_constant__ CUtensorMap tm, int rows_total, int box_rows, int iters,
                         unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full[S];
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const uint32_t CH = box_rows * 128;
    const int nch = rows_total / box_rows;
    unsigned long long t0 = clock64();
    int64_t issued = 0;
    auto issue = [&](int64_t k) {
        const int s = k % S;
        mbar_arrive_expect_tx(&full[s], CH);
        const int row = ((blockIdx.x * 7 + k) % nch) * box_rows;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
            ::"r"(smem_u32(sm + s * CH)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(smem_u32(&full[s])), "r"(0), "r"(row)
            : "memory");
    };
    for (; issued < S && issued < iters; ++issued) issue(issued);
    for (int64_t i = 0; i < iters; ++i) {
        mbar_wait(&full[i % S], (i / S) & 1);
        if (issued < iters) issue(issued++);
    }
    out[blockIdx.x] = clock64() - t0;
}

template <int S>
void run2d(void* src, size_t bytes, int box_rows, unsigned long long* d, int grid) {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p; cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
        fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    CUtensorMap tm;
    const int rows = bytes / 128;
    cuuint64_t dims[2] = {128, (cuuint64_t)rows};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    fn(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int iters = 2000;
    const int smem = S * box_rows * 128;
    cudaFuncSetAttribute(tma2d_bw<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    tma2d_bw<S><<<grid, 32, smem>>>(tm, rows, box_rows, 100, d);
    tma2d_bw<S><<<grid, 32, smem>>>(tm, rows, box_rows, iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("2D grid %3d stages %d chunk %5d: worst %.1f B/clk/SM, %.0f cyc/copy (%s)\n", grid, S, box_rows * 128,
           double(iters) * box_rows * 128 / mx, double(mx) / iters, cudaGetErrorString(e));
}

template <int S, int CH>
void run(const uint8_t* src, size_t bytes, unsigned long long* d, int grid) {
    const int iters = 2000;
    cudaFuncSetAttribute(tma_bw<S, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * CH);
    tma_bw<S, CH><<<grid, 32, S * CH>>>(src, bytes, 100, d);
    tma_bw<S, CH><<<grid, 32, S * CH>>>(src, bytes, iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0, sum = 0;
    for (int i = 0; i < grid; ++i) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
    printf("grid %3d stages %d chunk %5d: avg %.1f B/clk/SM, worst %.1f B/clk/SM, chip %.0f B/clk (%s)\n", grid, S, CH,
           double(iters) * CH / (double(sum) / grid), double(iters) * CH / mx, double(iters) * CH * grid / mx,
           cudaGetErrorString(e));
}

int main() {
    const size_t bytes = 3670016;
    uint8_t* src;
    cudaMalloc(&src, bytes);
    cudaMemset(src, 1, bytes);
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    // latency: one copy in flight at a time (stages = 1), all SMs
    run2d<1>(src, bytes, 128, d, 148);
    run2d<1>(src, bytes, 256, d, 148);
    run2d<2>(src, bytes, 256, d, 148);
    run2d<3>(src, bytes, 256, d, 148);
    run2d<1>(src, bytes, 128, d, 1);
    run2d<1>(src, bytes, 256, d, 1);
    run2d<2>(src, bytes, 128, d, 148);
    run2d<5>(src, bytes, 128, d, 148);
    return 0;
}
