// abi_internal.cuh — shared internals of the C-ABI implementation (abi_model.cu,
// abi_query.cu, abi_gcc.cu): the model object, error helpers, scratch / staging, and the
// kernel sequencing entry points the public functions are built from.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges for Nsight tools, no-ops otherwise

#include "../../include/sweptnet_b200.h"
#include "fused.cuh"
#include "gcc.cuh"
#include "ptx.cuh"

namespace svn {
namespace abi {

// thread-local state behind svn_last_error / svn_launch_count / svn_kernel_timing_*
extern thread_local std::string g_err;
extern thread_local int64_t g_launches;
extern thread_local bool g_timing;
extern thread_local std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_events;
extern thread_local unsigned long long g_prof[kProfSlots];

bool prof_enabled();
svn_status fail(svn_status code, const std::string& msg);
svn_status cuda_fail(cudaError_t e, const char* what);
svn_status host_exception();  // call from a catch (...) block

#define SVN_CUDA(call, what)                       \
    do {                                           \
        cudaError_t e_ = (call);                   \
        if (e_ != cudaSuccess) return cuda_fail(e_, what); \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

int layer_k(const svn_layer* layers, int l, int N, int in);
std::vector<float> fold_affine_bf16(const svn_model_desc* d, const float* params, int64_t n_params,
                                    std::vector<char>& folded);
svn_status validate_desc(const svn_model_desc* d);
svn_status encode_blob_map(CUtensorMap* map, const void* base, uint64_t row_bytes, uint64_t rows, uint32_t box_rows);
void split_bf16_host(float x, __nv_bfloat16& hi, __nv_bfloat16& lo);

}  // namespace abi
}  // namespace svn

struct svn_model {
    int device = 0;
    uint64_t serial = 0;  // unique per created model: keys the per-thread graph cache (abi_query.cu)
    int L = 0, N = 0, dof = 0, in = 0;
    int num_sms = 148;
    int n_mb = 0;
    std::vector<svn_layer> layers;
    std::vector<void*> allocs;
    svn::FusedArgs base{};        // model part of the kernel arguments
    svn::FusedArgs base_split{};  // width 256: fp32-accurate split-fp16 tensor-core kernel (kernels_split.cu)
    bool has_split = false;
    float* d_wq = nullptr;     // [n_mb][2dof][N]
    float* d_mbbase = nullptr; // [n_mb][N]
    float* d_wxslots = nullptr; // [n_mb][3][N] x-part columns of the concat layers
    bool has_bf16 = false;
    bool has_mixed = false;   // width-512 bf16: rows of mixed motions without per-motion folding
    svn::FusedArgs base_bf16{};       // bf16 kernels: base with the BN affine folded (see fold_affine_bf16)
    svn::FusedArgs base_f16{};        // the same kernels on fp16 operands (precision fp16): own weight / extension images
    bool has_f16 = false;             // every folded parameter fits the fp16 range
    float* d_wq_bf = nullptr;     // K0 inputs of the bf16 kernels, from the folded parameters
    float* d_mbbase_bf = nullptr;
    float* d_wxslots_bf = nullptr;

    template <class T>
    svn_status upload(const T* host, size_t count, T** out) {
        void* p = nullptr;
        cudaError_t e = cudaMalloc(&p, sizeof(T) * (count ? count : 1));
        if (e != cudaSuccess) return svn::abi::cuda_fail(e, "cudaMalloc(model)");
        allocs.push_back(p);
        if (count) {
            e = cudaMemcpy(p, host, sizeof(T) * count, cudaMemcpyHostToDevice);
            if (e != cudaSuccess) return svn::abi::cuda_fail(e, "cudaMemcpy(model)");
        }
        *out = static_cast<T*>(p);
        return SVN_OK;
    }
    ~svn_model() {
        svn::abi::DeviceGuard g(device);
        for (void* p : allocs) cudaFree(p);
    }
};

namespace svn {
namespace abi {

enum class Kind { BF16, SPLIT, SIMT };
svn_status check_prec(const svn_model* m, svn_precision prec);
Kind kernel_kind(const svn_model*, svn_precision prec);
int tile_rows(Kind k, int N);
int tile_rows_for(Kind k, int N, int64_t big_tiles, int num_sms);

// NVTX range for the duration of a scope (names the entry points and kernels in Nsight).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// Per-thread device scratch for the synchronous host-buffer entry points: a call's scratch
// (keys, counters, tile counter, extension rows) is carved from one block that is reused by
// the thread's next call (the call syncs its stream before returning), so a small call makes
// no allocation API calls.  A call that needs more falls back to stream-ordered allocation and
// the block grows to fit before the next one.
struct Arena {
    int device = -1;
    uint8_t* base = nullptr;
    size_t cap = 0, used = 0, need = 0;
    void begin() { used = need = 0; }
    static constexpr size_t kMaxBytes = size_t(64) << 20;  // larger calls keep stream-ordered scratch
    cudaError_t grow_to_need() {  // after the call's stream sync
        if (need <= cap || need > kMaxBytes) return cudaSuccess;
        release();
        size_t n = size_t(1) << 20;
        while (n < need) n <<= 1;
        cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&base), n);
        if (e == cudaSuccess) cap = n;
        return e;
    }
    void release() {
        if (base) cudaFree(base);
        base = nullptr;
        cap = 0;
    }
    ~Arena() { release(); }
};
extern thread_local Arena* g_arena;  // set for the duration of a synchronous call (ArenaScope)

struct ArenaScope {
    Arena* prev;
    explicit ArenaScope(Arena* a) : prev(g_arena) {
        a->begin();
        g_arena = a;
    }
    ~ArenaScope() { g_arena = prev; }
};

// Scratch buffers freed on the stream when the call's kernels are done (or carved from the
// thread's arena inside an ArenaScope).
struct Scratch {
    cudaStream_t st;
    std::vector<void*> ptrs;
    explicit Scratch(cudaStream_t s) : st(s) {}
    cudaError_t alloc(void** p, size_t bytes) {
        const size_t b = (bytes ? bytes : 16) + 255 & ~static_cast<size_t>(255);
        if (Arena* a = g_arena) {
            a->need += b;
            if (a->used + b <= a->cap) {
                *p = a->base + a->used;
                a->used += b;
                return cudaSuccess;
            }
        }
        cudaError_t e = cudaMallocAsync(p, b, st);
        if (e == cudaSuccess) ptrs.push_back(*p);
        return e;
    }
    ~Scratch() {
        for (void* p : ptrs) cudaFreeAsync(p, st);
    }
};

// Per-thread, per-device staging of the host-buffer entry points: one pinned host block and
// one device block, grown on demand and reused, so a call costs one H2D, one D2H and no
// allocation (calls are synchronous, so reuse after the stream sync is safe).
struct Staging {
    int device = -1;
    uint8_t* host = nullptr;
    uint8_t* dev = nullptr;
    size_t bytes = 0;
    cudaError_t reserve(int dev_id, size_t need) {
        if (need <= bytes && device == dev_id) return cudaSuccess;
        release();
        size_t n = 1 << 16;
        while (n < need) n <<= 1;
        cudaError_t e = cudaMallocHost(reinterpret_cast<void**>(&host), n);
        if (e != cudaSuccess) return e;
        e = cudaMalloc(reinterpret_cast<void**>(&dev), n);
        if (e != cudaSuccess) {
            cudaFreeHost(host);
            host = nullptr;
            return e;
        }
        bytes = n;
        device = dev_id;
        return cudaSuccess;
    }
    void release() {
        if (host) cudaFreeHost(host);
        if (dev) {
            int prev = 0;
            cudaGetDevice(&prev);
            cudaSetDevice(device);
            cudaFree(dev);
            cudaSetDevice(prev);
        }
        host = dev = nullptr;
        bytes = 0;
    }
    ~Staging() { release(); }  // thread exit (worker threads come and go)
};

Staging& thread_staging(int device);
Arena& thread_arena(int device);
inline size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }
void ensure_pool(int device);
cudaStream_t thread_stream(int device);

cudaError_t launch_k1(const FusedArgs& a, Kind kind, int num_sms, cudaStream_t st);
svn_status motion_ext(const svn_model* m, FusedArgs& a, int64_t M, unsigned long long* keys, unsigned int* counters,
                      int64_t n_keys, Scratch& sc, cudaStream_t st, bool split = false);
svn_status query_dense(const svn_model* m, svn_precision prec, const float* points, int64_t P, int64_t index_offset,
                       const float* q01, int64_t M, double margin, float* min_out, int32_t* argmin_out,
                       uint8_t* free_out, float* per_point, uint64_t* keys_partial, cudaStream_t st);
svn_status forward_rows(const svn_model* m, svn_precision prec, const float* raw_host, const float* raw_dev,
                        int64_t B, int64_t cols, float* out_dev, cudaStream_t st);

}  // namespace abi
}  // namespace svn
