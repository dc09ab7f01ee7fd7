// fused.cuh — launch parameters shared by the host ABI and the device kernels.
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace svn {

constexpr int kMaxLayers = 32;
constexpr int kMaxIn = 32;  // input_dim = 3 + 2*dof <= 32
// fp32_split truncation compensation per width (FusedArgs::rz_comp), calibrated on the B200
constexpr float kSplitRzComp256 = 0.18f;
constexpr float kSplitRzComp512 = 0.17f;
constexpr int kFp32SmallTile = 32;  // SIMT tile rows when a query has fewer big tiles than SMs

enum : int { kConcat = 1, kAct = 2, kAffine = 4, kResidual = 8 };

struct LayerDev {
    const float* bias;  // [N] layer bias (used when the layer has no folded motion bias)
    const float* s;     // [N] folded BN scale (affine layers)
    const float* t;     // [N] folded BN shift
    const float* wx;    // [3][N] fp32 x-part columns (concat layers), SoA
    int flags;          // kConcat | kAct | kAffine | kResidual
    int mb_slot;        // slot in the per-motion bias buffer, -1 if none
    int bias_zero;      // 1: every b_l == 0 and no folded motion bias (the add is skipped)
    int ext;            // bf16 pair kernel: K=16 extension slab 0 none, 1 model-constant, 2 per-motion
    int64_t ext_row;    // ext == 1: first 32-byte row of this layer in the model extension stream
};

// One unit of work: `nrows` consecutive rows of one motion.
struct TileDesc {
    int64_t point_base;  // first point (row) index
    int64_t out_base;    // first per-point output index
    int32_t motion;
    int32_t nrows;
};

struct FusedArgs {
    // TMA descriptors (bf16 CTA-pair kernel): blobs of pre-arranged smem images
    alignas(64) CUtensorMap tmap_w;   // weight stream viewed as [rows][128 B]
    alignas(64) CUtensorMap tmap_xm;  // model extension stream [rows][32 B]
    alignas(64) CUtensorMap tmap_xq;  // per-motion extension stream [rows][32 B]
    alignas(64) CUtensorMap tmap_xmix;  // width-512 bf16, rows of mixed motions: per (concat slot,
                                        // n-half, CTA half) 16 KiB = [b + x-part slab | 3 q slabs]
    // model
    int L, N, dof, in;
    LayerDev layer[kMaxLayers];
    const float* wo;  // [N]
    float bo;
    float shift[kMaxIn], scale[kMaxIn];  // input normaliser
    // weights
    const void* wstream;        // bf16: pre-swizzled tcgen05 weight stream for layers 1..L-1
    const float* wt[kMaxLayers];  // fp32: [K_l][N] transposed weights, rows (h | x | q)
    int wt_rows[kMaxLayers];      // rows in wt[l]
    // inputs
    const float* points;  // row r -> points[r * point_stride + 0..2]
    int64_t point_stride;
    int64_t P;            // points per motion (dense mode)
    const float* q01;     // [M][2*dof]
    int64_t M;
    const float* motion_bias;  // [M][n_mb][N]
    int n_mb;
    // work decomposition
    int64_t tiles_per_motion;  // dense mode
    int64_t n_tiles;
    const TileDesc* tiles;     // non-null: explicit tile table (forward_eval segments)
    int exact;                 // fp32 exact order (no q fold)
    int row_q;                 // exact mode: each row's q0|q1 follows its x in `points` (forward_eval
                               // rows of mixed motions; tiles then span motions)
    int mixed;                 // width-512 bf16 kernel (64 rows per CTA): rows of mixed motions, the
                               // q-part of every concat layer by the tensor core from per-row A slabs
    int tile_rows;             // rows per work item the host cut the tiles with (SIMT: 128/64, or 32)
    unsigned int* sched;       // width-512 bf16 kernel: dynamic tile counter (zeroed by K0)
    int tile_group;            // width-512 bf16 kernel: tiles per claimed chunk (1: per tile)
    int f16;                   // single-pass tensor-core kernels: operands in fp16 (precision fp16) instead of bf16
    // width-512 bf16 kernel: the per-motion K=16 extension rows (folded bias + x-part splits)
    // are built inside the fused kernel, by each CTA's output warp for the tile two ahead, into a
    // per-CTA ring of two tile slots (L2-resident) that tmap_xq views; null = the K0-built stream
    uint8_t* ext_ring;
    const float* xq_wq;    // [n_mb][2dof][N] q-columns of the concat layers (bf16 path's folded params)
    const float* xq_base;  // [n_mb][N] their bias
    // outputs
    unsigned long long* keys;  // [M] packed (orderable(delta) << 32 | index), or null
    unsigned int* counters;    // [M] tiles done, for the fused finaliser, or null
    int64_t index_offset;      // added to point indices in keys
    float* min_out;
    int32_t* argmin_out;
    uint8_t* free_out;
    double margin;
    float* per_point;          // [.. out_base + row], or null
    unsigned long long* prof;  // optional wait-time counters (clock64 cycles), see kProf*
    // fp32_split: the tensor core's fp32 accumulation truncates (rounds toward zero) once per
    // MMA instruction; the epilogue scales the main accumulator by 1 + rz_comp x (instructions
    // in the chain) x 2^-23 (scripts/emulate_split.py)
    float rz_comp;
};

// Wait/work accounting of the tensor-core kernels (scripts/profsum.py) costs ~1.3 % on c3, so
// its clock reads are compiled in only with -DSVN_KERNEL_PROF (SVN_NVCC_DEFINES=SVN_KERNEL_PROF
// python paper_2402_15281_b200/build.py); otherwise the counters stay zero.
__device__ __forceinline__ unsigned long long prof_clock() {
#ifdef SVN_KERNEL_PROF
    return clock64();
#else
    return 0ull;
#endif
}

// Instrumentation slots (summed over CTAs) when FusedArgs::prof is set.
enum : int {
    kProfMmaWaitA = 0,   // MMA issuer waiting for epilogue (a_ready)
    kProfMmaWaitFull,    // MMA issuer waiting for TMA (full)
    kProfMmaWaitAx,      // MMA issuer waiting for the A extension
    kProfMmaTotal,       // MMA issuer loop
    kProfEpiWaitD,       // epilogue waiting for the accumulator (d_full)
    kProfEpiWork,        // epilogue TMEM load + math + smem store
    kProfEpiArrive,      // epilogue fences + arrive
    kProfEpiOut,         // output dot exchange + keys
    kProfEpiAx,          // A extension writes
    kProfProdWaitEmpty,  // producer waiting for free slots
    kProfTimeline = 16,  // pp kernel: one round of CTA 0, [MMA wait, ready, committed] x (layer, slot), then
                         // [epilogue woke, worked, arrived] x (layer, slot)
    kProfSlots = 96
};

// Orderable-u32 map of a float: unsigned compare == float compare; NaN -> max.
__device__ __forceinline__ uint32_t orderable(float f) {
    uint32_t u = __float_as_uint(f);
    if ((u & 0x7fffffffu) > 0x7f800000u) return 0xffffffffu;  // NaN: never the min
    if (u == 0x80000000u) u = 0u;  // -0 == +0 under '<' (ties then go to the lowest index)
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ float from_orderable(uint32_t o) {
    const uint32_t u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
    return __uint_as_float(u);
}

// Key of one row.  A NaN at point index 0 sticks (nn.cpp:476-478: best starts at
// 0 and `pred[i] < NaN` is always false), so it gets key 0, the global minimum.
__device__ __forceinline__ unsigned long long row_key(float delta, int64_t point_index) {
    const bool nan = isnan(delta);
    if (nan && point_index == 0) return 0ull;
    return (static_cast<unsigned long long>(orderable(delta)) << 32) | static_cast<uint32_t>(point_index);
}

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}

// Decode a reduced key into the reference's (min, argmin) and the margin class.
__device__ __forceinline__ void decode_key(unsigned long long key, double margin, float* min_out,
                                           int32_t* argmin_out, uint8_t* free_out) {
    const uint32_t hi = static_cast<uint32_t>(key >> 32);
    float v;
    int32_t idx = static_cast<int32_t>(static_cast<uint32_t>(key));
    if (key == 0ull) {
        v = __uint_as_float(0x7fc00000u);  // NaN at index 0
        idx = 0;
    } else if (hi == 0xffffffffu) {
        v = __uint_as_float(0x7fc00000u);  // every row NaN (index 0 handled above)
    } else {
        v = from_orderable(hi);
    }
    *min_out = v;
    *argmin_out = idx;
    *free_out = static_cast<double>(v) > margin ? 1 : 0;  // strict, in double (collision.cpp:68)
}

// Work item t -> (motion, first point, first output index, valid rows).
__device__ __forceinline__ void tile_decode(const FusedArgs& a, int64_t t, int64_t TM, int32_t& motion,
                                            int64_t& pbase, int64_t& obase, int32_t& nrows) {
    if (a.tiles) {
        const TileDesc d = a.tiles[t];
        motion = d.motion;
        pbase = d.point_base;
        obase = d.out_base;
        nrows = d.nrows;
    } else {
        motion = static_cast<int32_t>(t / a.tiles_per_motion);
        pbase = (t % a.tiles_per_motion) * TM;
        obase = static_cast<int64_t>(motion) * a.P + pbase;
        const int64_t rem = a.P - pbase;
        nrows = static_cast<int32_t>(rem < TM ? rem : TM);
    }
}

// Opt a kernel into > 48 KiB of dynamic shared memory once per device; safe under concurrent
// host callers (a repeated set is idempotent, the per-device bit only skips the call).
struct SmemOptIn {
    std::atomic<unsigned long long> done{0ull};
    cudaError_t ensure(const void* kernel, int bytes) {
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return e;
        const unsigned long long bit = dev < 64 ? (1ull << dev) : 0ull;
        if (bit && (done.load(std::memory_order_acquire) & bit)) return cudaSuccess;
        e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        if (e == cudaSuccess && bit) done.fetch_or(bit, std::memory_order_release);
        return e;
    }
};

// The fused kernels are launched with programmatic stream serialization: their prologue
// (barrier init, TMEM allocation, tensor-map prefetch, w_o staging) overlaps the tail of K0,
// and they pdl_wait() before reading anything K0 wrote.  SVN_PDL=0 turns it off (A/B hook).
inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SVN_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <typename Kernel>
cudaError_t launch_fused_pdl(Kernel kernel, unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                             const FusedArgs& a) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, a);
}

// Launchers (kernels_*.cu).
cudaError_t launch_motion_bias(const FusedArgs& a, const float* wq /*[n_mb][2dof][N]*/,
                               const float* mb_base_bias /*[n_mb][N]*/, float* motion_bias,
                               unsigned long long* keys_init, unsigned int* counters_init, int64_t n_keys,
                               cudaStream_t st);
cudaError_t launch_keys_init(unsigned long long* keys, int64_t M, cudaStream_t st);
cudaError_t launch_stage_in(const void* host_src, void* dev_dst, size_t bytes, cudaStream_t st);
cudaError_t launch_grid_points(const double* origin, double voxel, const int32_t* dims, float* pts, cudaStream_t st);
cudaError_t launch_keys_finalize(const unsigned long long* keys, int64_t M, double margin, float* min_out,
                                 int32_t* argmin_out, uint8_t* free_out, cudaStream_t st);
cudaError_t launch_fused_fp32(const FusedArgs& a, int num_sms, cudaStream_t st);
cudaError_t launch_fused_bf16_pair(const FusedArgs& a, int num_sms, cudaStream_t st);
cudaError_t launch_fused_bf16_pp(const FusedArgs& a, int num_sms, cudaStream_t st);
cudaError_t launch_fused_split(const FusedArgs& a, int num_sms, cudaStream_t st);
cudaError_t launch_split_ext(const FusedArgs& a, const float* wq, const float* mb_base_bias, const float* wx_slots,
                             uint8_t* ext, unsigned long long* keys_init, unsigned int* counters_init, int64_t n_keys,
                             cudaStream_t st);
cudaError_t launch_ext_ring_init(uint8_t* ring, int64_t ctas, int n_mb, int N, const float* wx_slots, int f16,
                                 cudaStream_t st);
cudaError_t launch_motion_ext(const FusedArgs& a, const float* wq, const float* mb_base_bias, const float* wx_slots,
                              uint8_t* ext, unsigned long long* keys_init, unsigned int* counters_init,
                              int64_t n_keys, unsigned int* sched_reset, cudaStream_t st);

}  // namespace svn
