// kernels_fp32.cu — K0 (per-motion q-fold), key init/finalise, and K1f: the fused
// fp32 SIMT MLP + min/argmin + margin kernel.
//
// K1f replaces the row loop of forward_eval (/root/reference/proj/src/nn.cpp:116-128)
// plus the argmin of predict_min_distance (nn.cpp:476-478) and the margin test
// (collision.cpp:68).  Each CTA owns a 64-row tile of one motion.  Activations stay
// in shared memory, transposed (actT[k][row]), between layers; weight rows stream
// through a 2-stage ring of 32 KiB bulk copies (cp.async.bulk, TMA engine).  Each
// hidden output is one sequential fmaf chain over k ascending — the same order as the
// reference's column axpy — and the output dot is the reference build's rounded-product
// in-order sum, so with `exact` set (no q-fold: bias, h part, x, q0, q1) the per-point
// delta matches the reference's own nn.cpp (oracle/ref) and the C restatement bit for bit.
#include <cuda_runtime.h>

#include <algorithm>

#include <cstdlib>

#include "fused.cuh"
#include "ptx.cuh"

namespace svn {

// ------------------------------------------------------------------ K0 ------
struct QNorm {
    float shift[kMaxIn], scale[kMaxIn];
};

// motion_bias[m][slot][c] = b[c] + sum_k Wq[slot][k][c] * zq_m[k]   (k ascending:
// q0 then q1), zq = (q - shift) * scale.  Block (m, slot), one thread per column.
// Also resets the per-motion keys/counters used by the fused finaliser.
__global__ void motion_bias_kernel(const float* __restrict__ q01, int64_t M, int dof, int N, int n_mb,
                                   const float* __restrict__ wq, const float* __restrict__ base_bias,
                                   float* __restrict__ motion_bias, const QNorm qn, unsigned long long* keys,
                                   unsigned int* counters, int64_t n_keys) {
    pdl_launch_dependents();  // the fused kernel may start its prologue now (it pdl_wait()s for our writes)
    const int64_t m = blockIdx.x;
    const int slot = blockIdx.y;
    if (keys && slot == 0 && threadIdx.x == 0 && m < n_keys) {
        keys[m] = ~0ull;
        counters[m] = 0u;
    }
    if (slot >= n_mb) return;
    __shared__ float zq[kMaxIn];
    const int nq = 2 * dof;
    if (threadIdx.x < nq) {
        const float q = q01[m * nq + threadIdx.x];
        zq[threadIdx.x] = __fmul_rn(__fsub_rn(q, qn.shift[threadIdx.x]), qn.scale[threadIdx.x]);
    }
    __syncthreads();
    const float* w = wq + static_cast<int64_t>(slot) * nq * N;
    for (int c = threadIdx.x; c < N; c += blockDim.x) {
        float acc = base_bias[slot * N + c];
        for (int k = 0; k < nq; ++k) acc = __fmaf_rn(zq[k], w[k * N + c], acc);
        motion_bias[(m * n_mb + slot) * N + c] = acc;
    }
}

cudaError_t launch_motion_bias(const FusedArgs& a, const float* wq, const float* mb_base_bias,
                               float* motion_bias, unsigned long long* keys_init, unsigned int* counters_init,
                               int64_t n_keys, cudaStream_t st) {
    if (a.M <= 0) return cudaSuccess;
    dim3 grid(static_cast<unsigned>(a.M), a.n_mb > 0 ? a.n_mb : 1);
    const int threads = a.N >= 256 ? 256 : 128;
    QNorm qn;
    for (int k = 0; k < 2 * a.dof && k < kMaxIn; ++k) {
        qn.shift[k] = a.shift[3 + k];
        qn.scale[k] = a.scale[3 + k];
    }
    motion_bias_kernel<<<grid, threads, 0, st>>>(a.q01, a.M, a.dof, a.N, a.n_mb, wq, mb_base_bias, motion_bias,
                                                 qn, keys_init, counters_init, n_keys);
    return cudaGetLastError();
}

__global__ void keys_init_kernel(unsigned long long* keys, int64_t M) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < M) keys[i] = ~0ull;
}

// Small host-buffer calls: the pinned staging block's inputs copied to the device by a kernel
// reading host memory directly (unified addressing) — for a few tens of KiB this lands sooner
// than a DMA copy, whose setup latency dominates at that size.  16-byte words, grid-stride.
__global__ void stage_in_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, int64_t n16) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n16;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        dst[i] = src[i];
}

cudaError_t launch_stage_in(const void* host_src, void* dev_dst, size_t bytes, cudaStream_t st) {
    const int64_t n16 = static_cast<int64_t>((bytes + 15) / 16);
    if (n16 <= 0) return cudaSuccess;
    const int64_t blocks = std::min<int64_t>((n16 + 255) / 256, 256);
    stage_in_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(static_cast<const uint4*>(host_src),
                                                                   static_cast<uint4*>(dev_dst), n16);
    return cudaGetLastError();
}

cudaError_t launch_keys_init(unsigned long long* keys, int64_t M, cudaStream_t st) {
    if (M <= 0) return cudaSuccess;
    keys_init_kernel<<<static_cast<unsigned>((M + 255) / 256), 256, 0, st>>>(keys, M);
    return cudaGetLastError();
}

__global__ void keys_finalize_kernel(const unsigned long long* keys, int64_t M, double margin, float* min_out,
                                     int32_t* argmin_out, uint8_t* free_out) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < M) decode_key(keys[i], margin, min_out + i, argmin_out + i, free_out + i);
}

cudaError_t launch_keys_finalize(const unsigned long long* keys, int64_t M, double margin, float* min_out,
                                 int32_t* argmin_out, uint8_t* free_out, cudaStream_t st) {
    if (M <= 0) return cudaSuccess;
    keys_finalize_kernel<<<static_cast<unsigned>((M + 255) / 256), 256, 0, st>>>(keys, M, margin, min_out,
                                                                                 argmin_out, free_out);
    return cudaGetLastError();
}

// Called by one thread after this CTA's atomicMin for `motion` is done.
__device__ __forceinline__ void tile_done(const FusedArgs& a, int32_t motion) {
    if (!a.counters) return;
    __threadfence();
    const unsigned int prev = atomicAdd(a.counters + motion, 1u);
    if (prev + 1 == static_cast<unsigned int>(a.tiles_per_motion)) {
        __threadfence();
        const unsigned long long key = atomicOr(a.keys + motion, 0ull);
        decode_key(key, a.margin, a.min_out + motion, a.argmin_out + motion, a.free_out + motion);
    }
}

// ------------------------------------------------------------------ K1f -----
// Packed fp32 pairs: fma.rn.f32x2 is two independent round-to-nearest fp32 FMAs, i.e. the
// same bits as two fmaf calls, at half the issue slots (an 8 x 8 register tile reaches 126
// FMA/clk/SM with it against 100 with FFMA, scripts/microbench_ffma2_tile.cu).
__device__ __forceinline__ unsigned long long f2_pack(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float f2_lo(unsigned long long v) { return __uint_as_float(static_cast<uint32_t>(v)); }
__device__ __forceinline__ float f2_hi(unsigned long long v) { return __uint_as_float(static_cast<uint32_t>(v >> 32)); }
__device__ __forceinline__ void f2_fma(unsigned long long& d, unsigned long long a, unsigned long long b) {
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}

// Weight chunks of 32 KiB, double-buffered: one barrier per 32 (width 256) or 16 (width 512)
// k steps, and the k loop over a full chunk unrolled completely.  Measured: 32 KiB x 2 with
// unroll 8 +6 % over 16 KiB x 4 with unroll 4 (FFMA); with the packed FFMA2 loop, unrolling
// the whole 32-step chunk +9 % on c2 over unroll 8 (+4 % on c3's network, where a chunk is
// 16 steps) (scripts/gpu_ab_fp32.sh; the -D overrides are A/B hooks).
#ifndef SVN_FP32_UNROLL
#define SVN_FP32_UNROLL 32
#endif
constexpr int kFp32Unroll = SVN_FP32_UNROLL;
#ifndef SVN_FP32_STAGES
#define SVN_FP32_STAGES 2
#endif
#ifndef SVN_FP32_CHUNK
#define SVN_FP32_CHUNK 8192  // floats per weight chunk
#endif
template <int N, int CG = 32, int TMO = 0>
struct Fp32Cfg {
    // rows per tile (activations must fit in smem); TMO = 32 for workloads with fewer tiles
    // than SMs, where per-warp issue, not the SM's FMA rate, bounds a tile
    static constexpr int TM = TMO ? TMO : (N >= 512 ? 64 : 128);
    static constexpr int THREADS = TM / 8 * CG;     // TM/8 row groups x CG column groups
    static constexpr int NC = N / CG;               // columns per thread (8 x NC register tile)
    static constexpr int KS = SVN_FP32_CHUNK / N;  // weight rows per chunk
    static constexpr int STAGES = SVN_FP32_STAGES;
    static constexpr int ACT_ROWS = N + kMaxIn;   // h rows then z rows
    static constexpr size_t ACT_BYTES = static_cast<size_t>(ACT_ROWS) * TM * 4;
    static constexpr size_t STAGE_BYTES = static_cast<size_t>(KS) * N * 4;
    static constexpr size_t SMEM = ACT_BYTES + STAGES * STAGE_BYTES + 64 + N * 4;  // + w_o
};

struct ChunkIter {
    int layer, chunk;
};

template <int N>
__device__ __forceinline__ int layer_rows(const FusedArgs& a, int l) {
    // exact: every row of wt[l]; folded: drop the q rows of concat layers.
    const bool concat = (l == 0) || (a.layer[l].flags & kConcat);
    return (a.exact || !concat) ? a.wt_rows[l] : a.wt_rows[l] - 2 * a.dof;
}

template <int N, int CG, int TMO>
__global__ void __launch_bounds__(Fp32Cfg<N, CG, TMO>::THREADS, 1) fused_fp32_kernel(const __grid_constant__ FusedArgs a) {
    using C = Fp32Cfg<N, CG, TMO>;
    extern __shared__ __align__(128) uint8_t smem[];
    float* actT = reinterpret_cast<float*>(smem);
    float* wst = reinterpret_cast<float*>(smem + C::ACT_BYTES);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::ACT_BYTES + C::STAGES * C::STAGE_BYTES);
    float* wo_s = reinterpret_cast<float*>(smem + C::ACT_BYTES + C::STAGES * C::STAGE_BYTES + 64);

    const int tid = threadIdx.x;
    const int cg = tid % CG, rg = tid / CG;
    // actT[k][row]: at width <= 256 the 16-byte chunks of row k are XOR-swizzled by
    // (k / 4) mod 8, so the epilogue's float4 stores (lanes of a warp 4 columns = 4 rows of
    // actT apart) hit 8 distinct bank groups instead of one (c2 +2.4 %); the k loop's loads
    // are warp broadcasts either way, and with 32-row weight chunks the XOR folds into the
    // unrolled k loop's constant offsets.  At width 512 (16-row chunks) it does not fold and
    // costs more than the conflicts (-7 %), so that layout stays plain.
    constexpr bool kSwizzle = N <= 256;
    auto act_at = [&](int k, int r) {
        return actT + k * C::TM + (kSwizzle ? (r ^ (((k >> 2) & 7) << 2)) : r);
    };
    const int L = a.L;

    // chunks per tile
    int chunks_per_tile = 0;
    for (int l = 0; l < L; ++l) chunks_per_tile += (layer_rows<N>(a, l) + C::KS - 1) / C::KS;
    int64_t my_tiles = 0;
    if (blockIdx.x < a.n_tiles) my_tiles = (a.n_tiles - 1 - blockIdx.x) / gridDim.x + 1;
    const int64_t total_chunks = my_tiles * chunks_per_tile;

    for (int k = tid; k < N; k += C::THREADS) wo_s[k] = a.wo[k];
    if (tid == 0) {
        for (int s = 0; s < C::STAGES; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    pdl_wait();  // K0 (per-motion biases, keys, counters) has completed

    // producer state (thread 0): issues chunk g_prod into stage g_prod % STAGES
    ChunkIter prod{0, 0};
    int64_t g_prod = 0;
    const uint64_t pol = policy_evict_last();
    auto issue = [&]() {
        const int rows = layer_rows<N>(a, prod.layer);
        const int r0 = prod.chunk * C::KS;
        const int nr = rows - r0 < C::KS ? rows - r0 : C::KS;
        const int s = static_cast<int>(g_prod % C::STAGES);
        const uint32_t bytes = static_cast<uint32_t>(nr) * N * 4u;
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(wst + static_cast<size_t>(s) * C::KS * N, a.wt[prod.layer] + static_cast<size_t>(r0) * N, bytes,
                 &full[s], pol);
        ++g_prod;
        if (r0 + C::KS >= rows) {
            prod.chunk = 0;
            prod.layer = prod.layer + 1 == L ? 0 : prod.layer + 1;
        } else {
            ++prod.chunk;
        }
    };
    if (tid == 0)
        while (g_prod < total_chunks && g_prod < C::STAGES) issue();

    int64_t g = 0;  // consumer chunk counter
    // phase accounting of thread 0 (SVN_KERNEL_PROF builds, scripts/fp32prof.py; zero otherwise)
    unsigned long long t_full = 0, t_bar = 0, t_epi = 0, t_out = 0;
    const unsigned long long t_start = prof_clock();
    for (int64_t t = blockIdx.x; t < a.n_tiles; t += gridDim.x) {
        int32_t motion, nrows;
        int64_t pbase, obase;
        tile_decode(a, t, C::TM, motion, pbase, obase, nrows);

        // z rows: actT[N + k][row] = (raw_k - shift_k) * scale_k
        if (tid < C::TM) {
            const int64_t pr = pbase + (tid < nrows ? tid : 0);
            const float* xp = a.points + pr * a.point_stride;
#pragma unroll
            for (int k = 0; k < 3; ++k)
                *act_at(N + k, tid) = __fmul_rn(__fsub_rn(xp[k], a.shift[k]), a.scale[k]);
            if (a.exact) {
                const float* q = a.row_q ? xp + 3 : a.q01 + static_cast<int64_t>(motion) * 2 * a.dof;
                for (int k = 0; k < 2 * a.dof; ++k)
                    *act_at(N + 3 + k, tid) = __fmul_rn(__fsub_rn(q[k], a.shift[3 + k]), a.scale[3 + k]);
            }
        }
        __syncthreads();

        for (int l = 0; l < L; ++l) {
            const LayerDev& ld = a.layer[l];
            const bool concat = (l == 0) || (ld.flags & kConcat);
            const float* bias = (!a.exact && concat && ld.mb_slot >= 0)
                                    ? a.motion_bias + (static_cast<int64_t>(motion) * a.n_mb + ld.mb_slot) * N
                                    : ld.bias;
            // acc[i][2p], acc[i][2p+1] as one packed pair (column pairs of the 8 x NC tile)
            unsigned long long acc[8][C::NC / 2];
#pragma unroll
            for (int j4 = 0; j4 < C::NC / 4; ++j4) {
                const float4 b4 = *reinterpret_cast<const float4*>(bias + cg * 4 + j4 * CG * 4);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    acc[i][j4 * 2 + 0] = f2_pack(b4.x, b4.y);
                    acc[i][j4 * 2 + 1] = f2_pack(b4.z, b4.w);
                }
            }
            const int rows = layer_rows<N>(a, l);
            const int a_off = (l == 0) ? N : 0;
            for (int r0 = 0; r0 < rows; r0 += C::KS) {
                const int s = static_cast<int>(g % C::STAGES);
                const unsigned long long w0 = prof_clock();
                mbar_wait(&full[s], static_cast<uint32_t>((g / C::STAGES) & 1));
                t_full += prof_clock() - w0;
                const float* w = wst + static_cast<size_t>(s) * C::KS * N;
                const int nk = rows - r0 < C::KS ? rows - r0 : C::KS;
                auto kstep = [&](int kk) {
                    const float4 a0 = *reinterpret_cast<const float4*>(act_at(a_off + r0 + kk, rg * 8));
                    const float4 a1 = *reinterpret_cast<const float4*>(act_at(a_off + r0 + kk, rg * 8 + 4));
                    const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                    unsigned long long wv[C::NC / 2];  // weight column pairs straight from a 16-byte load
#pragma unroll
                    for (int j4 = 0; j4 < C::NC / 4; ++j4) {
                        const ulonglong2 w2 = *reinterpret_cast<const ulonglong2*>(w + kk * N + cg * 4 + j4 * CG * 4);
                        wv[j4 * 2 + 0] = w2.x;
                        wv[j4 * 2 + 1] = w2.y;
                    }
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const unsigned long long ap = f2_pack(av[i], av[i]);
#pragma unroll
                        for (int j = 0; j < C::NC / 2; ++j) f2_fma(acc[i][j], ap, wv[j]);
                    }
                };
                if (nk == C::KS) {
                    // full chunk: unrolled so the next k's shared-memory loads are scheduled
                    // under the current k's FMAs (each output keeps its own k-ordered chain)
#pragma unroll kFp32Unroll
                    for (int kk = 0; kk < C::KS; ++kk) kstep(kk);
                } else {
                    for (int kk = 0; kk < nk; ++kk) kstep(kk);
                }
                const unsigned long long b0 = prof_clock();
                __syncthreads();  // every thread is done with stage s
                t_bar += prof_clock() - b0;
                if (tid == 0 && g_prod < total_chunks) issue();
                ++g;
            }
            const unsigned long long e0 = prof_clock();
            // epilogue: activation / folded BN / residual, written back in place
            const int fl = ld.flags;
            const bool act = fl & kAct, aff = fl & kAffine, res = (l > 0) && (fl & kResidual);
#pragma unroll
            for (int j4 = 0; j4 < C::NC / 4; ++j4) {
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const int col = cg * 4 + j4 * CG * 4 + jj;
                    const float sv = aff ? ld.s[col] : 0.f, tv = aff ? ld.t[col] : 0.f;
                    float* hlo = act_at(col, rg * 8);
                    float* hhi = act_at(col, rg * 8 + 4);
                    float hv[8];
                    if (res) {
                        const float4 h0 = *reinterpret_cast<const float4*>(hlo);
                        const float4 h1 = *reinterpret_cast<const float4*>(hhi);
                        hv[0] = h0.x, hv[1] = h0.y, hv[2] = h0.z, hv[3] = h0.w;
                        hv[4] = h1.x, hv[5] = h1.y, hv[6] = h1.z, hv[7] = h1.w;
                    }
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const unsigned long long pr = acc[i][j4 * 2 + (jj >> 1)];
                        float r = (jj & 1) ? f2_hi(pr) : f2_lo(pr);
                        if (act) r = r > 0.f ? r : 0.f;
                        if (aff) r = __fmaf_rn(r, sv, tv);
                        hv[i] = res ? __fadd_rn(hv[i], r) : r;
                    }
                    *reinterpret_cast<float4*>(hlo) = make_float4(hv[0], hv[1], hv[2], hv[3]);
                    *reinterpret_cast<float4*>(hhi) = make_float4(hv[4], hv[5], hv[6], hv[7]);
                }
            }
            __syncthreads();
            t_epi += prof_clock() - e0;
        }
        const unsigned long long o0 = prof_clock();

        // output layer: delta = sum_k w_o[k] h[k] + b_o; min/argmin.  nn.cpp:127's dot as the
        // reference's own build computes it (oracle/ref, g++ -O3 on Eigen's scalar redux): the
        // products rounded, then added in k order — no fused multiply-add in this chain
        if (tid < C::TM) {
            float acc = __fmul_rn(wo_s[0], *act_at(0, tid));
            // one k-ordered chain; unrolled so the shared loads run ahead of the adds
#pragma unroll 16
            for (int k = 1; k < N; ++k) acc = __fadd_rn(acc, __fmul_rn(wo_s[k], *act_at(k, tid)));
            const float delta = __fadd_rn(acc, a.bo);
            const bool valid = tid < nrows;
            if (valid && a.per_point) a.per_point[obase + tid] = delta;
            if (a.keys) {
                unsigned long long key = valid ? row_key(delta, a.index_offset + pbase + tid) : ~0ull;
                key = warp_min_u64(key);
                if ((tid & 31) == 0) atomicMin(a.keys + motion, key);
            }
        }
        __syncthreads();
        if (tid == 0 && a.keys) tile_done(a, motion);
        t_out += prof_clock() - o0;
    }
    if (a.prof && tid == 0) {  // slots: total, weight wait, chunk barrier, epilogue, output layer
        atomicAdd(a.prof + 0, prof_clock() - t_start);
        atomicAdd(a.prof + 1, t_full);
        atomicAdd(a.prof + 2, t_bar);
        atomicAdd(a.prof + 3, t_epi);
        atomicAdd(a.prof + 4, t_out);
    }
}

template <int N, int CG, int TMO = 0>
static cudaError_t launch_fp32_n(const FusedArgs& a, int num_sms, cudaStream_t st) {
    using C = Fp32Cfg<N, CG, TMO>;
    static SmemOptIn opt;
    cudaError_t e = opt.ensure(reinterpret_cast<const void*>(fused_fp32_kernel<N, CG, TMO>), (int)C::SMEM);
    if (e != cudaSuccess) return e;
    int64_t grid = a.n_tiles < num_sms ? a.n_tiles : num_sms;
    if (grid < 1) return cudaSuccess;
    const cudaError_t le = launch_fused_pdl(fused_fp32_kernel<N, CG, TMO>, static_cast<unsigned>(grid), C::THREADS,
                                            C::SMEM, st, a);
    return le != cudaSuccess ? le : cudaGetLastError();
}

static int fp32_cg() {
    static const int v = [] {
        const char* e = std::getenv("SVN_FP32_CG");
        return e ? std::atoi(e) : 16;  // 8x16 register tiles measured +5% over 8x8 on c2
    }();
    return v;
}

static int fp32_small_cg() {
    static const int v = [] {
        const char* e = std::getenv("SVN_FP32_SMALL_CG");
        return e ? std::atoi(e) : 64;  // width 512: 8 warps per 32-row tile, -3 % per call at 3000 points
    }();
    return v;
}

cudaError_t launch_fused_fp32(const FusedArgs& a, int num_sms, cudaStream_t st) {
    if (a.tile_rows == kFp32SmallTile) {  // few tiles: 32-row tiles, 4 warps each (64 columns gave 8 warps
        switch (a.N) {                     // but measured 8 % slower on c1)
            case 128: return launch_fp32_n<128, 32, kFp32SmallTile>(a, num_sms, st);
            case 256: return launch_fp32_n<256, 32, kFp32SmallTile>(a, num_sms, st);
            case 512:  // 8 warps per 32-row tile (8 x 8 register tiles); SVN_FP32_SMALL_CG=32: 4 warps
                return fp32_small_cg() == 64 ? launch_fp32_n<512, 64, kFp32SmallTile>(a, num_sms, st)
                                             : launch_fp32_n<512, 32, kFp32SmallTile>(a, num_sms, st);
            default: return cudaErrorInvalidValue;
        }
    }
    switch (a.N) {
        case 128: return launch_fp32_n<128, 32>(a, num_sms, st);
        case 256: return fp32_cg() == 16 ? launch_fp32_n<256, 16>(a, num_sms, st) : launch_fp32_n<256, 32>(a, num_sms, st);
        case 512: return launch_fp32_n<512, 32>(a, num_sms, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace svn

namespace svn {

// Voxel centres for dense-grid evaluation (SdfGrid::voxel_center, sweptvol.hpp:73-75):
// c = origin + voxel_size * i per axis, in double (contracted to one fma, as GCC emits for
// the reference's -march=native build), then cast to float like nn.cpp:469-471.
__global__ void grid_points_kernel(double ox, double oy, double oz, double vs, int dy, int dz, int64_t n,
                                   float* __restrict__ pts) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const int64_t iz = i % dz, iy = (i / dz) % dy, ix = i / (static_cast<int64_t>(dz) * dy);
    pts[3 * i + 0] = static_cast<float>(fma(vs, static_cast<double>(ix), ox));
    pts[3 * i + 1] = static_cast<float>(fma(vs, static_cast<double>(iy), oy));
    pts[3 * i + 2] = static_cast<float>(fma(vs, static_cast<double>(iz), oz));
}

cudaError_t launch_grid_points(const double* origin, double voxel, const int32_t* dims, float* pts, cudaStream_t st) {
    const int64_t n = static_cast<int64_t>(dims[0]) * dims[1] * dims[2];
    if (n <= 0) return cudaSuccess;
    grid_points_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(origin[0], origin[1], origin[2], voxel,
                                                                               dims[1], dims[2], n, pts);
    return cudaGetLastError();
}

}  // namespace svn
