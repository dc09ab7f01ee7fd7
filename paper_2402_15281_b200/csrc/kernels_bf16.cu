// kernels_bf16.cu — K1: fused swept-volume MLP on tcgen05 tensor cores (sm_100a).
//
// Replaces, for one 128-point tile of one motion, the row loop of forward_eval
// (/root/reference/proj/src/nn.cpp:116-128), the argmin of predict_min_distance
// (nn.cpp:476-478) and the margin predicate (collision.cpp:68).
//
// Per CTA (persistent, one per SM), 10 warps:
//   warp 0      producer: streams the hidden-layer weights (bf16, pre-swizzled on the
//               host into the exact SW128 K-major smem image) with cp.async.bulk into a
//               ring of stages; one 16/32 KiB chunk = (N/2 rows) x (64 K) per stage.
//   warp 1      TMEM owner + MMA issuer: tcgen05.mma.cta_group::1.kind::f16, M=128,
//               N=N/2, K=16, A = activations in smem, B = weight stage, D in TMEM.
//   warps 2-9   epilogue: tcgen05.ld D -> +bias (per-motion folded bias on concat
//               layers) + fp32 x-part FMAs -> ReLU -> folded BN -> residual -> bf16 ->
//               st.shared into the next layer's A operand; on the last layer the
//               output dot, min/argmin key and the margin class.
// A layer is issued as four quarter-steps (n-half, k-half) in the order
// (0,0) (1,0) (0,1) (1,1).  The epilogue of output half 0 runs under MMA step (1,1);
// the epilogue of half 1 runs under step (0,0) of the next layer.  The activation
// tile is updated in place: k-half j of layer l+1's A is n-half j of layer l's output.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "fused.cuh"
#include "ptx.cuh"

namespace svn {

template <int N>
struct Bf16Cfg {
    static constexpr int TM = 128;                      // rows per tile (MMA M)
    static constexpr int NH = N / 2;                    // MMA N (one output half)
    static constexpr int KSL = NH / 64;                 // 64-wide K slabs per k-half
    static constexpr uint32_t A_SLAB = TM * 128;        // 16 KiB per 64-column slab
    static constexpr uint32_t A_BYTES = TM * N * 2;     // whole activation tile
    static constexpr uint32_t CHUNK = NH * 128;         // one weight stage
    static constexpr int STAGES = N >= 512 ? 3 : 6;
    static constexpr int EPI_WARPS = 8;
    static constexpr int THREADS = 64 + EPI_WARPS * 32;
    static constexpr int CPT = NH / 2 / 32;             // 32-col chunks per thread per half
    static constexpr uint32_t OFF_STAGE = A_BYTES;
    static constexpr uint32_t OFF_BAR = OFF_STAGE + STAGES * CHUNK;
    static constexpr uint32_t OFF_DOT = OFF_BAR + 256;
    static constexpr uint32_t SMEM = OFF_DOT + 2 * 2 * TM * 4;
    static_assert(SMEM <= 232448, "shared memory budget");
};

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    const __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&p);
}

__device__ __forceinline__ float bf16_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t u) { return __uint_as_float(u & 0xffff0000u); }

// Epilogue of one 32-column chunk for one row (this thread's row).
template <int N>
__device__ __forceinline__ void epi_chunk(const FusedArgs& a, const LayerDev& ld, int l, bool last,
                                          const float* __restrict__ bias, float (&v)[32], int c0, uint32_t row,
                                          float z0, float z1, float z2, uint8_t* A, float& dot) {
    const bool concat = (l == 0) || (ld.flags & kConcat);
    const int fl = ld.flags;
    const bool act = fl & kAct, aff = fl & kAffine, res = (l > 0) && (fl & kResidual);
    if (!concat && !aff && !res && !last) {
        // fast path (plain hidden layer): [+ bias] -> ReLU fused into the bf16 pack -> smem
        if (!ld.bias_zero) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
                const float4 b = __ldg(reinterpret_cast<const float4*>(bias + c0 + i));
                v[i + 0] += b.x;
                v[i + 1] += b.y;
                v[i + 2] += b.z;
                v[i + 3] += b.w;
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            uint4 p;
            if (act) {
                p.x = pack_bf16_relu(v[8 * u + 0], v[8 * u + 1]);
                p.y = pack_bf16_relu(v[8 * u + 2], v[8 * u + 3]);
                p.z = pack_bf16_relu(v[8 * u + 4], v[8 * u + 5]);
                p.w = pack_bf16_relu(v[8 * u + 6], v[8 * u + 7]);
            } else {
                p.x = pack_bf16(v[8 * u + 0], v[8 * u + 1]);
                p.y = pack_bf16(v[8 * u + 2], v[8 * u + 3]);
                p.z = pack_bf16(v[8 * u + 4], v[8 * u + 5]);
                p.w = pack_bf16(v[8 * u + 6], v[8 * u + 7]);
            }
            *reinterpret_cast<uint4*>(A + sw128_offset(row, c0 + 8 * u, 128)) = p;
        }
        return;
    }
    if (!ld.bias_zero) {
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
        const float4 b = __ldg(reinterpret_cast<const float4*>(bias + c0 + i));
        v[i + 0] += b.x;
        v[i + 1] += b.y;
        v[i + 2] += b.z;
        v[i + 3] += b.w;
    }
    }
    if (concat) {
        const float* wx = ld.wx;
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
            const float4 w0 = __ldg(reinterpret_cast<const float4*>(wx + c0 + i));
            const float4 w1 = __ldg(reinterpret_cast<const float4*>(wx + N + c0 + i));
            const float4 w2 = __ldg(reinterpret_cast<const float4*>(wx + 2 * N + c0 + i));
            v[i + 0] = fmaf(w2.x, z2, fmaf(w1.x, z1, fmaf(w0.x, z0, v[i + 0])));
            v[i + 1] = fmaf(w2.y, z2, fmaf(w1.y, z1, fmaf(w0.y, z0, v[i + 1])));
            v[i + 2] = fmaf(w2.z, z2, fmaf(w1.z, z1, fmaf(w0.z, z0, v[i + 2])));
            v[i + 3] = fmaf(w2.w, z2, fmaf(w1.w, z1, fmaf(w0.w, z0, v[i + 3])));
        }
    }
    if (act) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = v[i] > 0.f ? v[i] : 0.f;
    }
    if (aff) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
            const float4 s = __ldg(reinterpret_cast<const float4*>(ld.s + c0 + i));
            const float4 t = __ldg(reinterpret_cast<const float4*>(ld.t + c0 + i));
            v[i + 0] = fmaf(v[i + 0], s.x, t.x);
            v[i + 1] = fmaf(v[i + 1], s.y, t.y);
            v[i + 2] = fmaf(v[i + 2], s.z, t.z);
            v[i + 3] = fmaf(v[i + 3], s.w, t.w);
        }
    }
    if (res) {  // residual stream lives in the bf16 A tile (same address we overwrite)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint4 o = *reinterpret_cast<const uint4*>(A + sw128_offset(row, c0 + 8 * u, 128));
            v[8 * u + 0] += bf16_lo(o.x);
            v[8 * u + 1] += bf16_hi(o.x);
            v[8 * u + 2] += bf16_lo(o.y);
            v[8 * u + 3] += bf16_hi(o.y);
            v[8 * u + 4] += bf16_lo(o.z);
            v[8 * u + 5] += bf16_hi(o.z);
            v[8 * u + 6] += bf16_lo(o.w);
            v[8 * u + 7] += bf16_hi(o.w);
        }
    }
    if (last) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
            const float4 w = __ldg(reinterpret_cast<const float4*>(a.wo + c0 + i));
            dot = fmaf(w.x, v[i + 0], dot);
            dot = fmaf(w.y, v[i + 1], dot);
            dot = fmaf(w.z, v[i + 2], dot);
            dot = fmaf(w.w, v[i + 3], dot);
        }
    } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            uint4 p;
            p.x = pack_bf16(v[8 * u + 0], v[8 * u + 1]);
            p.y = pack_bf16(v[8 * u + 2], v[8 * u + 3]);
            p.z = pack_bf16(v[8 * u + 4], v[8 * u + 5]);
            p.w = pack_bf16(v[8 * u + 6], v[8 * u + 7]);
            *reinterpret_cast<uint4*>(A + sw128_offset(row, c0 + 8 * u, 128)) = p;
        }
    }
}

template <int N>
__global__ void __launch_bounds__(Bf16Cfg<N>::THREADS, 1) fused_bf16_kernel(const __grid_constant__ FusedArgs a) {
    using C = Bf16Cfg<N>;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* A = smem;
    uint8_t* stages = smem + C::OFF_STAGE;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
    uint64_t* full = bars;                   // [STAGES]
    uint64_t* empty = bars + C::STAGES;      // [STAGES]
    uint64_t* d_full = bars + 2 * C::STAGES; // [2]
    uint64_t* a_ready = d_full + 2;          // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a_ready + 2);
    float* dotbuf = reinterpret_cast<float*>(smem + C::OFF_DOT);  // [2 parity][2 ch][TM]

    const int warp = threadIdx.x >> 5;
    const uint32_t lane = lane_id();
    const int L = a.L;

    if (threadIdx.x == 0) {
        if (smem_u32(smem) & 1023u) __trap();  // SW128 operands need 1024-byte alignment
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(&d_full[0], 1);
        mbar_init(&d_full[1], 1);
        mbar_init(&a_ready[0], C::EPI_WARPS);
        mbar_init(&a_ready[1], C::EPI_WARPS);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, N);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------------ producer --
        if (lane == 0 && L > 1) {
            const uint64_t pol = policy_evict_last();
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t t = blockIdx.x; t < a.n_tiles; t += gridDim.x) {
                const uint8_t* src = static_cast<const uint8_t*>(a.wstream);
                for (int l = 1; l < L; ++l)
                    for (int step = 0; step < 4; ++step)
                        for (int ks = 0; ks < C::KSL; ++ks) {
                            mbar_wait(&empty[stage], phase ^ 1u);
                            mbar_arrive_expect_tx(&full[stage], C::CHUNK);
                            bulk_g2s(stages + stage * C::CHUNK, src, C::CHUNK, &full[stage], pol);
                            src += C::CHUNK;
                            if (++stage == C::STAGES) stage = 0, phase ^= 1u;
                        }
            }
        }
    } else if (warp == 1) {
        // ----------------------------------------------------------- MMA issuer --
        if (lane == 0 && L > 1) {
            constexpr uint32_t idesc = idesc_bf16(C::TM, C::NH);
            const uint32_t a_base = smem_u32(A);
            const uint32_t s_base = smem_u32(stages);
            int stage = 0;
            uint32_t phase = 0;
            uint32_t ar_phase[2] = {0u, 0u};
            for (int64_t t = blockIdx.x; t < a.n_tiles; t += gridDim.x) {
                for (int l = 1; l < L; ++l) {
                    for (int step = 0; step < 4; ++step) {
                        const int nh = step & 1, kh = step >> 1;
                        if (step < 2) {
                            mbar_wait(&a_ready[step], ar_phase[step]);
                            ar_phase[step] ^= 1u;
                            tc_fence_after();
                        }
                        const uint32_t d_addr = tmem + static_cast<uint32_t>(nh * C::NH);
                        for (int ks = 0; ks < C::KSL; ++ks) {
                            mbar_wait(&full[stage], phase);
                            tc_fence_after();
                            const uint32_t a_slab = a_base + static_cast<uint32_t>(kh * C::KSL + ks) * C::A_SLAB;
                            const uint32_t b_stage = s_base + static_cast<uint32_t>(stage) * C::CHUNK;
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk) {
                                const uint32_t acc = (kh | ks | kk) ? 1u : 0u;
                                mma_bf16(d_addr, sw128_desc(a_slab + kk * 32), sw128_desc(b_stage + kk * 32), idesc,
                                         acc);
                            }
                            mma_commit(&empty[stage]);
                            if (++stage == C::STAGES) stage = 0, phase ^= 1u;
                        }
                        if (step == 2) mma_commit(&d_full[0]);
                        if (step == 3) mma_commit(&d_full[1]);
                    }
                }
            }
        }
    } else {
        // ------------------------------------------------------------- epilogue --
        const int e = warp - 2;
        const uint32_t quad = static_cast<uint32_t>(warp & 3);
        const int ch = e >> 2;  // which quarter of each output half this warp owns
        const uint32_t row = quad * 32 + lane;
        const uint32_t t_lane = (quad * 32u) << 16;
        uint32_t dp[2] = {0u, 0u};
        int par = 0;
        for (int64_t t = blockIdx.x; t < a.n_tiles; t += gridDim.x) {
            int32_t motion, nrows;
            int64_t pbase, obase;
            tile_decode(a, t, C::TM, motion, pbase, obase, nrows);
            const bool valid = static_cast<int32_t>(row) < nrows;
            const float* xp = a.points + (pbase + (valid ? row : 0)) * a.point_stride;
            const float z0 = (xp[0] - a.shift[0]) * a.scale[0];
            const float z1 = (xp[1] - a.shift[1]) * a.scale[1];
            const float z2 = (xp[2] - a.shift[2]) * a.scale[2];
            const float* mb = a.motion_bias + static_cast<int64_t>(motion) * a.n_mb * N;
            float dot = 0.f;
            for (int l = 0; l < L; ++l) {
                const LayerDev& ld = a.layer[l];
                const bool last = (l == L - 1);
                const float* bias = ld.mb_slot >= 0 ? mb + ld.mb_slot * N : ld.bias;
                for (int j = 0; j < 2; ++j) {
                    if (l > 0) {
                        mbar_wait(&d_full[j], dp[j]);
                        dp[j] ^= 1u;
                        tc_fence_after();
                    }
#pragma unroll 1
                    for (int cc = 0; cc < C::CPT; cc += 2) {
                        const int c0 = j * C::NH + ch * (C::NH / 2) + cc * 32;
                        float v[64];
                        if (l > 0) {
                            tmem_ld64(tmem + t_lane + static_cast<uint32_t>(c0), v);
                        } else {
#pragma unroll
                            for (int i = 0; i < 64; ++i) v[i] = 0.f;
                        }
                        epi_chunk<N>(a, ld, l, last, bias, *reinterpret_cast<float(*)[32]>(&v[0]), c0, row, z0,
                                     z1, z2, A, dot);
                        epi_chunk<N>(a, ld, l, last, bias, *reinterpret_cast<float(*)[32]>(&v[32]), c0 + 32, row,
                                     z0, z1, z2, A, dot);
                    }
                    if (!last) {
                        tc_fence_before();
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&a_ready[j]);
                    }
                }
            }
            // output: combine the two column quarters, add b_o, reduce min/argmin
            dotbuf[(par * 2 + ch) * C::TM + row] = dot;
            named_bar_sync(1, C::EPI_WARPS * 32);
            if (ch == 0) {
                const float delta = (dotbuf[(par * 2) * C::TM + row] + dotbuf[(par * 2 + 1) * C::TM + row]) + a.bo;
                if (valid && a.per_point) a.per_point[obase + row] = delta;
                if (a.keys) {
                    unsigned long long key = valid ? row_key(delta, a.index_offset + pbase + row) : ~0ull;
                    key = warp_min_u64(key);
                    if (lane == 0) atomicMin(a.keys + motion, key);
                    named_bar_sync(2, 4 * 32);
                    if (e == 0 && lane == 0) {
                        if (a.counters) {
                            __threadfence();
                            const unsigned int prev = atomicAdd(a.counters + motion, 1u);
                            if (prev + 1 == static_cast<unsigned int>(a.tiles_per_motion)) {
                                __threadfence();
                                const unsigned long long k = atomicOr(a.keys + motion, 0ull);
                                decode_key(k, a.margin, a.min_out + motion, a.argmin_out + motion,
                                           a.free_out + motion);
                            }
                        }
                    }
                }
            }
            par ^= 1;
        }
    }

    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem, N);
}

template <int N>
static cudaError_t launch_bf16_n(const FusedArgs& a, int num_sms, cudaStream_t st) {
    using C = Bf16Cfg<N>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e =
            cudaFuncSetAttribute(fused_bf16_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    int64_t grid = a.n_tiles < num_sms ? a.n_tiles : num_sms;
    if (grid < 1) return cudaSuccess;
    fused_bf16_kernel<N><<<static_cast<unsigned>(grid), C::THREADS, C::SMEM, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_fused_bf16(const FusedArgs& a, int num_sms, cudaStream_t st) {
    switch (a.N) {
        case 256: return launch_bf16_n<256>(a, num_sms, st);
        case 512: return launch_bf16_n<512>(a, num_sms, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace svn
