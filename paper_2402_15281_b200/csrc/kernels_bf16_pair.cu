// kernels_bf16_pair.cu — K1 (bf16): the fused swept-volume MLP on a CTA pair.
//
// Replaces, for a 256-point tile of one motion, the row loop of forward_eval
// (/root/reference/proj/src/nn.cpp:116-128), the argmin of predict_min_distance
// (nn.cpp:476-478) and the margin predicate (collision.cpp:68).
//
// Layout of the work: a cluster of 2 CTAs on one TPC issues tcgen05.mma.cta_group::2
// with M = 256 (128 rows per CTA), N = width/2 (one output half), K = 16.  Each CTA
// holds its 128 activation rows (bf16, SW128 K-major, the A operand) and half of each
// weight chunk (B operand); both are fed by TMA (cp.async.bulk.tensor ... cta_group::2)
// whose completion is counted on the leader CTA's mbarrier.  The accumulator for a
// whole layer (128 x width fp32 per CTA) lives in TMEM.
//
// Every affine term of a layer that is not the width x width product is computed by
// the tensor core too, as one extra K=16 "extension" slab: A_ext row = (1, 1, z_x in
// bf16 hi/lo splits), B_ext row = (b_hi, b_lo, W_x in bf16 hi/lo splits), giving the
// (per-motion folded) bias and the x-part to ~2^-16 relative.  Layer 0 is the extension
// alone.  The epilogue therefore only does ReLU (fused into the bf16 pack) and the
// store of the next layer's A operand — or, on the last layer, the output dot.
//
// Warps (per CTA): 0 TMA producer, 1 TMEM owner + MMA issuer (leader CTA only),
// 2..9 epilogue (two warps per TMEM lane quadrant, each owning half of every
// output half), 10 output warp (keys, per-point stores, the A extension of the tile
// two ahead — all off the epilogue warps' critical path).  A layer runs as quarter steps (n-half, k-half) in the order
// (0,0) (1,0) (0,1) (1,1); the epilogue of output half 0 overlaps step (1,1), that
// of half 1 overlaps step (0,0) of the next layer.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "fused.cuh"
#include "ptx.cuh"

namespace svn {

// TM_ = rows per CTA: 128 (M=256 pair MMAs, the throughput kernel) or 64 (M=128 pair MMAs,
// for launches with fewer 256-row tiles than CTA pairs: half the rows per tile halves the
// latency of a tile's pass through the network).  At TM=64 a CTA's 64 x NH accumulator sits in
// TMEM's "2x2" layout (lanes 0-63: columns 0..NH/2-1, lanes 64-127: columns NH/2..NH-1, NH/2
// TMEM columns); the B side (weights, extension rows) is the same at both sizes.
template <int N, int TM_ = 128>
struct PairCfg {
    static constexpr int TM = TM_;                   // rows per CTA (pair tile = 2 TM)
    static constexpr int NH = N / 2;                 // MMA N = one output half
    static constexpr int BR = NH / 2;                // B rows per CTA per chunk
    static constexpr int KSL = NH / 64;              // 64-wide K slabs per k-half
    static constexpr uint32_t A_SLAB = TM * 128;     // 16 KiB
    static constexpr uint32_t A_BYTES = TM * N * 2;
    static constexpr uint32_t AX_BYTES = TM * 32;    // K=16 extension of A (one slab)
    // per tile parity: the x slab, and at TM=64 three more for the per-row q-part of rows of
    // mixed motions (FusedArgs::mixed)
    static constexpr uint32_t AXP = TM == 64 ? 4 * AX_BYTES : AX_BYTES;
    static constexpr uint32_t CHUNK = BR * 128;      // per-CTA main weight chunk
    static constexpr uint32_t XCHUNK = BR * 32;      // per-CTA extension chunk
    static constexpr int STAGES = N >= 512 ? (TM == 128 ? 5 : 8) : 8;
    static constexpr int EPI_WARPS = 8;
    static constexpr int OUT_WARP = 2 + EPI_WARPS;   // keys / per-point outputs / A extensions
    static constexpr int THREADS = 64 + EPI_WARPS * 32 + 32;
    static constexpr int COLS = TM == 128 ? NH / 2 : NH / 4;  // columns per epilogue thread per half
    static constexpr int PARTS = TM == 128 ? 2 : 4;  // partial output dots per row (epilogue threads)
    static constexpr int RQ = TM / 32;               // 32-row groups per CTA (output warp)
    static constexpr uint32_t OFF_AX = A_BYTES;
    static constexpr uint32_t OFF_STAGE = OFF_AX + 2 * AXP;
    static constexpr uint32_t OFF_WO = OFF_STAGE + STAGES * CHUNK;
    static constexpr uint32_t OFF_DOT = OFF_WO + N * 4;
    static constexpr uint32_t OFF_BAR = OFF_DOT + 2 * PARTS * TM * 4;
    static constexpr int TQ = 8;                     // tile queue entries (dynamic schedule)
    static constexpr int XR = 3;                     // ext ring slots per CTA (tiles in flight)
    static constexpr uint32_t SMEM = OFF_BAR + 384;  // 22 + TQ barriers, TQ tile ids, TMEM slot
    static_assert(SMEM <= 232448, "shared memory budget");
    static_assert(COLS % 32 == 0, "epilogue works in 32-column TMEM loads");
};

// The A extension row of a point: (1, 1, z_x splits) against the B rows (b_hi, b_lo, W_x splits).
template <class F>
__device__ __forceinline__ void write_ax(uint8_t* ax, uint32_t row, float z0, float z1, float z2) {
    uint16_t h0, l0, h1, l1, h2, l2;
    F::split(z0, h0, l0);
    F::split(z1, h1, l1);
    F::split(z2, h2, l2);
    constexpr uint16_t one = F::kOne, zero = F::kZero;
    __align__(16) uint16_t v[16] = {one, one, h0, h0, l0, h1, h1, l1, h2, h2, l2, zero, zero, zero, zero, zero};
    *reinterpret_cast<uint4*>(ax + ext_offset(row, 0)) = *reinterpret_cast<const uint4*>(&v[0]);
    *reinterpret_cast<uint4*>(ax + ext_offset(row, 8)) = *reinterpret_cast<const uint4*>(&v[8]);
}

// Rows of mixed motions (FusedArgs::mixed): the row's own z_q as three more K=16 A slabs, z_q
// (motion_ext_kernel's arithmetic) in (hi, hi, lo) triples against the model's (hi, lo, hi) W_q
// triples — the same three-product split as the x-part.
template <class F>
__device__ __forceinline__ void write_axq(uint8_t* axq, uint32_t slab_bytes, uint32_t row, const float* q,
                                          const FusedArgs& a) {
    __align__(16) uint16_t v[48];
#pragma unroll
    for (int i = 0; i < 48; ++i) v[i] = F::kZero;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        if (k < 2 * a.dof) {
            uint16_t h, l;
            F::split(__fmul_rn(__fsub_rn(q[k], a.shift[3 + k]), a.scale[3 + k]), h, l);
            v[3 * k] = h;
            v[3 * k + 1] = h;
            v[3 * k + 2] = l;
        }
    }
#pragma unroll
    for (int sl = 0; sl < 3; ++sl)
#pragma unroll
        for (int h8 = 0; h8 < 2; ++h8)
            *reinterpret_cast<uint4*>(axq + sl * slab_bytes + ext_offset(row, 8 * h8)) =
                *reinterpret_cast<const uint4*>(&v[16 * sl + 8 * h8]);
}

// Epilogue of 32 columns of one row (the MMA already added bias and x-part).
template <int N, int TM, class F>
__device__ __forceinline__ void pair_epi32(const LayerDev& ld, int l, bool last, float* v, int c0, uint32_t row,
                                           uint8_t* A, const float* wo_s, float4& dot) {
    // fp16 operands: an activation (or input) beyond the fp16 range is stored as an infinity, and
    // every accumulator of that row in the next layer is then inf or NaN — which the ReLU pack
    // would turn into 0.  Two accumulators per 32-column chunk are tested; a hit poisons the
    // row's output dot (-inf, or NaN once the last layer adds to it), and the output warp
    // reports any non-finite delta as -inf.
    if (F::kHalf && (!(fabsf(v[0]) <= 3.0e38f) || !(fabsf(v[21]) <= 3.0e38f))) dot.x = -INFINITY;
    const int fl = ld.flags;
    const bool act = fl & kAct, aff = fl & kAffine, res = (l > 0) && (fl & kResidual);
    if (!aff && !res && last) {  // plain last layer: straight-line ReLU + output dot (four partial sums)
        if (act) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
                const float4 w = *reinterpret_cast<const float4*>(wo_s + c0 + i);
                dot.x = fmaf(w.x, v[i + 0] > 0.f ? v[i + 0] : 0.f, dot.x);
                dot.y = fmaf(w.y, v[i + 1] > 0.f ? v[i + 1] : 0.f, dot.y);
                dot.z = fmaf(w.z, v[i + 2] > 0.f ? v[i + 2] : 0.f, dot.z);
                dot.w = fmaf(w.w, v[i + 3] > 0.f ? v[i + 3] : 0.f, dot.w);
            }
        } else {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
                const float4 w = *reinterpret_cast<const float4*>(wo_s + c0 + i);
                dot.x = fmaf(w.x, v[i + 0], dot.x);
                dot.y = fmaf(w.y, v[i + 1], dot.y);
                dot.z = fmaf(w.z, v[i + 2], dot.z);
                dot.w = fmaf(w.w, v[i + 3], dot.w);
            }
        }
        return;
    }
    if (!aff && !res && !last) {  // hidden layer: ReLU fused into the bf16 pack
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            uint4 p;
            if (act) {
                p.x = F::pack_relu(v[8 * u + 0], v[8 * u + 1]);
                p.y = F::pack_relu(v[8 * u + 2], v[8 * u + 3]);
                p.z = F::pack_relu(v[8 * u + 4], v[8 * u + 5]);
                p.w = F::pack_relu(v[8 * u + 6], v[8 * u + 7]);
            } else {
                p.x = F::pack(v[8 * u + 0], v[8 * u + 1]);
                p.y = F::pack(v[8 * u + 2], v[8 * u + 3]);
                p.z = F::pack(v[8 * u + 4], v[8 * u + 5]);
                p.w = F::pack(v[8 * u + 6], v[8 * u + 7]);
            }
            *reinterpret_cast<uint4*>(A + sw128_offset(row, c0 + 8 * u, TM)) = p;
        }
        return;
    }
    if (act && res && !aff && !last) {  // folded Fig. 2 block: h~ += ReLU(a), as bf16x2
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            uint4* slot = reinterpret_cast<uint4*>(A + sw128_offset(row, c0 + 8 * u, TM));
            const uint4 o = *slot;
            uint4 p;
            p.x = F::add2(F::pack_relu(v[8 * u + 0], v[8 * u + 1]), o.x);
            p.y = F::add2(F::pack_relu(v[8 * u + 2], v[8 * u + 3]), o.y);
            p.z = F::add2(F::pack_relu(v[8 * u + 4], v[8 * u + 5]), o.z);
            p.w = F::add2(F::pack_relu(v[8 * u + 6], v[8 * u + 7]), o.w);
            *slot = p;
        }
        return;
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
    if (res) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint4 o = *reinterpret_cast<const uint4*>(A + sw128_offset(row, c0 + 8 * u, TM));
            v[8 * u + 0] += F::lo(o.x);
            v[8 * u + 1] += F::hi(o.x);
            v[8 * u + 2] += F::lo(o.y);
            v[8 * u + 3] += F::hi(o.y);
            v[8 * u + 4] += F::lo(o.z);
            v[8 * u + 5] += F::hi(o.z);
            v[8 * u + 6] += F::lo(o.w);
            v[8 * u + 7] += F::hi(o.w);
        }
    }
    if (last) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
            const float4 w = *reinterpret_cast<const float4*>(wo_s + c0 + i);
            dot.x = fmaf(w.x, v[i + 0], dot.x);
            dot.y = fmaf(w.y, v[i + 1], dot.y);
            dot.z = fmaf(w.z, v[i + 2], dot.z);
            dot.w = fmaf(w.w, v[i + 3], dot.w);
        }
    } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            uint4 p;
            p.x = F::pack(v[8 * u + 0], v[8 * u + 1]);
            p.y = F::pack(v[8 * u + 2], v[8 * u + 3]);
            p.z = F::pack(v[8 * u + 4], v[8 * u + 5]);
            p.w = F::pack(v[8 * u + 6], v[8 * u + 7]);
            *reinterpret_cast<uint4*>(A + sw128_offset(row, c0 + 8 * u, TM)) = p;
        }
    }
}

// The extension rows of one motion for this CTA's 2 x BR columns of every concat slot (four per
// lane per n-half) into `ring` ([slot][n-half] blobs of BR rows): b_m = b + W_q . z_q in fp32 with
// motion_ext_kernel's arithmetic (z_q = (q - shift) * scale; bias first, then q0, q1 in order),
// then its bf16 hi/lo split into the row's first word.  NQ = 2 * dof at compile time
// (0: runtime), so all 4 x NQ weight loads of an n-half are independent and issued together.
template <int BR, int NH, int NQ, class F>
__device__ __noinline__ void build_ext(const FusedArgs& a, int32_t motion, uint8_t* ring, uint32_t rank, uint32_t lane) {
    const int N = 2 * NH;
    const int nq = NQ > 0 ? NQ : 2 * a.dof;
    float zq[NQ > 0 ? NQ : kMaxIn];
#pragma unroll
    for (int j = 0; j < (NQ > 0 ? NQ : kMaxIn - 3); ++j)
        zq[j] = j < nq ? __fmul_rn(__fsub_rn(a.q01[static_cast<int64_t>(motion) * nq + j], a.shift[3 + j]), a.scale[3 + j])
                       : 0.f;
    for (int sl = 0; sl < a.n_mb; ++sl) {
        const float* __restrict__ w = a.xq_wq + static_cast<int64_t>(sl) * nq * N;
        const float* __restrict__ bb = a.xq_base + static_cast<int64_t>(sl) * N;
    #pragma unroll
        for (int nh = 0; nh < 2; ++nh) {
            int n[4];
            float acc[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                n[j] = nh * NH + static_cast<int>(rank) * BR + j * 32 + static_cast<int>(lane);
                acc[j] = __ldg(bb + n[j]);
            }
            if constexpr (NQ > 0) {
#pragma unroll
                for (int kq = 0; kq < NQ; ++kq)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[j] = __fmaf_rn(zq[kq], __ldg(w + kq * N + n[j]), acc[j]);
            } else {
                for (int kq = 0; kq < nq; ++kq)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[j] = __fmaf_rn(zq[kq], __ldg(w + kq * N + n[j]), acc[j]);
            }
            // only the b_m word of each row changes with the motion: the x-column splits of the
            // row (model constants) were written once per call by ext_ring_init_kernel
            uint8_t* blob = ring + (sl * 2 + nh) * BR * 32;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint16_t bh, bl;
                F::split(acc[j], bh, bl);
                const uint32_t rr = static_cast<uint32_t>(j * 32) + lane;
                *reinterpret_cast<uint32_t*>(blob + ext_offset(rr, 0)) =
                    static_cast<uint32_t>(bh) | (static_cast<uint32_t>(bl) << 16);
            }
        }
    }
}

template <int N, int TMR, class F>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PairCfg<N, TMR>::THREADS, 1)
    fused_bf16_pair_kernel(const __grid_constant__ FusedArgs a) {
    using C = PairCfg<N, TMR>;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* A = smem;
    uint8_t* AX = smem + C::OFF_AX;  // [2][AX_BYTES]
    uint8_t* stages = smem + C::OFF_STAGE;
    float* wo_s = reinterpret_cast<float*>(smem + C::OFF_WO);
    float* dotbuf = reinterpret_cast<float*>(smem + C::OFF_DOT);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
    uint64_t* full = bars;                      // [STAGES] leader: TMA bytes of both CTAs
    uint64_t* empty = full + C::STAGES;         // [STAGES] each CTA: slot consumed (MMA commit)
    uint64_t* d_full = empty + C::STAGES;       // [2] each CTA: output half j in TMEM
    uint64_t* a_ready = d_full + 2;             // [2] leader: epilogues of half j done (16 warps)
    uint64_t* ax_full = a_ready + 2;            // [2] leader: A extension buffer b written (2 output warps)
    uint64_t* out_full = ax_full + 2;           // [tile parity] each CTA: dotbuf holds a finished tile (8 warps)
    uint64_t* out_empty = out_full + 2;         // [tile parity] each CTA: output warp has read dotbuf
    uint64_t* tq_full = out_empty + 2;          // [TQ] each CTA: tile queue entry published
    uint64_t* xq_full = tq_full + C::TQ;        // [XR] each CTA: ext ring slot written (output warp)
    long long* tq = reinterpret_cast<long long*>(xq_full + C::XR);  // [TQ] each CTA: tile ids
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tq + C::TQ);

    const int warp = threadIdx.x >> 5;
    const uint32_t lane = lane_id();
    const uint32_t rank = cluster_ctarank();
    const int L = a.L;
    const int64_t pair = blockIdx.x >> 1;
    const int64_t npairs = gridDim.x >> 1;
    // Dynamic tile schedule: the pair's k-th tile is entry k of a queue that the leader's
    // output warp fills (tiles 0 and 1 = pair, pair + npairs; then the next unclaimed tile of
    // a global counter, two tiles ahead of use) and publishes to both CTAs.  Pairs whose SMs
    // run slower (e.g. farther from the L2 slices holding the weights) take fewer tiles
    // instead of finishing last; an id >= n_tiles ends the sequence.
    auto tile_at = [&](int64_t k) -> int64_t {
        mbar_wait_cluster(&tq_full[k % C::TQ], static_cast<uint32_t>((k / C::TQ) & 1));
        return *reinterpret_cast<volatile long long*>(&tq[k % C::TQ]);
    };

    if (threadIdx.x == 0) {
        if (smem_u32(smem) & 1023u) __trap();
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int j = 0; j < 2; ++j) {
            mbar_init(&d_full[j], 1);
            mbar_init(&a_ready[j], 2 * C::EPI_WARPS);
            mbar_init(&ax_full[j], 2);
            mbar_init(&out_full[j], C::EPI_WARPS);
            mbar_init(&out_empty[j], 1);
        }
        for (int q = 0; q < C::TQ; ++q) mbar_init(&tq_full[q], 1);
        for (int j = 0; j < C::XR; ++j) mbar_init(&xq_full[j], 1);
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < N; i += blockDim.x) wo_s[i] = a.wo[i];
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&a.tmap_w);
        prefetch_tmap(&a.tmap_xm);
        prefetch_tmap(&a.tmap_xq);
        if (C::TM == 64 && a.mixed) prefetch_tmap(&a.tmap_xmix);
    }
    if (warp == 1) tmem_alloc_pair(tmem_slot, N);
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();  // K0 (keys, counters, tile queue, extension rows) has completed

    if (warp == 0) {
        // ---------------------------------------------------------------- producer --
        if (lane == 0) {
            const uint64_t pol = policy_evict_last();
            const uint32_t full0 = mapa_shared(smem_u32(full), 0);
            int stage = 0;
            uint32_t phase = 0;
            unsigned long long pw_e = 0;
            auto slot = [&](uint32_t bytes_one_cta) {
                const unsigned long long c0 = prof_clock();
                mbar_wait(&empty[stage], phase ^ 1u);
                pw_e += prof_clock() - c0;
                if (rank == 0) mbar_arrive_expect_tx_local(&full[stage], 2 * bytes_one_cta);
            };
            auto advance = [&]() {
                if (++stage == C::STAGES) stage = 0, phase ^= 1u;
            };
            uint32_t xq_ph = 0u;  // phase bit per ring slot
            for (int64_t k = 0;; ++k) {
                const int64_t t = tile_at(k);
                if (t >= a.n_tiles) break;
                int32_t motion, nrows;
                int64_t pbase, obase;
                tile_decode(a, t, 2 * C::TM, motion, pbase, obase, nrows);
                const int xb = static_cast<int>(k % C::XR);
                if (a.ext_ring) {  // this tile's extension rows are in ring slot xb once the output warp says so
                    mbar_wait(&xq_full[xb], (xq_ph >> xb) & 1u);
                    xq_ph ^= 1u << xb;
                }
                int64_t wrow = 0;  // 128-byte row of the weight stream
                for (int l = 0; l < L; ++l) {
                    const LayerDev& ld = a.layer[l];
                    const int steps = l == 0 ? 2 : 4;
                    for (int step = 0; step < steps; ++step) {
                        const int nh = step & 1, kh = step >> 1;
                        if (kh == 0 && ld.ext) {
                            const uint32_t fb = full0 + stage * 8u;
                            uint8_t* dst = stages + stage * C::CHUNK;
                            if (C::TM == 64 && a.mixed && ld.ext == 2) {
                                // rows of mixed motions: the model's [b + x-part | q-part] slabs
                                slot(C::CHUNK);
                                tma_load_2d_pair(dst, &a.tmap_xmix, 0,
                                                 static_cast<int32_t>(((ld.mb_slot * 2 + nh) * 2 + rank) * 128), fb, pol);
                            } else if (ld.ext == 2) {
                                slot(C::XCHUNK);
                                const int64_t blob =
                                    a.ext_ring ? ((static_cast<int64_t>(blockIdx.x) * C::XR + xb) * a.n_mb + ld.mb_slot) * 2 + nh
                                               : ((static_cast<int64_t>(motion) * a.n_mb + ld.mb_slot) * 2 + nh) * 2 + rank;
                                tma_load_2d_pair(dst, &a.tmap_xq, 0, static_cast<int32_t>(blob * C::BR), fb, pol);
                            } else {
                                slot(C::XCHUNK);
                                const int64_t r0 = ld.ext_row + (nh * 2 + rank) * C::BR;
                                tma_load_2d_pair(dst, &a.tmap_xm, 0, static_cast<int32_t>(r0), fb, pol);
                            }
                            advance();
                        }
                        if (l > 0) {
                            for (int ks = 0; ks < C::KSL; ++ks) {
                                slot(C::CHUNK);
                                tma_load_2d_pair(stages + stage * C::CHUNK, &a.tmap_w, 0,
                                                 static_cast<int32_t>(wrow + rank * C::BR), full0 + stage * 8u, pol);
                                wrow += C::NH;
                                advance();
                            }
                        }
                    }
                }
            }
            if (a.prof && rank == 0) atomicAdd(a.prof + kProfProdWaitEmpty, pw_e);
        }
    } else if (warp == 1) {
        // -------------------------------------------------------------- MMA issuer --
        if (lane == 0 && rank == 0) {
            constexpr uint32_t idesc = F::idesc(2 * C::TM, C::NH);
            const uint32_t a_base = smem_u32(A), s_base = smem_u32(stages), ax_base = smem_u32(AX);
            int stage = 0;
            uint32_t phase = 0;
            uint32_t ar_ph[2] = {0u, 0u}, ax_ph[2] = {0u, 0u};
            unsigned long long pw_a = 0, pw_f = 0, pw_x = 0;
            const unsigned long long p_start = prof_clock();
            for (int64_t k = 0;; ++k) {  // local tile counter
                if (tile_at(k) >= a.n_tiles) break;
                const int b = static_cast<int>(k & 1);
                {
                    const unsigned long long c0 = prof_clock();
                    mbar_wait(&ax_full[b], ax_ph[b]);
                    pw_x += prof_clock() - c0;
                }
                ax_ph[b] ^= 1u;
                for (int l = 0; l < L; ++l) {
                    const LayerDev& ld = a.layer[l];
                    const int steps = l == 0 ? 2 : 4;
                    for (int step = 0; step < steps; ++step) {
                        const int nh = step & 1, kh = step >> 1;
                        if (kh == 0 && (k > 0 || l > 0)) {  // D[nh] drained / A[k-half nh] written
                            const unsigned long long c0 = prof_clock();
                            mbar_wait(&a_ready[nh], ar_ph[nh]);
                            pw_a += prof_clock() - c0;
                            ar_ph[nh] ^= 1u;
                        }
                        tc_fence_after();
                        const uint32_t d_addr = tmem + static_cast<uint32_t>(nh * C::NH);
                        bool acc = false;
                        if (kh == 0 && ld.ext) {
                            {
                                const unsigned long long c0 = prof_clock();
                                mbar_wait(&full[stage], phase);
                                pw_f += prof_clock() - c0;
                            }
                            tc_fence_after();
                            const uint32_t axb = ax_base + b * C::AXP, xs = s_base + stage * C::CHUNK;
                            mma_bf16_pair(d_addr, noswz_desc(axb, 128, 256), noswz_desc(xs, 128, 256), idesc, 0u);
                            if (C::TM == 64 && a.mixed && ld.ext == 2) {  // + the rows' q-part
#pragma unroll
                                for (int i = 1; i < 4; ++i)
                                    mma_bf16_pair(d_addr, noswz_desc(axb + i * C::AX_BYTES, 128, 256),
                                                  noswz_desc(xs + i * C::XCHUNK, 128, 256), idesc, 1u);
                            }
                            mma_commit_pair(&empty[stage], 3);
                            if (++stage == C::STAGES) stage = 0, phase ^= 1u;
                            acc = true;
                        }
                        if (l > 0) {
                            for (int ks = 0; ks < C::KSL; ++ks) {
                                {
                                    const unsigned long long c0 = prof_clock();
                                    mbar_wait(&full[stage], phase);
                                    pw_f += prof_clock() - c0;
                                }
                                tc_fence_after();
                                const uint32_t a_slab = a_base + static_cast<uint32_t>(kh * C::KSL + ks) * C::A_SLAB;
                                const uint32_t b_stage = s_base + static_cast<uint32_t>(stage) * C::CHUNK;
#pragma unroll
                                for (int kk = 0; kk < 4; ++kk) {
                                    mma_bf16_pair(d_addr, sw128_desc(a_slab + kk * 32), sw128_desc(b_stage + kk * 32),
                                                  idesc, (acc || kh || ks || kk) ? 1u : 0u);
                                }
                                mma_commit_pair(&empty[stage], 3);
                                if (++stage == C::STAGES) stage = 0, phase ^= 1u;
                            }
                        }
                        if (l == 0) mma_commit_pair(&d_full[nh], 3);
                        else if (step >= 2) mma_commit_pair(&d_full[step - 2], 3);
                    }
                }
            }
            if (a.prof) {
                atomicAdd(a.prof + kProfMmaWaitA, pw_a);
                atomicAdd(a.prof + kProfMmaWaitFull, pw_f);
                atomicAdd(a.prof + kProfMmaWaitAx, pw_x);
                atomicAdd(a.prof + kProfMmaTotal, prof_clock() - p_start);
            }
        }
    } else if (warp < C::OUT_WARP) {
        // ---------------------------------------------------------------- epilogue --
        const int e = warp - 2;
        const uint32_t quad = static_cast<uint32_t>(warp & 3);
        const int ch = e >> 2;
        // TM=128: lane quadrant = 32 rows, all of the n-half's columns.  TM=64 ("2x2"
        // accumulator): quadrants 0/1 = rows 0-31/32-63 of the n-half's columns 0..NH/2-1,
        // 2/3 = the same rows of columns NH/2..NH-1.
        const uint32_t row = (C::TM == 128 ? quad : (quad & 1u)) * 32 + lane;  // row within this CTA
        const int cq = C::TM == 128 ? 0 : static_cast<int>(quad >> 1) * (C::NH / 2);
        const int part = (C::TM == 128 ? 0 : static_cast<int>(quad >> 1) * 2) + ch;
        const uint32_t t_lane = (quad * 32u) << 16;
        const uint32_t a_ready0 = mapa_shared(smem_u32(a_ready), 0);
        uint32_t dp[2] = {0u, 0u}, oe_ph[2] = {0u, 0u};
        unsigned long long pe_d = 0, pe_w = 0, pe_a = 0, pe_o = 0;
        for (int64_t k = 0;; ++k) {
            if (tile_at(k) >= a.n_tiles) break;
            float4 dot = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int l = 0; l < L; ++l) {
                const LayerDev& ld = a.layer[l];
                const bool last = (l == L - 1);
                for (int j = 0; j < 2; ++j) {
                    const unsigned long long c0 = prof_clock();
                    mbar_wait(&d_full[j], dp[j]);
                    const unsigned long long c1 = prof_clock();
                    pe_d += c1 - c0;
                    dp[j] ^= 1u;
                    tc_fence_after();
                    {
                        // rolling pipeline over 32-column chunks: the next TMEM load is in
                        // flight while the current chunk is packed and stored
                        const int tc0 = j * C::NH + ch * C::COLS;  // TMEM column of the chunk
                        const int c0 = tc0 + cq;                   // its output column
                        constexpr int NCH = C::COLS / 32;
                        uint32_t ra[32], rb[32];
                        const uint32_t tb = tmem + t_lane;
                        tmem_ld32_async(tb + static_cast<uint32_t>(tc0), ra);
                        tmem_ld32_async(tb + static_cast<uint32_t>(tc0 + 32), rb);
                        tmem_wait_tied2(ra, rb);
#pragma unroll
                        for (int q = 0; q < NCH; q += 2) {
                            pair_epi32<N, C::TM, F>(ld, l, last, reinterpret_cast<float*>(ra), c0 + 32 * q, row, A, wo_s, dot);
                            if (q + 2 < NCH) tmem_ld32_async(tb + static_cast<uint32_t>(tc0 + 32 * (q + 2)), ra);
                            pair_epi32<N, C::TM, F>(ld, l, last, reinterpret_cast<float*>(rb), c0 + 32 * (q + 1), row, A, wo_s, dot);
                            if (q + 3 < NCH) tmem_ld32_async(tb + static_cast<uint32_t>(tc0 + 32 * (q + 3)), rb);
                            if (q + 2 < NCH) tmem_wait_tied2(ra, rb);
                        }
                    }
                    const unsigned long long c2 = prof_clock();
                    pe_w += c2 - c1;
                    tc_fence_before();
                    if (!last) fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_remote(a_ready0 + j * 8u);
                    pe_a += prof_clock() - c2;
                }
            }
            // hand the row's partial dot to the output warp (dotbuf[parity] is reused two tiles later)
            const unsigned long long c3 = prof_clock();
            const int b = static_cast<int>(k & 1);
            if (k >= 2) {
                mbar_wait(&out_empty[b], oe_ph[b]);
                oe_ph[b] ^= 1u;
            }
            dotbuf[(b * C::PARTS + part) * C::TM + row] = (dot.x + dot.y) + (dot.z + dot.w);
            __syncwarp();
            if (lane == 0) mbar_arrive(&out_full[b]);
            pe_o += prof_clock() - c3;
        }
        if (a.prof && e == 0 && lane == 0 && rank == 0) {
            atomicAdd(a.prof + kProfEpiWaitD, pe_d);
            atomicAdd(a.prof + kProfEpiWork, pe_w);
            atomicAdd(a.prof + kProfEpiArrive, pe_a);
            atomicAdd(a.prof + kProfEpiOut, pe_o);
        }
    } else {
        // ------------------------------------------------------------- output warp --
        // Per finished tile: delta = dot + bo for this CTA's 128 rows, per-point stores, one
        // packed-key atomicMin and the per-motion completion counter; then the A extension of
        // the tile two ahead (same parity), whose point loads are issued before the wait.
        const uint32_t ax_full0 = mapa_shared(smem_u32(ax_full), 0);
        uint32_t of_ph[2] = {0u, 0u};
        float px[C::RQ][3];
        float pq[C::TM == 64 ? C::RQ : 1][16];  // rows of mixed motions: each row's q0|q1
        unsigned long long pe_x = 0;
        auto load_points = [&](int64_t t) {
            int32_t motion, nrows;
            int64_t pbase, obase;
            tile_decode(a, t, 2 * C::TM, motion, pbase, obase, nrows);
#pragma unroll
            for (int q = 0; q < C::RQ; ++q) {
                const int32_t r = static_cast<int32_t>(rank * C::TM + q * 32 + lane);
                const float* xp = a.points + (pbase + (r < nrows ? r : 0)) * a.point_stride;
                px[q][0] = xp[0];
                px[q][1] = xp[1];
                px[q][2] = xp[2];
                if constexpr (C::TM == 64) {
                    if (a.mixed) {
#pragma unroll
                        for (int k = 0; k < 16; ++k) pq[q][k] = k < 2 * a.dof ? xp[3 + k] : 0.f;
                    }
                }
            }
        };
        auto store_ax = [&](int b) {
#pragma unroll
            for (int q = 0; q < C::RQ; ++q) {
                write_ax<F>(AX + b * C::AXP, static_cast<uint32_t>(q * 32) + lane,
                         (px[q][0] - a.shift[0]) * a.scale[0], (px[q][1] - a.shift[1]) * a.scale[1],
                         (px[q][2] - a.shift[2]) * a.scale[2]);
                if constexpr (C::TM == 64) {
                    if (a.mixed)
                        write_axq<F>(AX + b * C::AXP + C::AX_BYTES, C::AX_BYTES, static_cast<uint32_t>(q * 32) + lane, pq[q], a);
                }
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(ax_full0 + b * 8u);
        };
        // The per-motion extension rows of this CTA's 2 x BR columns per concat slot, for the tile
        // three ahead, into ring slot b (free: every MMA of the tile that used it has completed).
        // Same arithmetic as motion_ext_kernel (b_m = b + W_q . z_q in fp32, q0 then q1, then the
        // bf16 hi/lo splits); skipped when slot b already holds the tile's motion.
        int32_t ring_motion[C::XR];
#pragma unroll
        for (int j = 0; j < C::XR; ++j) ring_motion[j] = -1;
        auto write_ext = [&](int64_t t, int b) {
            if (!a.ext_ring) return;
            int32_t motion, nrows;
            int64_t pbase, obase;
            tile_decode(a, t, 2 * C::TM, motion, pbase, obase, nrows);
            if (motion != ring_motion[b]) {
                ring_motion[b] = motion;
                uint8_t* ring = a.ext_ring + (static_cast<int64_t>(blockIdx.x) * C::XR + b) * a.n_mb * 2 * C::BR * 32;
                switch (2 * a.dof) {  // compile-time q width: every load of a slot in flight at once
                    case 12: build_ext<C::BR, C::NH, 12, F>(a, motion, ring, rank, lane); break;
                    case 14: build_ext<C::BR, C::NH, 14, F>(a, motion, ring, rank, lane); break;
                    case 4: build_ext<C::BR, C::NH, 4, F>(a, motion, ring, rank, lane); break;
                    case 6: build_ext<C::BR, C::NH, 6, F>(a, motion, ring, rank, lane); break;
                    case 8: build_ext<C::BR, C::NH, 8, F>(a, motion, ring, rank, lane); break;
                    case 10: build_ext<C::BR, C::NH, 10, F>(a, motion, ring, rank, lane); break;
                    default: build_ext<C::BR, C::NH, 0, F>(a, motion, ring, rank, lane); break;
                }
                fence_proxy_async_global();  // generic-proxy writes -> the producer's TMA reads
                __threadfence();
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&xq_full[b]);
        };
        // the pair's scheduler: lane 0 of the leader's output warp
        const bool sched = rank == 0 && lane == 0;
        long long last_pub = 0;
        auto publish = [&](int64_t k, long long t) {
            const int q = static_cast<int>(k % C::TQ);
            tq[q] = t;
            st_cluster_s64(mapa_shared(smem_u32(&tq[q]), 1), t);
            mbar_arrive_cluster(mapa_shared(smem_u32(&tq_full[q]), 0));
            mbar_arrive_cluster(mapa_shared(smem_u32(&tq_full[q]), 1));
            last_pub = t;
        };
        // Tiles are handed out in chunks of G consecutive ids (one motion, mostly), so the ext ring
        // is rebuilt about once per chunk rather than per tile: the pair's first S = ceil(XR/G)
        // chunks are static (pair, pair + npairs, ...), later ones come from the counter.
        const int G = a.tile_group > 0 ? a.tile_group : 1;
        const int S = (C::XR + G - 1) / G;
        int s_used = 0, c_left = 0;
        long long c_next = 0;
        auto next_tile = [&]() -> long long {
            if (last_pub >= a.n_tiles) return last_pub;  // end marker, repeated
            if (c_left == 0) {
                const long long c = s_used < S ? pair + static_cast<long long>(s_used++) * npairs
                                               : static_cast<long long>(S) * npairs +
                                                     static_cast<long long>(atomicAdd(a.sched, 1u));
                c_next = c * G;
                c_left = G;
            }
            --c_left;
            const long long t = c_next++;
            return t < a.n_tiles ? t : a.n_tiles;
        };
        if (sched) {
            for (int j = 0; j < C::XR; ++j) publish(j, next_tile());
        }
        for (int b = 0; b < 2; ++b) {
            const int64_t t = tile_at(b);
            if (t < a.n_tiles) {
                load_points(t);
                store_ax(b);
            }
        }
        for (int j = 0; j < C::XR; ++j) {
            const int64_t t = tile_at(j);
            if (t < a.n_tiles) write_ext(t, j);
        }
        for (int64_t k = 0;; ++k) {
            const int64_t t = tile_at(k);
            if (t >= a.n_tiles) break;
            const int b = static_cast<int>(k & 1);
            if (sched)  // tile k+XR: the next unclaimed one, or the end marker once the counter ran out
                publish(k + C::XR, next_tile());
            __syncwarp();
            const int64_t t2 = tile_at(k + 2);
            const bool next = t2 < a.n_tiles;
            if (next) load_points(t2);
            int32_t motion, nrows;
            int64_t pbase, obase;
            tile_decode(a, t, 2 * C::TM, motion, pbase, obase, nrows);
            mbar_wait(&out_full[b], of_ph[b]);
            of_ph[b] ^= 1u;
            const unsigned long long c0 = prof_clock();
            // every MMA of tile t has completed, so AX[b] is free for tile t + 2 npairs
            if (next) store_ax(b);
            float delta[C::RQ];
#pragma unroll
            for (int q = 0; q < C::RQ; ++q) {
                const int r = q * 32 + static_cast<int>(lane);
                const float* d = dotbuf + (b * C::PARTS) * C::TM + r;
                delta[q] = (C::PARTS == 2 ? d[0] + d[C::TM] : (d[0] + d[C::TM]) + (d[2 * C::TM] + d[3 * C::TM])) + a.bo;
                // fp16 operands: an activation beyond the fp16 range is an infinity that spreads over
                // the row's later layers and arrives here as inf or NaN.  Such a row is reported as
                // -inf (its motion: min -inf, class "not free", handed to the exact checker — the safe
                // side of collision.cpp:68) instead of dropping out of the min as a NaN.
                if (F::kHalf && !(fabsf(delta[q]) <= 3.0e38f)) delta[q] = -INFINITY;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&out_empty[b]);
            unsigned long long key = ~0ull;
#pragma unroll
            for (int q = 0; q < C::RQ; ++q) {
                const int32_t rr = static_cast<int32_t>(rank * C::TM + q * 32 + lane);
                if (rr < nrows) {
                    if (a.per_point) a.per_point[obase + rr] = delta[q];
                    const unsigned long long kk = row_key(delta[q], a.index_offset + pbase + rr);
                    key = kk < key ? kk : key;
                }
            }
            if (a.keys) {
                key = warp_min_u64(key);
                if (lane == 0) {
                    atomicMin(a.keys + motion, key);
                    if (a.counters) {
                        __threadfence();
                        const unsigned int prev = atomicAdd(a.counters + motion, 1u);
                        if (prev + 1 == 2u * static_cast<unsigned int>(a.tiles_per_motion)) {
                            __threadfence();
                            const unsigned long long kk = atomicOr(a.keys + motion, 0ull);
                            decode_key(kk, a.margin, a.min_out + motion, a.argmin_out + motion, a.free_out + motion);
                        }
                    }
                }
            }
            // tile k+XR's extension rows into the slot tile k just released (needed when the producer
            // reaches that tile, about two tiles from now)
            {
                const int64_t t3 = tile_at(k + C::XR);
                if (t3 < a.n_tiles) write_ext(t3, static_cast<int>(k % C::XR));
            }
            pe_x += prof_clock() - c0;
        }
        if (a.prof && lane == 0 && rank == 0) atomicAdd(a.prof + kProfEpiAx, pe_x);
    }

    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    if (warp == 1) tmem_dealloc_pair(tmem, N);
}

template <int N, int TM, class F>
static cudaError_t launch_pair_n(const FusedArgs& a, int num_sms, cudaStream_t st) {
    using C = PairCfg<N, TM>;
    static SmemOptIn opt;
    cudaError_t e = opt.ensure(reinterpret_cast<const void*>(fused_bf16_pair_kernel<N, TM, F>), (int)C::SMEM);
    if (e != cudaSuccess) return e;
    int64_t pairs = num_sms / 2;
    if (a.n_tiles < pairs) pairs = a.n_tiles;
    if (pairs < 1) return cudaSuccess;
    const cudaError_t le = launch_fused_pdl(fused_bf16_pair_kernel<N, TM, F>, static_cast<unsigned>(2 * pairs),
                                            C::THREADS, C::SMEM, st, a);
    return le != cudaSuccess ? le : cudaGetLastError();
}

cudaError_t launch_fused_bf16_pair(const FusedArgs& a, int num_sms, cudaStream_t st) {
    switch (a.N) {
        case 256: return launch_fused_bf16_pp(a, num_sms, st);  // two tiles in flight (kernels_bf16_pp.cu)
        case 512:  // 128-row pair tiles for launches with fewer 256-row tiles than pairs (abi tile_rows_for)
            if (a.f16)  // fp16 operands (precision fp16): the same kernel on the other 16-bit format
                return a.tile_rows == 128 ? launch_pair_n<512, 64, FmtF16>(a, num_sms, st)
                                          : launch_pair_n<512, 128, FmtF16>(a, num_sms, st);
            return a.tile_rows == 128 ? launch_pair_n<512, 64, FmtBf16>(a, num_sms, st)
                                      : launch_pair_n<512, 128, FmtBf16>(a, num_sms, st);
        default: return cudaErrorInvalidValue;
    }
}

// The motion-independent part of every ext ring row (K slots 2..15: the slot's x-column splits;
// slots 0..1, the b_m word, are written by the fused kernel per motion).  One thread per row of
// the ring [cta slot][mb slot][n-half] blobs of N/4 rows; column n of a row follows the pair
// kernel's blob order (n-half, CTA rank within the pair).
template <class F>
__global__ void ext_ring_init_kernel(uint8_t* __restrict__ ring, int64_t n_blobs, int n_mb, int N,
                                     const float* __restrict__ wx_slots, int xr) {
    const int BR = N / 4, NH = N / 2;
    const int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (row >= n_blobs * BR) return;
    const int64_t blob = row / BR;
    const uint32_t rr = static_cast<uint32_t>(row % BR);
    const int nh = static_cast<int>(blob % 2);
    const int sl = static_cast<int>((blob / 2) % n_mb);
    const int64_t cta = blob / (2 * n_mb) / xr;
    const int n = nh * NH + static_cast<int>(cta & 1) * BR + static_cast<int>(rr);
    const float* wx = wx_slots + static_cast<int64_t>(sl) * 3 * N;
    uint16_t h0, l0, h1, l1, h2, l2;
    F::split(wx[n], h0, l0);
    F::split(wx[N + n], h1, l1);
    F::split(wx[2 * N + n], h2, l2);
    constexpr uint16_t z = F::kZero;
    __align__(16) uint16_t v[16] = {z, z, h0, l0, h0, h1, l1, h1, h2, l2, h2, z, z, z, z, z};
    uint8_t* base = ring + blob * BR * 32;
    *reinterpret_cast<uint4*>(base + ext_offset(rr, 0)) = *reinterpret_cast<const uint4*>(&v[0]);
    *reinterpret_cast<uint4*>(base + ext_offset(rr, 8)) = *reinterpret_cast<const uint4*>(&v[8]);
}

cudaError_t launch_ext_ring_init(uint8_t* ring, int64_t ctas, int n_mb, int N, const float* wx_slots, int f16,
                                 cudaStream_t st) {
    constexpr int xr = PairCfg<512>::XR;
    const int64_t n_blobs = ctas * xr * n_mb * 2;
    const int64_t rows = n_blobs * (N / 4);
    const unsigned grid = static_cast<unsigned>((rows + 255) / 256);
    if (f16)
        ext_ring_init_kernel<FmtF16><<<grid, 256, 0, st>>>(ring, n_blobs, n_mb, N, wx_slots, xr);
    else
        ext_ring_init_kernel<FmtBf16><<<grid, 256, 0, st>>>(ring, n_blobs, n_mb, N, wx_slots, xr);
    return cudaGetLastError();
}

// ------------------------------------------------------------- K0 (bf16) -----
// Per motion m and concat slot s: b_m = b + Wq . zq (fp32, q0 then q1), then the
// extension rows (b_hi, b_lo, W_x hi/lo splits) in the no-swizzle K=16 layout,
// cut into (n-half, CTA-half) blobs of N/4 rows.  Also resets keys/counters.
struct QNormX {
    float shift[kMaxIn], scale[kMaxIn];
};

template <class F>
__global__ void motion_ext_kernel(const float* __restrict__ q01, int dof, int N, int n_mb,
                                  const float* __restrict__ wq, const float* __restrict__ base_bias,
                                  const float* __restrict__ wx_slots, uint8_t* __restrict__ ext, const QNormX qn,
                                  unsigned long long* keys, unsigned int* counters, int64_t n_keys, int pp_layout,
                                  unsigned int* sched) {
    pdl_launch_dependents();  // the fused kernel may start its prologue now (it pdl_wait()s for our writes)
    const int64_t m = blockIdx.x;
    const int slot = blockIdx.y;
    if (sched && m == 0 && slot == 0 && threadIdx.x == 0) *sched = 0u;  // the fused kernel's tile counter
    if (keys && slot == 0 && threadIdx.x == 0 && m < n_keys) {
        keys[m] = ~0ull;
        counters[m] = 0u;
    }
    if (slot >= n_mb || ext == nullptr) return;  // no ext: the fused kernel builds the rows itself
    __shared__ float zq[kMaxIn];
    const int nq = 2 * dof;
    if (threadIdx.x < nq) {
        const float q = q01[m * nq + threadIdx.x];
        zq[threadIdx.x] = __fmul_rn(__fsub_rn(q, qn.shift[threadIdx.x]), qn.scale[threadIdx.x]);
    }
    __syncthreads();
    const float* w = wq + static_cast<int64_t>(slot) * nq * N;
    const float* wx = wx_slots + static_cast<int64_t>(slot) * 3 * N;
    const int NH = N / 2, BR = N / 4;
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
        float acc = base_bias[slot * N + n];
        for (int k = 0; k < nq; ++k) acc = __fmaf_rn(zq[k], w[k * N + n], acc);
        uint16_t bh, bl, h0, l0, h1, l1, h2, l2;
        F::split(acc, bh, bl);
        F::split(wx[n], h0, l0);
        F::split(wx[N + n], h1, l1);
        F::split(wx[2 * N + n], h2, l2);
        constexpr uint16_t z = F::kZero;
        __align__(16) uint16_t v[16] = {bh, bl, h0, l0, h0, h1, l1, h1, h2, l2, h2, z, z, z, z, z};
        uint8_t* base;
        int rr;
        if (pp_layout) {  // width-256 ping-pong kernel: blobs [r] of N/2 rows
            const int r = n / NH;
            rr = n % NH;
            base = ext + ((m * n_mb + slot) * 2 + r) * NH * 32;
        } else {          // pair kernel: blobs [n-half][r] of N/4 rows
            const int nh = n / NH, wi = n % NH, r = wi / BR;
            rr = wi % BR;
            base = ext + (((m * n_mb + slot) * 2 + nh) * 2 + r) * BR * 32;
        }
        *reinterpret_cast<uint4*>(base + ext_offset(rr, 0)) = *reinterpret_cast<const uint4*>(&v[0]);
        *reinterpret_cast<uint4*>(base + ext_offset(rr, 8)) = *reinterpret_cast<const uint4*>(&v[8]);
    }
}

}  // namespace svn

namespace svn {

cudaError_t launch_motion_ext(const FusedArgs& a, const float* wq, const float* mb_base_bias, const float* wx_slots,
                              uint8_t* ext, unsigned long long* keys_init, unsigned int* counters_init,
                              int64_t n_keys, unsigned int* sched_reset, cudaStream_t st) {
    if (a.M <= 0) return cudaSuccess;
    QNormX qn;
    for (int k = 0; k < 2 * a.dof && k < kMaxIn; ++k) {
        qn.shift[k] = a.shift[3 + k];
        qn.scale[k] = a.scale[3 + k];
    }
    dim3 grid(static_cast<unsigned>(a.M), (a.n_mb > 0 && ext) ? a.n_mb : 1);
    if (a.f16)
        motion_ext_kernel<FmtF16><<<grid, ext ? 256 : 32, 0, st>>>(a.q01, a.dof, a.N, a.n_mb, wq, mb_base_bias, wx_slots,
                                                                  ext, qn, keys_init, counters_init, n_keys,
                                                                  a.N == 256 ? 1 : 0, sched_reset);
    else
        motion_ext_kernel<FmtBf16><<<grid, ext ? 256 : 32, 0, st>>>(a.q01, a.dof, a.N, a.n_mb, wq, mb_base_bias, wx_slots,
                                                                   ext, qn, keys_init, counters_init, n_keys,
                                                                   a.N == 256 ? 1 : 0, sched_reset);
    return cudaGetLastError();
}

}  // namespace svn
