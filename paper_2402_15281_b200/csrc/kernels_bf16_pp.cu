// kernels_bf16_pp.cu — K1 (bf16) for width 256: two tiles ping-ponging on a CTA pair.
//
// Same math and operand formats as kernels_bf16_pair.cu (K=16 extension slab for bias and
// x-part, ReLU fused into the bf16 pack, fp32 output dot, packed-key min), but at width 256
// a whole layer fits one MMA chain (M=256 per pair, N=256, K=16) and TMEM holds two
// 256-column accumulators.  So each CTA pair keeps two tiles in flight (slots 0/1, each
// with its own activation tile and TMEM accumulator): the tensor core runs layer l of one
// slot while the epilogue warps drain the other slot's layer, and every weight slab is
// fetched once and used by both slots.
//
// Per CTA (width 256): A[2] 2 x 64 KiB, A-ext[2] 2 x 4 KiB, weight ring 4 x 16 KiB (one
// 64-wide K slab of this CTA's 128 B-rows each), extension ring 2 x 4 KiB.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "fused.cuh"
#include "ptx.cuh"

namespace svn {

namespace pp {

constexpr int N = 256;
constexpr int BR = N / 2;                  // B rows per CTA (M=256 x N=256 MMA: CTA r holds rows r*128..)
constexpr int KSL = N / 64;                // K slabs per layer
constexpr uint32_t SLAB_B = BR * 128;      // 16 KiB
constexpr uint32_t XCHUNK = BR * 32;       // 4 KiB
constexpr int WSTAGES = 4;
// One-round timeline of CTA 0 into FusedArgs::prof (scripts/pp_timeline.py); costs ~2.5%, so
// compiled in only with -DSVN_PP_TIMELINE.
#ifdef SVN_PP_TIMELINE
constexpr bool kTimeline = true;
#else
constexpr bool kTimeline = false;
#endif
constexpr int XSTAGES = 2;
constexpr int EPI_WARPS = 8;
constexpr int OUT_WARP = 2 + EPI_WARPS;    // first output warp: keys / per-point outputs / next tile's A extension
constexpr int OUT_WARPS = 2;              // one per slot
constexpr int THREADS = 64 + EPI_WARPS * 32 + OUT_WARPS * 32;
// Rows per CTA: 128 (M=256 MMAs, the throughput form) or 64 for launches with fewer 256-row
// tiles than CTA pairs (M=128 MMAs: each CTA's 64 x 256 accumulator in TMEM's "2x2" layout —
// lanes 0-63 hold columns 0-127, lanes 64-127 columns 128-255 — so twice the tiles, each
// through the network in ~0.6x the time).  The B side (weights, extension rows) is the same.
template <int TM_>
struct Cfg {
    static constexpr int TM = TM_;
    static constexpr uint32_t A_SLAB = TM * 128;
    static constexpr uint32_t A_BYTES = TM * N * 2;
    static constexpr uint32_t AX_BYTES = TM * 32;
    static constexpr int COLS = TM == 128 ? N / 2 : N / 4;  // columns per epilogue thread
    static constexpr int PARTS = TM == 128 ? 2 : 4;         // partial output dots per row
    static constexpr int RQ = TM / 32;                      // 32-row groups per CTA (output warps)
    static constexpr uint32_t OFF_AX = 2 * A_BYTES;
    static constexpr uint32_t OFF_W = OFF_AX + 2 * AX_BYTES;
    static constexpr uint32_t OFF_X = OFF_W + WSTAGES * SLAB_B;
    static constexpr uint32_t OFF_WO = OFF_X + XSTAGES * XCHUNK;
    static constexpr uint32_t OFF_DOT = OFF_WO + N * 4;
    static constexpr uint32_t OFF_BAR = OFF_DOT + 2 * PARTS * TM * 4;
    static constexpr uint32_t SMEM = OFF_BAR + 256;
    static_assert(SMEM <= 232448, "shared memory budget");
};

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

// 32 columns of one row: activation (+ Fig. 2 affine/residual) then bf16 store or output dot
// (accumulated in four partial sums so the 128-column dot is not one dependent FMA chain).
template <int TM, class F>
__device__ __forceinline__ void epi32(const LayerDev& ld, int l, bool last, float* v, int c0, uint32_t row,
                                      uint8_t* A, const float* wo_s, float4& dot) {
    // fp16 operands: a value beyond the fp16 range is stored as an infinity and makes every
    // accumulator of its row inf or NaN in the next layer; a hit poisons the row's output dot
    // (kernels_bf16_pair.cu: pair_epi32)
    if (F::kHalf && (!(fabsf(v[0]) <= 3.0e38f) || !(fabsf(v[21]) <= 3.0e38f))) dot.x = -INFINITY;
    const int fl = ld.flags;
    const bool act = fl & kAct, aff = fl & kAffine, res = (l > 0) && (fl & kResidual);
    if (!aff && !res && last) {
        // straight-line activation + output dot (no branches between the TMEM loads and the math)
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
    if (!aff && !res && !last) {
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
            dot.x = fmaf(w.x, v[i + 0], dot.x);  // four independent chains (column mod 4)
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

}  // namespace pp

#ifdef SVN_CTA_TIMES
// Per-CTA globaltimer stamps of the last launch (entry, after the prologue and pdl_wait,
// exit) and the SM it ran on, read back by svn_debug_cta_times (scripts/cta_times.py); instrumented builds only.
__device__ unsigned long long g_cta_times[4 * 1024];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

template <int TMR, class F>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(pp::THREADS, 1)
    fused_bf16_pp_kernel(const __grid_constant__ FusedArgs a) {
    using namespace pp;
    using C = Cfg<TMR>;
    constexpr int TM = C::TM, COLS = C::COLS, PARTS = C::PARTS, RQ = C::RQ;
    constexpr uint32_t A_SLAB = C::A_SLAB, A_BYTES = C::A_BYTES, AX_BYTES = C::AX_BYTES;
    constexpr uint32_t OFF_AX = C::OFF_AX, OFF_W = C::OFF_W, OFF_X = C::OFF_X, OFF_WO = C::OFF_WO,
                       OFF_DOT = C::OFF_DOT, OFF_BAR = C::OFF_BAR;
#ifdef SVN_CTA_TIMES
    if (threadIdx.x == 0 && blockIdx.x < 1024) g_cta_times[4 * blockIdx.x] = gtimer();
#endif
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* Abuf = smem;                      // [2][A_BYTES]
    uint8_t* AX = smem + OFF_AX;               // [2][AX_BYTES]
    uint8_t* wring = smem + OFF_W;
    uint8_t* xring = smem + OFF_X;
    float* wo_s = reinterpret_cast<float*>(smem + OFF_WO);
    float* dotbuf = reinterpret_cast<float*>(smem + OFF_DOT);  // [slot][ch][TM]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    uint64_t* wfull = bars;                     // [WSTAGES] leader
    uint64_t* wempty = wfull + WSTAGES;         // [WSTAGES] each CTA
    uint64_t* xfull = wempty + WSTAGES;         // [XSTAGES] leader
    uint64_t* xempty = xfull + XSTAGES;         // [XSTAGES] each CTA
    uint64_t* d_full = xempty + XSTAGES;        // [2] each CTA: slot s accumulator ready
    uint64_t* a_ready = d_full + 2;             // [2] leader: slot s drained + A_s written (16 warps)
    uint64_t* ax_ready = a_ready + 2;           // [2] leader: AX_s holds the slot's next tile (2 output warps)
    uint64_t* out_full = ax_ready + 2;          // [2] each CTA: dotbuf_s holds a finished tile (8 warps)
    uint64_t* out_empty = out_full + 2;         // [2] each CTA: output warp has read dotbuf_s
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(out_empty + 2);

    const int warp = threadIdx.x >> 5;
    const uint32_t lane = lane_id();
    const uint32_t rank = cluster_ctarank();
    const int L = a.L;
    const int64_t pair = blockIdx.x >> 1;
    const int64_t npairs = gridDim.x >> 1;
    const int64_t T = pair < a.n_tiles ? (a.n_tiles - 1 - pair) / npairs + 1 : 0;  // tiles of this pair
    const int64_t R = (T + 1) / 2;                                                   // rounds
    auto tile_of = [&](int64_t j, int s) { return pair + (2 * j + s) * npairs; };
    auto has = [&](int64_t j, int s) { return 2 * j + s < T; };

    if (threadIdx.x == 0) {
        if (smem_u32(smem) & 1023u) __trap();
        for (int s = 0; s < WSTAGES; ++s) {
            mbar_init(&wfull[s], 1);
            mbar_init(&wempty[s], 1);
        }
        for (int s = 0; s < XSTAGES; ++s) {
            mbar_init(&xfull[s], 1);
            mbar_init(&xempty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&d_full[s], 1);
            mbar_init(&a_ready[s], 2 * EPI_WARPS);
            mbar_init(&ax_ready[s], 2);
            mbar_init(&out_full[s], EPI_WARPS);
            mbar_init(&out_empty[s], 1);
        }
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < N; i += blockDim.x) wo_s[i] = a.wo[i];
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&a.tmap_w);
        prefetch_tmap(&a.tmap_xm);
        prefetch_tmap(&a.tmap_xq);
    }
    if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();  // K0 (keys, counters, tile queue, extension rows) has completed
#ifdef SVN_CTA_TIMES
    if (threadIdx.x == 0 && blockIdx.x < 1024) g_cta_times[4 * blockIdx.x + 1] = gtimer();
#endif

    if (warp == 0) {
        // ------------------------------------------------------------------ producer --
        if (lane == 0) {
            const uint64_t pol = policy_evict_last();
            const uint32_t wfull0 = mapa_shared(smem_u32(wfull), 0), xfull0 = mapa_shared(smem_u32(xfull), 0);
            int ws = 0, xs = 0;
            uint32_t wph = 0, xph = 0;
            for (int64_t j = 0; j < R; ++j) {
                int64_t wrow = 0;  // slab index in the stream
                for (int l = 0; l < L; ++l) {
                    const LayerDev& ld = a.layer[l];
                    if (ld.ext) {
                        for (int s = 0; s < 2; ++s) {
                            if (!has(j, s)) continue;
                            int32_t motion, nrows;
                            int64_t pbase, obase;
                            tile_decode(a, tile_of(j, s), 2 * TM, motion, pbase, obase, nrows);
                            mbar_wait(&xempty[xs], xph ^ 1u);
                            if (rank == 0) mbar_arrive_expect_tx_local(&xfull[xs], 2 * XCHUNK);
                            uint8_t* dst = xring + xs * XCHUNK;
                            if (ld.ext == 2) {
                                const int64_t blob = (static_cast<int64_t>(motion) * a.n_mb + ld.mb_slot) * 2 + rank;
                                tma_load_2d_pair(dst, &a.tmap_xq, 0, static_cast<int32_t>(blob * BR), xfull0 + xs * 8u, pol);
                            } else {
                                tma_load_2d_pair(dst, &a.tmap_xm, 0, static_cast<int32_t>(ld.ext_row + rank * BR),
                                                 xfull0 + xs * 8u, pol);
                            }
                            if (++xs == XSTAGES) xs = 0, xph ^= 1u;
                        }
                    }
                    if (l > 0) {
                        for (int ks = 0; ks < KSL; ++ks, ++wrow) {
                            mbar_wait(&wempty[ws], wph ^ 1u);
                            if (rank == 0) mbar_arrive_expect_tx_local(&wfull[ws], 2 * SLAB_B);
                            tma_load_2d_pair(wring + ws * SLAB_B, &a.tmap_w, 0,
                                             static_cast<int32_t>((wrow * 2 + rank) * BR), wfull0 + ws * 8u, pol);
                            if (++ws == WSTAGES) ws = 0, wph ^= 1u;
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------------- MMA issuer --
        if (lane == 0 && rank == 0) {
            constexpr uint32_t idesc = F::idesc(2 * TM, N);
            const uint32_t a_base = smem_u32(Abuf), ax_base = smem_u32(AX), w_base = smem_u32(wring);
            const uint32_t x_base = smem_u32(xring);
            int ws = 0, xs = 0;
            uint32_t wph = 0, xph = 0;
            uint32_t ar_ph[2] = {0u, 0u}, ax_ph[2] = {0u, 0u};
            unsigned long long pw_a = 0, pw_f = 0, pw_x = 0;
            const unsigned long long p_start = prof_clock();
            for (int64_t j = 0; j < R; ++j) {
                for (int l = 0; l < L; ++l) {
                    const LayerDev& ld = a.layer[l];
                    const int ws_layer = ws;  // ring slot of this layer's slab 0
                    const uint32_t wph_layer = wph;
                    const int nslots = has(j, 1) ? 2 : 1;
                    for (int s = 0; s < nslots; ++s) {
                        const unsigned long long c0 = prof_clock();
                        const bool tl = kTimeline && a.prof && blockIdx.x == 0 && j == R / 2 && l < 4;  // timeline sample
                        if (tl) a.prof[kProfTimeline + (l * 2 + s) * 3] = c0;
                        mbar_wait(&a_ready[s], ar_ph[s]);  // D_s drained, A_s written
                        if (l == 0) {
                            mbar_wait(&ax_ready[s], ax_ph[s]);  // AX_s holds this tile's points
                            ax_ph[s] ^= 1u;
                        }
                        pw_a += prof_clock() - c0;
                        if (tl) a.prof[kProfTimeline + (l * 2 + s) * 3 + 1] = prof_clock();
                        ar_ph[s] ^= 1u;
                        tc_fence_after();
                        const uint32_t d_addr = tmem + static_cast<uint32_t>(s * N);
                        bool acc = false;
                        if (ld.ext) {
                            const unsigned long long c1 = prof_clock();
                            mbar_wait(&xfull[xs], xph);
                            pw_x += prof_clock() - c1;
                            tc_fence_after();
                            mma_bf16_pair(d_addr, noswz_desc(ax_base + s * AX_BYTES, 128, 256),
                                          noswz_desc(x_base + xs * XCHUNK, 128, 256), idesc, 0u);
                            mma_commit_pair(&xempty[xs], 3);
                            if (++xs == XSTAGES) xs = 0, xph ^= 1u;
                            acc = true;
                        }
                        if (l > 0) {
                            int st = ws_layer;
                            uint32_t ph = wph_layer;
                            for (int ks = 0; ks < KSL; ++ks) {
                                if (s == 0) {
                                    const unsigned long long c2 = prof_clock();
                                    mbar_wait(&wfull[st], ph);
                                    pw_f += prof_clock() - c2;
                                    tc_fence_after();
                                }
                                const uint32_t a_slab = a_base + s * A_BYTES + ks * A_SLAB;
                                const uint32_t b_slab = w_base + st * SLAB_B;
#pragma unroll
                                for (int kk = 0; kk < 4; ++kk)
                                    mma_bf16_pair(d_addr, sw128_desc(a_slab + kk * 32), sw128_desc(b_slab + kk * 32),
                                                  idesc, (acc || ks || kk) ? 1u : 0u);
                                if (s == nslots - 1) mma_commit_pair(&wempty[st], 3);  // last user frees the slab
                                if (++st == WSTAGES) st = 0, ph ^= 1u;
                            }
                        }
                        mma_commit_pair(&d_full[s], 3);
                        if (tl) a.prof[kProfTimeline + (l * 2 + s) * 3 + 2] = prof_clock();
                    }
                    if (l > 0)
                        for (int ks = 0; ks < KSL; ++ks)
                            if (++ws == WSTAGES) ws = 0, wph ^= 1u;
                }
            }
            if (a.prof) {
                atomicAdd(a.prof + kProfMmaWaitA, pw_a);
                atomicAdd(a.prof + kProfMmaWaitFull, pw_f);
                atomicAdd(a.prof + kProfMmaWaitAx, pw_x);
                atomicAdd(a.prof + kProfMmaTotal, prof_clock() - p_start);
            }
        }
    } else if (warp < OUT_WARP) {
        // ------------------------------------------------------------------ epilogue --
        const int e = warp - 2;
        const uint32_t quad = static_cast<uint32_t>(warp & 3);
        const int ch = e >> 2;
        // TM=128: lane quadrant = 32 rows, all columns; TM=64 ("2x2"): quadrants 0/1 = rows
        // 0-31/32-63 of columns 0-127, 2/3 = the same rows of columns 128-255
        const uint32_t row = (TM == 128 ? quad : (quad & 1u)) * 32 + lane;
        const int cq = TM == 128 ? 0 : static_cast<int>(quad >> 1) * 128;
        const int part = (TM == 128 ? 0 : static_cast<int>(quad >> 1) * 2) + ch;
        const uint32_t t_lane = (quad * 32u) << 16;
        const uint32_t a_ready0 = mapa_shared(smem_u32(a_ready), 0);
        uint32_t dp[2] = {0u, 0u}, oe_ph[2] = {0u, 0u};
        // initial "slot free" arrivals (the output warp separately signals AX_s)
        for (int s = 0; s < 2; ++s) {
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(a_ready0 + s * 8u);
        }
        float4 dot[2] = {make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};
        unsigned long long pe_d = 0, pe_w = 0, pe_a = 0, pe_o = 0;
        for (int64_t j = 0; j < R; ++j) {
            const int nslots = has(j, 1) ? 2 : 1;
            for (int l = 0; l < L; ++l) {
                const LayerDev& ld = a.layer[l];
                const bool last = (l == L - 1);
                for (int s = 0; s < nslots; ++s) {
                    uint8_t* A = Abuf + s * A_BYTES;
                    const unsigned long long c0 = prof_clock();
                    mbar_wait(&d_full[s], dp[s]);
                    const unsigned long long c1 = prof_clock();
                    pe_d += c1 - c0;
                    const bool tl = kTimeline && a.prof && blockIdx.x == 0 && e == 0 && lane == 0 && j == R / 2 && l < 4;
                    if (tl) a.prof[kProfTimeline + 24 + (l * 2 + s) * 3] = c1;
                    dp[s] ^= 1u;
                    tc_fence_after();
                    const int c0c = ch * COLS;
                    constexpr int NCH = COLS / 32;
                    const uint32_t tbase = tmem + t_lane + static_cast<uint32_t>(s * N);
                    {
                        uint32_t ra[32], rb[32];
                        tmem_ld32_async(tbase + static_cast<uint32_t>(c0c), ra);
                        tmem_wait_tied(ra);
#pragma unroll
                        for (int q = 0; q < NCH; ++q) {
                            uint32_t(&cur)[32] = (q & 1) ? rb : ra;
                            uint32_t(&nxt)[32] = (q & 1) ? ra : rb;
                            if (q + 1 < NCH) tmem_ld32_async(tbase + static_cast<uint32_t>(c0c + 32 * (q + 1)), nxt);
                            epi32<TM, F>(ld, l, last, reinterpret_cast<float*>(cur), cq + c0c + 32 * q, row, A, wo_s, dot[s]);
                            if (q + 1 < NCH) tmem_wait_tied(nxt);
                        }
                    }
                    const unsigned long long c2 = prof_clock();
                    pe_w += c2 - c1;
                    if (tl) a.prof[kProfTimeline + 24 + (l * 2 + s) * 3 + 1] = c2;
                    tc_fence_before();
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_remote(a_ready0 + s * 8u);
                    const unsigned long long c3 = prof_clock();
                    pe_a += c3 - c2;
                    if (tl) a.prof[kProfTimeline + 24 + (l * 2 + s) * 3 + 2] = c3;
                    if (last) {
                        // hand this row's partial dot to the output warp (dotbuf_s is read a round later)
                        if (j > 0) {
                            mbar_wait(&out_empty[s], oe_ph[s]);
                            oe_ph[s] ^= 1u;
                        }
                        dotbuf[(s * PARTS + part) * TM + row] = (dot[s].x + dot[s].y) + (dot[s].z + dot[s].w);
                        dot[s] = make_float4(0.f, 0.f, 0.f, 0.f);
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&out_full[s]);
                    }
                    pe_o += prof_clock() - c3;
                }
            }
        }
        if (a.prof && e == 0 && lane == 0 && rank == 0) {
            atomicAdd(a.prof + kProfEpiWaitD, pe_d);
            atomicAdd(a.prof + kProfEpiWork, pe_w);
            atomicAdd(a.prof + kProfEpiArrive, pe_a);
            atomicAdd(a.prof + kProfEpiOut, pe_o);
        }
    } else {
        // ---------------------------------------------------------------- output warps --
        // One warp per slot.  Per finished tile of its slot: delta = dot + bo for this CTA's
        // 128 rows, per-point stores, one packed-key atomicMin, the per-motion completion
        // counter; and the A extension (bias / x columns) of the slot's next tile.  The point
        // loads run a whole round ahead (tile j+2 of the slot is loaded when tile j+1's AX is
        // written), and the two slots never queue behind each other's atomics, so AX_s is
        // ready as soon as the slot's last epilogue has finished.
        const int s = warp - OUT_WARP;
        const uint32_t ax_ready0 = mapa_shared(smem_u32(ax_ready), 0);
        uint32_t of_ph = 0u;
        float px[RQ][3];
        auto load_points = [&](int64_t t) {
            int32_t motion, nrows;
            int64_t pbase, obase;
            tile_decode(a, t, 2 * TM, motion, pbase, obase, nrows);
#pragma unroll
            for (int k = 0; k < RQ; ++k) {
                const int32_t r = static_cast<int32_t>(rank * TM + k * 32 + lane);
                const float* xp = a.points + (pbase + (r < nrows ? r : 0)) * a.point_stride;
                px[k][0] = xp[0];
                px[k][1] = xp[1];
                px[k][2] = xp[2];
            }
        };
        auto store_ax = [&]() {
#pragma unroll
            for (int k = 0; k < RQ; ++k)
                write_ax<F>(AX + s * AX_BYTES, static_cast<uint32_t>(k * 32) + lane, (px[k][0] - a.shift[0]) * a.scale[0],
                         (px[k][1] - a.shift[1]) * a.scale[1], (px[k][2] - a.shift[2]) * a.scale[2]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(ax_ready0 + s * 8u);
        };
        unsigned long long pe_x = 0;
        if (has(0, s)) {
            load_points(tile_of(0, s));
            store_ax();
            if (has(1, s)) load_points(tile_of(1, s));
        }
        for (int64_t j = 0; j < R && has(j, s); ++j) {
            int32_t motion, nrows;
            int64_t pbase, obase;
            tile_decode(a, tile_of(j, s), 2 * TM, motion, pbase, obase, nrows);
            mbar_wait(&out_full[s], of_ph);
            of_ph ^= 1u;
            const unsigned long long c0 = prof_clock();
            // every MMA of tile (j, s) has completed, so AX_s is free for the next tile
            if (has(j + 1, s)) {
                store_ax();
                if (has(j + 2, s)) load_points(tile_of(j + 2, s));
            }
            float delta[RQ];
#pragma unroll
            for (int k = 0; k < RQ; ++k) {
                const int r = k * 32 + static_cast<int>(lane);
                const float* d = dotbuf + (s * PARTS) * TM + r;
                delta[k] = (PARTS == 2 ? d[0] + d[TM] : (d[0] + d[TM]) + (d[2 * TM] + d[3 * TM])) + a.bo;
                // fp16 operands: a row that left the fp16 range arrives as inf / NaN and is reported as
                // -inf (class "not free") instead of dropping out of the min (kernels_bf16_pair.cu)
                if (F::kHalf && !(fabsf(delta[k]) <= 3.0e38f)) delta[k] = -INFINITY;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&out_empty[s]);
            unsigned long long key = ~0ull;
#pragma unroll
            for (int k = 0; k < RQ; ++k) {
                const int32_t rr = static_cast<int32_t>(rank * TM + k * 32 + lane);
                if (rr < nrows) {
                    if (a.per_point) a.per_point[obase + rr] = delta[k];
                    const unsigned long long kk = row_key(delta[k], a.index_offset + pbase + rr);
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
            pe_x += prof_clock() - c0;
        }
        if (a.prof && lane == 0 && rank == 0 && s == 0) atomicAdd(a.prof + kProfEpiAx, pe_x);
    }

    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    if (warp == 1) tmem_dealloc_pair(tmem, 512);
#ifdef SVN_CTA_TIMES
    if (threadIdx.x == 0 && blockIdx.x < 1024) {
        unsigned int smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_cta_times[4 * blockIdx.x + 2] = gtimer();
        g_cta_times[4 * blockIdx.x + 3] = smid;
    }
#endif
}

#ifdef SVN_CTA_TIMES
extern "C" __attribute__((visibility("default"))) int svn_debug_cta_times(unsigned long long* out, int n) {
    return static_cast<int>(cudaMemcpyFromSymbol(out, g_cta_times, sizeof(unsigned long long) * 4 * n));
}
#endif

template <int TM, class F>
static cudaError_t launch_pp_n(const FusedArgs& a, int num_sms, cudaStream_t st) {
    static SmemOptIn opt;
    constexpr uint32_t smem = pp::Cfg<TM>::SMEM;
    cudaError_t e = opt.ensure(reinterpret_cast<const void*>(fused_bf16_pp_kernel<TM, F>), (int)smem);
    if (e != cudaSuccess) return e;
    int64_t pairs = num_sms / 2;
    // two tiles in flight per pair, unless there are too few tiles to fill the SMs that way:
    // then one tile per pair (latency-bound queries finish ~2x sooner)
    const int64_t need = a.n_tiles <= pairs ? a.n_tiles : (a.n_tiles + 1) / 2;
    if (need < pairs) pairs = need;
    if (pairs < 1) return cudaSuccess;
    const cudaError_t le = launch_fused_pdl(fused_bf16_pp_kernel<TM, F>, static_cast<unsigned>(2 * pairs), pp::THREADS,
                                            smem, st, a);
    return le != cudaSuccess ? le : cudaGetLastError();
}

cudaError_t launch_fused_bf16_pp(const FusedArgs& a, int num_sms, cudaStream_t st) {
    // 128-row pair tiles for launches with fewer 256-row tiles than pairs (abi tile_rows_for)
    if (a.f16) return a.tile_rows == 128 ? launch_pp_n<64, FmtF16>(a, num_sms, st) : launch_pp_n<128, FmtF16>(a, num_sms, st);
    return a.tile_rows == 128 ? launch_pp_n<64, FmtBf16>(a, num_sms, st) : launch_pp_n<128, FmtBf16>(a, num_sms, st);
}

}  // namespace svn
