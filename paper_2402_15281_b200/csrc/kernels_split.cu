// kernels_split.cu — K1 (fp32-accurate) on tcgen05 for width 256 and 512: split-fp16 products.
//
// The fp32 path's 1e-5 per-point bar (BASELINE.json north_star) without SIMT FFMA: every
// operand x is split into fp16 hi = fp16(x) and scaled lo' = fp16((x - hi) * 2^11) (22
// significant bits), and each width x width product runs as three kind::f16 MMAs into two
// fp32 TMEM accumulators:
//     main += A_hi . B_hi          corr += A_hi . B_lo' + A_lo' . B_hi
//     D = main + corr * 2^-11      (the lo' . lo' term, ~2^-22 relative, is dropped)
// Measured (scripts/microbench_split.cu): 2.7e-6 max error vs fp64 on a 128x256x256 product
// with |D| ~ 5, against 2.3e-6 for a sequential fp32 FMA chain.  Bias, the per-motion q-fold
// and the x-part ride in a K=16 extension slab split the same way.  The tensor core truncates
// its fp32 accumulator once per instruction; the epilogue adds the expected loss back
// (combine() below).
//
// Structure = the CTA-pair kernel (kernels_bf16_pair.cu) with the layer output treated as two
// n-halves, each owning a main and a corr accumulator: 2 x (128 + 128) = all 512 TMEM columns.
// A layer runs as quarter steps (n-half, k-half) (0,0) (1,0) (0,1) (1,1); the epilogue of
// output half 0 overlaps step (1,1).  The activation tile is held as two fp16 planes (hi, lo'),
// 2 x 64 KiB per CTA at either width:
//   width 256: 128 rows per CTA, M=256 pair MMAs with N=128 (one n-half), each accumulator
//              128 lanes x 128 columns;
//   width 512: 64 rows per CTA, M=128 pair MMAs with N=256 — the accumulator of a CTA's 64
//              rows x 256 columns sits in TMEM's "2x2" layout (rows in lanes 0-63 for
//              columns 0-127 of the n-half, in lanes 64-127 for columns 128-255), again 128
//              TMEM columns, so the TMEM plan is the same; a weight slab (one plane of 128
//              B rows x 64 K per CTA) is one 16 KiB stage, its hi and lo' planes two stages.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "fused.cuh"
#include "ptx.cuh"

namespace svn {

namespace sp {

template <int N_>
struct Cfg {
    static constexpr int N = N_;                        // layer width
    static constexpr int TM = N == 256 ? 128 : 64;      // rows per CTA (pair tile = 2 TM rows)
    static constexpr int NHO = N / 2;                   // output columns per n-half (MMA N)
    static constexpr int BRH = NHO / 2;                 // B rows per CTA per n-half (cta_group::2 split of N)
    static constexpr int KSL = (N / 2) / 64;            // 64-wide K slabs per k-half
    static constexpr uint32_t A_SLAB = TM * 128;        // one 64-K slab of an A plane
    static constexpr uint32_t A_PLANE = TM * N * 2;     // 64 KiB per fp16 plane
    static constexpr uint32_t AX_BYTES = TM * 32;
    static constexpr uint32_t STAGE = 16384;            // one TMA stage
    static constexpr uint32_t PLANE_B = BRH * 128;      // one plane of one weight slab for this CTA
    static constexpr int SPS = 2 * PLANE_B / STAGE;     // stages per weight slab: 1 ([hi|lo']) or 2 (hi, lo')
    static constexpr uint32_t XHALF = BRH * 32;         // extension rows (main or corr) for this CTA
    static constexpr int STAGES = 5;
    static constexpr int EPI_WARPS = 8;
    static constexpr int OUT_WARP = 2 + EPI_WARPS;      // keys / per-point outputs / A extensions of later tiles
    static constexpr int THREADS = 64 + EPI_WARPS * 32 + 32;
    static constexpr int COLS = 64;                     // columns per epilogue thread per n-half
    static constexpr int PARTS = N / 128;               // partial output dots per row (epilogue threads)
    static constexpr int RQ = TM / 32;                  // 32-row groups per CTA (output warp)
    static constexpr uint32_t OFF_AHI = 0;
    static constexpr uint32_t OFF_ALO = A_PLANE;
    static constexpr uint32_t OFF_AX = 2 * A_PLANE;
    static constexpr uint32_t OFF_STAGE = OFF_AX + 2 * AX_BYTES;
    static constexpr uint32_t OFF_WO = OFF_STAGE + STAGES * STAGE;
    static constexpr uint32_t OFF_DOT = OFF_WO + N * 4;
    static constexpr uint32_t OFF_BAR = OFF_DOT + 2 * PARTS * TM * 4;
    static constexpr uint32_t SMEM = OFF_BAR + 256;
    static_assert(SMEM <= 232448, "shared memory budget");
    static_assert(SPS == 1 || SPS == 2, "a weight slab is one or two stages");
    static_assert(2 * XHALF <= STAGE, "extension slab fits one stage");
    static_assert(OFF_STAGE % 1024 == 0, "SW128 stages need 1 KiB alignment");
};

constexpr float LO_SCALE = 2048.0f;
constexpr float LO_INV = 1.0f / 2048.0f;

// kind::f16 instruction descriptor with fp16 A/B (format 0) and fp32 D.
__host__ __device__ constexpr uint32_t idesc_f16(int m, int n) {
    return (1u << 4) | (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}

// |x| >= 65520 rounds to an fp16 infinity: such an activation cannot be held in the
// (hi, lo') planes.  The row is then reported as delta = -inf: its motion's min is -inf and
// its class "not free", i.e. it is handed to the exact checker (the safe side of
// collision.cpp:68) instead of silently dropping out of the min as a NaN.  The epilogue keeps
// the running max of |hi| per row (packed half2) and checks it once per tile.

__device__ __forceinline__ void split(float x, __half& hi, __half& lo) {
    hi = __float2half_rn(x);
    lo = __float2half_rn((x - __half2float(hi)) * LO_SCALE);
}

__device__ __forceinline__ uint32_t pack_h2(__half lo_elem, __half hi_elem) {
    return static_cast<uint32_t>(__half_as_ushort(lo_elem)) | (static_cast<uint32_t>(__half_as_ushort(hi_elem)) << 16);
}

// A extension row: (1, z0h, z1h, z2h, z0l', z1l', z2l', 0...) fp16.
__device__ __forceinline__ void write_ax(uint8_t* ax, uint32_t row, float z0, float z1, float z2) {
    __half h0, l0, h1, l1, h2, l2;
    split(z0, h0, l0);
    split(z1, h1, l1);
    split(z2, h2, l2);
    const __half one = __float2half_rn(1.0f), zero = __float2half_rn(0.0f);
    __align__(16) __half v[16] = {one, h0, h1, h2, l0, l1, l2, zero, zero, zero, zero, zero, zero, zero, zero, zero};
    *reinterpret_cast<uint4*>(ax + ext_offset(row, 0)) = *reinterpret_cast<const uint4*>(&v[0]);
    *reinterpret_cast<uint4*>(ax + ext_offset(row, 8)) = *reinterpret_cast<const uint4*>(&v[8]);
}

// main + corr / 2048, with main's expected truncation loss added back: the tensor core's
// fp32 accumulator drops the bits below its 24-bit significand at every MMA instruction
// (toward zero), so after n instructions main sits on average ~c x n ulps below |exact|.  The
// loss is taken proportional to |main| (one ulp is between 2^-24 and 2^-23 of |main|; c
// absorbs the mean): v = main x (1 + c n 2^-23) + corr x 2^-11, for two columns at once with
// the packed fp32 pair ops (two independent round-to-nearest results each) — one instruction
// per column, as many as the uncompensated fma(corr, 2^-11, main).
__device__ __forceinline__ void combine32(const uint32_t* m, const uint32_t* c, float kmul, float* v) {
    unsigned long long k2, s2;
    asm("mov.b64 %0, {%1, %1};" : "=l"(k2) : "f"(kmul));
    asm("mov.b64 %0, {%1, %1};" : "=l"(s2) : "f"(LO_INV));
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
        unsigned long long mm, cc, t;
        asm("mov.b64 %0, {%1, %2};" : "=l"(mm) : "r"(m[i]), "r"(m[i + 1]));
        asm("mov.b64 %0, {%1, %2};" : "=l"(cc) : "r"(c[i]), "r"(c[i + 1]));
        asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(cc), "l"(s2));
        asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(t) : "l"(mm), "l"(k2));
        asm("mov.b64 {%0, %1}, %2;" : "=f"(v[i]), "=f"(v[i + 1]) : "l"(t));
    }
}

// 32 output columns of one row: v (fp32, already main + corr/2048) -> act / affine /
// residual -> next layer's (hi, lo') planes, or the output dot on the last layer.
template <int TM>
__device__ __forceinline__ void epi32(const LayerDev& ld, int l, bool last, float* v, int c0, uint32_t row,
                                      uint8_t* Ahi, uint8_t* Alo, const float* wo_s, float4& dot, bool& ovf,
                                      __half2& hmax) {
    const int fl = ld.flags;
    const bool act = fl & kAct, aff = fl & kAffine, res = (l > 0) && (fl & kResidual);
#ifndef SVN_SPLIT_NO_NANCHECK  // A/B build without the non-finite input check
    if (l == 0 || (fl & kConcat)) {
#else
    if (false) {
#endif
        // the layer's K=16 extension carries z_x (and b_m) as fp16 splits: an input beyond the
        // fp16 range arrives as inf / NaN, which the ReLU below would turn into 0.  v * 0 is
        // NaN exactly for a non-finite v.
        unsigned long long nf = 0ull, z2 = 0ull;  // (0, 0) pairs; v * 0 + nf on packed fp32 pairs
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
            unsigned long long vv;
            asm("mov.b64 %0, {%1, %2};" : "=l"(vv) : "f"(v[i]), "f"(v[i + 1]));
            asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(nf) : "l"(vv), "l"(z2));
        }
        float n0, n1;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(n0), "=f"(n1) : "l"(nf));
        ovf |= (n0 != n0) || (n1 != n1);
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
    if (res) {  // residual stream = hi + lo'/2048 from the A planes (same addresses we overwrite)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t off = sw128_offset(row, c0 + 8 * u, TM);
            const uint4 h = *reinterpret_cast<const uint4*>(Ahi + off);
            const uint4 o = *reinterpret_cast<const uint4*>(Alo + off);
            const uint32_t hw[4] = {h.x, h.y, h.z, h.w}, ow[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const __half2 hh = *reinterpret_cast<const __half2*>(&hw[p]);
                const __half2 oo = *reinterpret_cast<const __half2*>(&ow[p]);
                v[8 * u + 2 * p] += fmaf(__low2float(oo), LO_INV, __low2float(hh));
                v[8 * u + 2 * p + 1] += fmaf(__high2float(oo), LO_INV, __high2float(hh));
            }
        }
    }
    if (last) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
            const float4 w = *reinterpret_cast<const float4*>(wo_s + c0 + i);
            dot.x = fmaf(w.x, v[i + 0], dot.x);  // four partial sums (column mod 4)
            dot.y = fmaf(w.y, v[i + 1], dot.y);
            dot.z = fmaf(w.z, v[i + 2], dot.z);
            dot.w = fmaf(w.w, v[i + 3], dot.w);
        }
        return;
    }
    unsigned long long s2;  // (2^11, 2^11) for the packed fp32 pair ops
    asm("mov.b64 %0, {%1, %1};" : "=l"(s2) : "f"(LO_SCALE));
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            // paired split: hi = f16x2(x0, x1); lo' = f16x2((x - hi) * 2^11), the difference and
            // the power-of-two scaling exact, on packed fp32 pairs
            const float x0 = v[8 * u + 2 * p], x1 = v[8 * u + 2 * p + 1];
            const __half2 h = __floats2half2_rn(x0, x1);
            // |hi| >= 65520 rounds to inf: the running max of |hi| tells the tile (checked once)
            hmax = __hmax2(hmax, __habs2(h));
            const float2 hf = __half22float2(h);
            unsigned long long xx, hh, d;
            asm("mov.b64 %0, {%1, %2};" : "=l"(xx) : "f"(x0), "f"(x1));
            asm("mov.b64 %0, {%1, %2};" : "=l"(hh) : "f"(hf.x), "f"(hf.y));
            asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(xx), "l"(hh));
            asm("mul.rn.f32x2 %0, %0, %1;" : "+l"(d) : "l"(s2));
            float d0, d1;
            asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(d));
            const __half2 lo = __floats2half2_rn(d0, d1);
            hw[p] = *reinterpret_cast<const uint32_t*>(&h);
            lw[p] = *reinterpret_cast<const uint32_t*>(&lo);
        }
        const uint32_t off = sw128_offset(row, c0 + 8 * u, TM);
        *reinterpret_cast<uint4*>(Ahi + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(Alo + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
}

}  // namespace sp

template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(sp::Cfg<N>::THREADS, 1)
    fused_split_kernel(const __grid_constant__ FusedArgs a) {
    using namespace sp;
    using C = Cfg<N>;
    constexpr int TM = C::TM, NHO = C::NHO, BRH = C::BRH, KSL = C::KSL, STAGES = C::STAGES, SPS = C::SPS;
    constexpr int EPI_WARPS = C::EPI_WARPS, OUT_WARP = C::OUT_WARP, COLS = C::COLS, PARTS = C::PARTS, RQ = C::RQ;
    constexpr uint32_t A_SLAB = C::A_SLAB, AX_BYTES = C::AX_BYTES, STAGE = C::STAGE, XHALF = C::XHALF;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* Ahi = smem + C::OFF_AHI;
    uint8_t* Alo = smem + C::OFF_ALO;
    uint8_t* AX = smem + C::OFF_AX;  // [2][AX_BYTES]
    uint8_t* stages = smem + C::OFF_STAGE;
    float* wo_s = reinterpret_cast<float*>(smem + C::OFF_WO);
    float* dotbuf = reinterpret_cast<float*>(smem + C::OFF_DOT);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
    uint64_t* full = bars;
    uint64_t* empty = full + STAGES;
    uint64_t* d_full = empty + STAGES;
    uint64_t* a_ready = d_full + 2;
    uint64_t* ax_full = a_ready + 2;    // [tile parity] leader: AX holds the tile's points (2 output warps)
    uint64_t* out_full = ax_full + 2;   // [tile parity] each CTA: dotbuf holds a finished tile (8 warps)
    uint64_t* out_empty = out_full + 2; // [tile parity] each CTA: output warp has read dotbuf
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(out_empty + 2);

    const int warp = threadIdx.x >> 5;
    const uint32_t lane = lane_id();
    const uint32_t rank = cluster_ctarank();
    const int L = a.L;
    const int64_t pair = blockIdx.x >> 1;
    const int64_t npairs = gridDim.x >> 1;

    if (threadIdx.x == 0) {
        if (smem_u32(smem) & 1023u) __trap();
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int j = 0; j < 2; ++j) {
            mbar_init(&d_full[j], 1);
            mbar_init(&a_ready[j], 2 * EPI_WARPS);
            mbar_init(&ax_full[j], 2);
            mbar_init(&out_full[j], EPI_WARPS);
            mbar_init(&out_empty[j], 1);
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

    if (warp == 0) {
        // ---------------------------------------------------------------- producer --
        if (lane == 0) {
            const uint64_t pol = policy_evict_last();
            const uint32_t full0 = mapa_shared(smem_u32(full), 0);
            int stage = 0;
            uint32_t phase = 0;
            auto slot = [&](uint32_t bytes_one_cta) {
                mbar_wait(&empty[stage], phase ^ 1u);
                if (rank == 0) mbar_arrive_expect_tx_local(&full[stage], 2 * bytes_one_cta);
            };
            auto advance = [&]() {
                if (++stage == STAGES) stage = 0, phase ^= 1u;
            };
            for (int64_t t = pair; t < a.n_tiles; t += npairs) {
                int32_t motion, nrows;
                int64_t pbase, obase;
                tile_decode(a, t, 2 * TM, motion, pbase, obase, nrows);
                int64_t wrow = 0;  // 128-byte row of the weight stream
                for (int l = 0; l < L; ++l) {
                    const LayerDev& ld = a.layer[l];
                    const int steps = l == 0 ? 2 : 4;
                    for (int step = 0; step < steps; ++step) {
                        const int nh = step & 1, kh = step >> 1;
                        if (kh == 0 && ld.ext) {
                            slot(2 * XHALF);
                            const uint32_t fb = full0 + stage * 8u;
                            uint8_t* dst = stages + stage * STAGE;
                            if (ld.ext == 2) {
                                const int64_t blob = ((static_cast<int64_t>(motion) * a.n_mb + ld.mb_slot) * 2 + nh) * 2 + rank;
                                tma_load_2d_pair(dst, &a.tmap_xq, 0, static_cast<int32_t>(blob * 2 * BRH), fb, pol);
                            } else {
                                const int64_t r0 = ld.ext_row + (nh * 2 + rank) * 2 * BRH;
                                tma_load_2d_pair(dst, &a.tmap_xm, 0, static_cast<int32_t>(r0), fb, pol);
                            }
                            advance();
                        }
                        if (l > 0) {
                            for (int ks = 0; ks < KSL; ++ks) {
                                // this CTA's [hi | lo'] rows of the slab: one 128-row box per stage
                                for (int sub = 0; sub < SPS; ++sub) {
                                    slot(STAGE);
                                    tma_load_2d_pair(stages + stage * STAGE, &a.tmap_w, 0,
                                                     static_cast<int32_t>(wrow + rank * 2 * BRH + sub * 128),
                                                     full0 + stage * 8u, pol);
                                    advance();
                                }
                                wrow += 4 * BRH;
                            }
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // -------------------------------------------------------------- MMA issuer --
        if (lane == 0 && rank == 0) {
            constexpr uint32_t idesc = idesc_f16(2 * TM, NHO);
            const uint32_t ahi = smem_u32(Ahi), alo = smem_u32(Alo), s_base = smem_u32(stages), ax_base = smem_u32(AX);
            int stage = 0;
            uint32_t phase = 0;
            uint32_t ar_ph[2] = {0u, 0u}, ax_ph[2] = {0u, 0u};
            unsigned long long pw_a = 0, pw_f = 0, pw_x = 0;  // SVN_KERNEL_PROF wait accounting
            const unsigned long long p_start = prof_clock();
            int64_t k = 0;
            for (int64_t t = pair; t < a.n_tiles; t += npairs, ++k) {
                const int b = static_cast<int>(k & 1);
                const unsigned long long cx = prof_clock();
                mbar_wait(&ax_full[b], ax_ph[b]);
                pw_x += prof_clock() - cx;
                ax_ph[b] ^= 1u;
                for (int l = 0; l < L; ++l) {
                    const LayerDev& ld = a.layer[l];
                    const int steps = l == 0 ? 2 : 4;
                    for (int step = 0; step < steps; ++step) {
                        const int nh = step & 1, kh = step >> 1;
                        if (kh == 0 && (k > 0 || l > 0)) {
                            const unsigned long long c0 = prof_clock();
                            mbar_wait(&a_ready[nh], ar_ph[nh]);
                            pw_a += prof_clock() - c0;
                            ar_ph[nh] ^= 1u;
                        }
                        tc_fence_after();
                        const uint32_t d_main = tmem + static_cast<uint32_t>(nh * 256);
                        const uint32_t d_corr = d_main + 128;
                        bool acc = false;
                        if (kh == 0 && ld.ext) {
                            const unsigned long long c0 = prof_clock();
                            mbar_wait(&full[stage], phase);
                            pw_f += prof_clock() - c0;
                            tc_fence_after();
                            const uint32_t xs = s_base + stage * STAGE;
                            const uint64_t adesc = noswz_desc(ax_base + b * AX_BYTES, 128, 256);
                            mma_bf16_pair(d_main, adesc, noswz_desc(xs, 128, 256), idesc, 0u);
                            mma_bf16_pair(d_corr, adesc, noswz_desc(xs + XHALF, 128, 256), idesc, 0u);
                            mma_commit_pair(&empty[stage], 3);
                            if (++stage == STAGES) stage = 0, phase ^= 1u;
                            acc = true;
                        }
                        if (l > 0) {
                            for (int ks = 0; ks < KSL; ++ks) {
                                // the slab's stages: [hi | lo'] in one, or hi then lo' in the next
                                const int st2 = (SPS == 2 && stage + 1 == STAGES) ? 0 : stage + SPS - 1;
                                const uint32_t ph2 = (SPS == 2 && stage + 1 == STAGES) ? phase ^ 1u : phase;
                                const unsigned long long c0 = prof_clock();
                                mbar_wait(&full[stage], phase);
                                if (SPS == 2) mbar_wait(&full[st2], ph2);
                                pw_f += prof_clock() - c0;
                                tc_fence_after();
                                const uint32_t aoff = static_cast<uint32_t>(kh * KSL + ks) * A_SLAB;
                                const uint32_t bhi = s_base + static_cast<uint32_t>(stage) * STAGE;
                                const uint32_t blo = SPS == 2 ? s_base + static_cast<uint32_t>(st2) * STAGE : bhi + C::PLANE_B;
#pragma unroll
                                for (int kk = 0; kk < 4; ++kk) {
                                    const uint32_t first = (acc || kh || ks || kk) ? 1u : 0u;
                                    const uint64_t a_hi = sw128_desc(ahi + aoff + kk * 32);
                                    const uint64_t b_hi = sw128_desc(bhi + kk * 32);
                                    mma_bf16_pair(d_main, a_hi, b_hi, idesc, first);
                                    mma_bf16_pair(d_corr, a_hi, sw128_desc(blo + kk * 32), idesc, first);
                                    mma_bf16_pair(d_corr, sw128_desc(alo + aoff + kk * 32), b_hi, idesc, 1u);
                                }
                                mma_commit_pair(&empty[stage], 3);
                                if (SPS == 2) mma_commit_pair(&empty[st2], 3);
                                for (int sub = 0; sub < SPS; ++sub)
                                    if (++stage == STAGES) stage = 0, phase ^= 1u;
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
    } else if (warp < OUT_WARP) {
        // ---------------------------------------------------------------- epilogue --
        const int e = warp - 2;
        const uint32_t quad = static_cast<uint32_t>(warp & 3);
        const int ch = e >> 2;
        // width 256: lane quadrant = 32 rows, all of the n-half's columns; width 512 ("2x2"
        // accumulator): quadrants 0/1 = rows 0-31/32-63 of n-half columns 0-127, 2/3 = the same
        // rows of columns 128-255
        const uint32_t row = (N == 256 ? quad : (quad & 1u)) * 32 + lane;
        const int cq = N == 256 ? 0 : static_cast<int>(quad >> 1) * 128;
        const int part = (N == 256 ? 0 : static_cast<int>(quad >> 1) * 2) + ch;
        const uint32_t t_lane = (quad * 32u) << 16;
        const uint32_t a_ready0 = mapa_shared(smem_u32(a_ready), 0);
        uint32_t dp[2] = {0u, 0u}, oe_ph[2] = {0u, 0u};
        unsigned long long pe_d = 0, pe_w = 0, pe_o = 0;  // SVN_KERNEL_PROF accounting
        int64_t k = 0;
        for (int64_t t = pair; t < a.n_tiles; t += npairs, ++k) {
            float4 dot = make_float4(0.f, 0.f, 0.f, 0.f);
            bool ovf = false;
            __half2 hmax = __float2half2_rn(0.f);
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
                    const uint32_t tb = tmem + t_lane + static_cast<uint32_t>(j * 256 + ch * COLS);
                    static_assert(COLS == 64, "two 32-column chunks per thread per half");
                    const int col0 = j * NHO + cq + ch * COLS;
                    // truncation compensation: main x (1 + rz_comp x (MMAs into main) x 2^-23)
                    const float kmul =
                        1.0f + a.rz_comp * static_cast<float>(l == 0 ? 1 : N / 16 + (ld.ext ? 1 : 0)) * (1.0f / 8388608.0f);
                    float v[32];
                    {
                        uint32_t rm[32], rc[32];
                        tmem_ld32_async(tb, rm);
                        tmem_ld32_async(tb + 128, rc);
                        tmem_wait_tied(rm);
                        tmem_wait_tied(rc);
                        combine32(rm, rc, kmul, v);
                    }
                    // second chunk's loads fly while the first chunk is split and stored
                    uint32_t rm2[32], rc2[32];
                    tmem_ld32_async(tb + 32, rm2);
                    tmem_ld32_async(tb + 128 + 32, rc2);
                    epi32<TM>(ld, l, last, v, col0, row, Ahi, Alo, wo_s, dot, ovf, hmax);
                    tmem_wait_tied(rm2);
                    tmem_wait_tied(rc2);
                    combine32(rm2, rc2, kmul, v);
                    epi32<TM>(ld, l, last, v, col0 + 32, row, Ahi, Alo, wo_s, dot, ovf, hmax);
                    pe_w += prof_clock() - c1;
                    tc_fence_before();
                    if (!last) fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_remote(a_ready0 + j * 8u);
                }
            }
            // hand the row's partial dot to the output warp (dotbuf[parity] is reused two tiles later)
            const unsigned long long c3 = prof_clock();
            const int b = static_cast<int>(k & 1);
            if (k >= 2) {
                mbar_wait(&out_empty[b], oe_ph[b]);
                oe_ph[b] ^= 1u;
            }
            ovf |= __hisinf(__low2half(hmax)) || __hisinf(__high2half(hmax));  // an activation beyond fp16
            dotbuf[(b * PARTS + part) * TM + row] = ovf ? -INFINITY : (dot.x + dot.y) + (dot.z + dot.w);
            __syncwarp();
            if (lane == 0) mbar_arrive(&out_full[b]);
            pe_o += prof_clock() - c3;
        }
        if (a.prof && e == 0 && lane == 0 && rank == 0) {
            atomicAdd(a.prof + kProfEpiWaitD, pe_d);
            atomicAdd(a.prof + kProfEpiWork, pe_w);
            atomicAdd(a.prof + kProfEpiOut, pe_o);
        }
    } else {
        // ------------------------------------------------------------- output warp --
        // Per finished tile: delta = dot + bo for this CTA's 128 rows, per-point stores, one
        // packed-key atomicMin and the per-motion completion counter; then the A extension of
        // the tile two ahead (same parity), whose point loads are issued before the wait.
        const uint32_t ax_full0 = mapa_shared(smem_u32(ax_full), 0);
        uint32_t of_ph[2] = {0u, 0u};
        float px[RQ][3];
        auto load_points = [&](int64_t t) {
            int32_t motion, nrows;
            int64_t pbase, obase;
            tile_decode(a, t, 2 * TM, motion, pbase, obase, nrows);
#pragma unroll
            for (int q = 0; q < RQ; ++q) {
                const int32_t r = static_cast<int32_t>(rank * TM + q * 32 + lane);
                const float* xp = a.points + (pbase + (r < nrows ? r : 0)) * a.point_stride;
                px[q][0] = xp[0];
                px[q][1] = xp[1];
                px[q][2] = xp[2];
            }
        };
        auto store_ax = [&](int b) {
#pragma unroll
            for (int q = 0; q < RQ; ++q)
                write_ax(AX + b * AX_BYTES, static_cast<uint32_t>(q * 32) + lane, (px[q][0] - a.shift[0]) * a.scale[0],
                         (px[q][1] - a.shift[1]) * a.scale[1], (px[q][2] - a.shift[2]) * a.scale[2]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(ax_full0 + b * 8u);
        };
        for (int b = 0; b < 2; ++b) {
            const int64_t t = pair + b * npairs;
            if (t < a.n_tiles) {
                load_points(t);
                store_ax(b);
            }
        }
        int64_t k = 0;
        for (int64_t t = pair; t < a.n_tiles; t += npairs, ++k) {
            const int b = static_cast<int>(k & 1);
            const bool next = t + 2 * npairs < a.n_tiles;
            if (next) load_points(t + 2 * npairs);
            int32_t motion, nrows;
            int64_t pbase, obase;
            tile_decode(a, t, 2 * TM, motion, pbase, obase, nrows);
            mbar_wait(&out_full[b], of_ph[b]);
            of_ph[b] ^= 1u;
            // every MMA of tile t has completed, so AX[b] is free for tile t + 2 npairs
            if (next) store_ax(b);
            float delta[RQ];
#pragma unroll
            for (int q = 0; q < RQ; ++q) {
                const int r = q * 32 + static_cast<int>(lane);
                float p[PARTS];
                bool inf = false;
#pragma unroll
                for (int i = 0; i < PARTS; ++i) {
                    p[i] = dotbuf[(b * PARTS + i) * TM + r];
                    inf |= p[i] == -INFINITY;
                }
                const float sum = PARTS == 2 ? p[0] + p[1] : (p[0] + p[1]) + (p[PARTS - 2] + p[PARTS - 1]);
                // a part saw an fp16 overflow: -inf, whatever the other parts hold
                delta[q] = inf ? -INFINITY : sum + a.bo;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&out_empty[b]);
            unsigned long long key = ~0ull;
#pragma unroll
            for (int q = 0; q < RQ; ++q) {
                const int32_t rr = static_cast<int32_t>(rank * TM + q * 32 + lane);
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
        }
    }

    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    if (warp == 1) tmem_dealloc_pair(tmem, 512);
}

template <int N>
static cudaError_t launch_split_n(const FusedArgs& a, int num_sms, cudaStream_t st) {
    using C = sp::Cfg<N>;
    static SmemOptIn opt;
    cudaError_t e = opt.ensure(reinterpret_cast<const void*>(fused_split_kernel<N>), (int)C::SMEM);
    if (e != cudaSuccess) return e;
    int64_t pairs = num_sms / 2;
    if (a.n_tiles < pairs) pairs = a.n_tiles;
    if (pairs < 1) return cudaSuccess;
    const cudaError_t le = launch_fused_pdl(fused_split_kernel<N>, static_cast<unsigned>(2 * pairs), C::THREADS,
                                            C::SMEM, st, a);
    return le != cudaSuccess ? le : cudaGetLastError();
}

cudaError_t launch_fused_split(const FusedArgs& a, int num_sms, cudaStream_t st) {
    switch (a.N) {
        case 256: return launch_split_n<256>(a, num_sms, st);
        case 512: return launch_split_n<512>(a, num_sms, st);
        default: return cudaErrorInvalidValue;
    }
}

// ---------------------------------------------------------------- K0 (split) --
// Per motion m and concat slot s: b_m = b + Wq . zq (fp32), then extension rows per
// (n-half, CTA half): [main: (b_h, w0h, w1h, w2h, 0..)] [corr: (b_l', w0l', w1l', w2l', w0h, w1h, w2h, 0..)].
struct QNormS {
    float shift[kMaxIn], scale[kMaxIn];
};

template <int N>
__global__ void split_ext_kernel(const float* __restrict__ q01, int dof, int n_mb, const float* __restrict__ wq,
                                 const float* __restrict__ base_bias, const float* __restrict__ wx_slots,
                                 uint8_t* __restrict__ ext, const QNormS qn, unsigned long long* keys,
                                 unsigned int* counters, int64_t n_keys) {
    pdl_launch_dependents();  // the fused kernel may start its prologue now (it pdl_wait()s for our writes)
    using namespace sp;
    constexpr int NHO = Cfg<N>::NHO, BRH = Cfg<N>::BRH;
    constexpr uint32_t XHALF = Cfg<N>::XHALF;
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
    const float* wx = wx_slots + static_cast<int64_t>(slot) * 3 * N;
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
        float acc = base_bias[slot * N + n];
        for (int k = 0; k < nq; ++k) acc = __fmaf_rn(zq[k], w[k * N + n], acc);
        __half bh, bl, h0, l0, h1, l1, h2, l2;
        split(acc, bh, bl);
        split(wx[n], h0, l0);
        split(wx[N + n], h1, l1);
        split(wx[2 * N + n], h2, l2);
        const __half z = __float2half_rn(0.0f);
        __align__(16) __half mv[16] = {bh, h0, h1, h2, z, z, z, z, z, z, z, z, z, z, z, z};
        __align__(16) __half cv[16] = {bl, l0, l1, l2, h0, h1, h2, z, z, z, z, z, z, z, z, z};
        const int nh = n / NHO, wi = n % NHO, r = wi / BRH, rr = wi % BRH;
        uint8_t* blob = ext + (((m * n_mb + slot) * 2 + nh) * 2 + r) * (2 * XHALF);
        *reinterpret_cast<uint4*>(blob + ext_offset(rr, 0)) = *reinterpret_cast<const uint4*>(&mv[0]);
        *reinterpret_cast<uint4*>(blob + ext_offset(rr, 8)) = *reinterpret_cast<const uint4*>(&mv[8]);
        *reinterpret_cast<uint4*>(blob + XHALF + ext_offset(rr, 0)) = *reinterpret_cast<const uint4*>(&cv[0]);
        *reinterpret_cast<uint4*>(blob + XHALF + ext_offset(rr, 8)) = *reinterpret_cast<const uint4*>(&cv[8]);
    }
}

cudaError_t launch_split_ext(const FusedArgs& a, const float* wq, const float* mb_base_bias, const float* wx_slots,
                             uint8_t* ext, unsigned long long* keys_init, unsigned int* counters_init, int64_t n_keys,
                             cudaStream_t st) {
    if (a.M <= 0) return cudaSuccess;
    QNormS qn;
    for (int k = 0; k < 2 * a.dof && k < kMaxIn; ++k) {
        qn.shift[k] = a.shift[3 + k];
        qn.scale[k] = a.scale[3 + k];
    }
    dim3 grid(static_cast<unsigned>(a.M), a.n_mb > 0 ? a.n_mb : 1);
    if (a.N == 512)
        split_ext_kernel<512><<<grid, 256, 0, st>>>(a.q01, a.dof, a.n_mb, wq, mb_base_bias, wx_slots, ext, qn, keys_init,
                                                    counters_init, n_keys);
    else
        split_ext_kernel<256><<<grid, 256, 0, st>>>(a.q01, a.dof, a.n_mb, wq, mb_base_bias, wx_slots, ext, qn, keys_init,
                                                    counters_init, n_keys);
    return cudaGetLastError();
}

}  // namespace svn
