// abi_query.cu — C-ABI: kernel selection and sequencing (K0 -> fused K1), dense queries
// (device and host buffers), forward_eval rows of mixed motions, predict_min_distance,
// dense-grid evaluation; scratch, staging and per-thread streams.
#include "abi_internal.cuh"

using namespace svn;
using namespace svn::abi;

namespace svn {
namespace abi {

svn_status check_prec(const svn_model* m, svn_precision prec) {
    if (prec == SVN_PREC_BF16) {
        if (!m->has_bf16) return fail(SVN_ERR_UNSUPPORTED, "bf16 path needs width 256 or 512");
    } else if (prec == SVN_PREC_FP16) {
        if (!m->has_f16)
            return fail(SVN_ERR_UNSUPPORTED, "fp16 path needs width 256 or 512 and every weight inside the fp16 range");
    } else if (prec == SVN_PREC_FP32 || prec == SVN_PREC_FP32_EXACT) {
        if (m->N != 128 && m->N != 256 && m->N != 512)
            return fail(SVN_ERR_UNSUPPORTED, "fp32 path needs width 128, 256 or 512");
    } else if (prec == SVN_PREC_FP32_SPLIT) {
        if (!m->has_split)
            return fail(SVN_ERR_UNSUPPORTED, "fp32_split path needs width 256 or 512, >= 2 layers and |W| < 1e4");
    } else {
        return fail(SVN_ERR_INVALID_ARGUMENT, "unknown precision");
    }
    return SVN_OK;
}

// Which fused kernel serves a (model, precision): bf16 tensor cores; fp32-grade split-fp16
// tensor cores (fp32_split, width 256); or SIMT FFMA in the oracle's order (fp32, fp32_exact).
Kind kernel_kind(const svn_model*, svn_precision prec) {
    if (prec == SVN_PREC_BF16 || prec == SVN_PREC_FP16) return Kind::BF16;  // one kernel family, two operand formats
    if (prec == SVN_PREC_FP32_SPLIT) return Kind::SPLIT;
    return Kind::SIMT;
}

// rows per tile (a CTA pair's tile for the tensor-core kernels; fp32_split at width 512 holds
// 64 rows per CTA)
int tile_rows(Kind k, int N) {
    if (k == Kind::SIMT) return N >= 512 ? 64 : 128;
    return (k == Kind::SPLIT && N == 512) ? 128 : 256;
}
// SIMT: a query with fewer big tiles than SMs is cut into 32-row tiles (4 warps per CTA,
// more SMs busy; each output's k-ordered FMA chain is unchanged)
// bf16 (width 512 and 256): a launch with fewer 256-row tiles than CTA pairs (one motion x a few
// thousand points — the reference's per-motion predict_min_distance) is latency-bound, so it
// runs 128-row pair tiles (64 rows per CTA, M=128 MMAs): twice the tiles, each through the
// network in about half the time.  SVN_PAIR_TILE=128|256 forces one (A/B hook).
// svn_set_whole_batch: the shape of the batch this thread's calls are shards of (0 = none)
thread_local int64_t g_whole_M = 0, g_whole_P = 0;

int tile_rows_for(Kind k, int N, int64_t big_tiles, int num_sms) {
    const int t = tile_rows(k, N);
    if (k == Kind::SIMT && big_tiles < num_sms) return kFp32SmallTile;
    if (k == Kind::BF16 && (N == 512 || N == 256)) {
        static const int forced = [] {
            const char* e = std::getenv("SVN_PAIR_TILE");
            return e ? std::atoi(e) : 0;
        }();
        if (forced == 128 || forced == 256) return forced;
        if (big_tiles < num_sms / 2) return 128;
    }
    return t;
}




thread_local Arena* g_arena = nullptr;

// SVN_HOST_TRACE=1: host-side time of the phases of a small host-buffer query, averaged and
// printed to stderr every 300 calls (where a per-motion call's fixed cost goes).
struct HostTrace {
    static bool on() {
        static const bool v = [] {
            const char* e = std::getenv("SVN_HOST_TRACE");
            return e && e[0] == '1';
        }();
        return v;
    }
    double acc[9] = {};
    int n = 0;
    std::chrono::steady_clock::time_point t;
    void start() { t = std::chrono::steady_clock::now(); }
    void lap(int i) {
        const auto now = std::chrono::steady_clock::now();
        acc[i] += std::chrono::duration<double, std::micro>(now - t).count();
        t = now;
    }
    void done() {
        if (++n < 300) return;
        std::fprintf(stderr, "[svn host] us/call: fill %.1f | stage %.1f | scratch %.1f | K0 %.1f | K1 %.1f | D2H %.1f | sync %.1f | out %.1f | pin %.1f\n",
                     acc[0] / n, acc[1] / n, acc[2] / n, acc[3] / n, acc[4] / n, acc[5] / n, acc[6] / n, acc[7] / n, acc[8] / n);
        n = 0;
        for (double& x : acc) x = 0;
    }
};
thread_local HostTrace g_trace;
thread_local bool g_trace_on = false;
#define SVN_TRACE(i) \
    do {             \
        if (g_trace_on) g_trace.lap(i); \
    } while (0)

Arena& thread_arena(int device) {
    thread_local Arena ar[8];
    thread_local Arena other;
    Arena& a = (device >= 0 && device < 8) ? ar[device] : other;
    a.device = device;
    return a;
}

Staging& thread_staging(int device) {
    thread_local Staging st[8];
    thread_local Staging other;
    return (device >= 0 && device < 8) ? st[device] : other;
}


void ensure_pool(int device) {
    static std::once_flag flags[64];
    if (device < 0 || device >= 64) return;
    std::call_once(flags[device], [device] {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t threshold = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
        }
    });
}

cudaError_t launch_k1(const FusedArgs& a, Kind kind, int num_sms, cudaStream_t st) {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (g_timing) {
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
    }
    unsigned long long* dprof = nullptr;
    FusedArgs ap = a;
    if (prof_enabled()) {
        cudaMalloc(&dprof, sizeof(unsigned long long) * kProfSlots);
        cudaMemsetAsync(dprof, 0, sizeof(unsigned long long) * kProfSlots, st);
        ap.prof = dprof;
    }
    cudaError_t e = kind == Kind::BF16    ? launch_fused_bf16_pair(ap, num_sms, st)
                    : kind == Kind::SPLIT ? launch_fused_split(ap, num_sms, st)
                                          : launch_fused_fp32(ap, num_sms, st);
    ++g_launches;
    if (dprof) {
        cudaMemcpyAsync(g_prof, dprof, sizeof(g_prof), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        cudaFree(dprof);
        std::fprintf(stderr, "[svn prof]");
        for (int i = 0; i < kProfSlots; ++i) std::fprintf(stderr, " %llu", g_prof[i]);
        std::fprintf(stderr, "\n");
    }
    if (g_timing) {
        cudaEventRecord(e1, st);
        g_events.emplace_back(e0, e1);
    }
    return e;
}

// bf16: per-motion K=16 extension rows (folded bias + x-part splits) and their TMA view.
svn_status motion_ext(const svn_model* m, FusedArgs& a, int64_t M, unsigned long long* keys, unsigned int* counters,
                      int64_t n_keys, Scratch& sc, cudaStream_t st, bool split) {
    uint8_t* ext = nullptr;
    if (split) {  // [motion][slot][n-half][CTA half][main N/4 rows | corr N/4 rows] x 32 B
        const size_t rows = static_cast<size_t>(M) * (m->n_mb ? m->n_mb : 1) * 2 * m->N;
        SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&ext), rows * 32), "cudaMallocAsync(split ext)");
        svn_status s = encode_blob_map(&a.tmap_xq, ext, 32, rows, static_cast<uint32_t>(m->N / 2));
        if (s != SVN_OK) return s;
        SVN_CUDA(launch_split_ext(a, m->d_wq, m->d_mbbase, m->d_wxslots, ext, keys, counters, n_keys, st),
                 "split_ext kernel");
        ++g_launches;
        return SVN_OK;
    }
    unsigned int* sched = nullptr;  // dynamic tile counter of the width-512 kernel, zeroed by K0
    SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&sched), sizeof(unsigned int)), "cudaMallocAsync(tile counter)");
    a.sched = sched;
    {
        // chunks of 4 consecutive tiles per claim once every pair has >= 32 tiles: the ext ring is
        // rebuilt about once per chunk; the end-of-kernel spread grows by at most 3 tiles (~0.1 ms)
        static const int g_env = [] {
            const char* e = std::getenv("SVN_TILE_GROUP");  // A/B hook
            return e ? std::atoi(e) : 0;
        }();
        const int64_t pairs = std::max<int64_t>(1, m->num_sms / 2);
        a.tile_group = g_env > 0 ? g_env : (a.n_tiles >= pairs * 32 ? 4 : 1);
    }
    static const int ext_mode = [] {  // test / A-B hook: SVN_BF16_EXT=k0 | ring (default: by size)
        const char* e = std::getenv("SVN_BF16_EXT");
        return !e ? 0 : std::strcmp(e, "k0") == 0 ? 1 : std::strcmp(e, "ring") == 0 ? 2 : 0;
    }();
    const size_t stream_bytes = static_cast<size_t>(M) * (m->n_mb ? m->n_mb : 1) * m->N * 32;
    // width 512, a per-motion stream that would not stay in L2 (> 16 MB: c3, c4, c5): the fused
    // kernel's output warps build each tile's extension rows in a ring of three tile slots per CTA
    // (grid x 3 x n_mb x 2 n-halves x N/4 rows x 32 B: 7.3 MB on c3, L2-resident) — no per-motion
    // stream in HBM; K0 only resets keys, counters and the queue.  Small batches (one motion per
    // call, the reference's predict_min_distance) keep K0's parallel build: its rows stay in L2
    // and the fused kernel's first tiles do not wait for an output warp to build them.
    const bool ring = ext_mode == 2 || (ext_mode == 0 && stream_bytes > (size_t(16) << 20));
    if (m->N == 512 && ring) {
        const int64_t ctas = 2 * std::min<int64_t>(m->num_sms / 2, std::max<int64_t>(a.n_tiles, 1));
        const size_t rows = static_cast<size_t>(ctas) * 3 * (m->n_mb ? m->n_mb : 1) * 2 * (m->N / 4);  // 3 slots
        SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&ext), rows * 32), "cudaMallocAsync(ext ring)");
        svn_status s = encode_blob_map(&a.tmap_xq, ext, 32, rows, static_cast<uint32_t>(m->N / 4));
        if (s != SVN_OK) return s;
        a.ext_ring = ext;
        a.xq_wq = m->d_wq_bf;
        a.xq_base = m->d_mbbase_bf;
        SVN_CUDA(launch_ext_ring_init(ext, ctas, m->n_mb ? m->n_mb : 1, m->N, m->d_wxslots_bf, a.f16, st),
                 "ext ring init");
        ++g_launches;
        SVN_CUDA(launch_motion_ext(a, m->d_wq_bf, m->d_mbbase_bf, m->d_wxslots_bf, nullptr, keys, counters, n_keys,
                                   sched, st),
                 "motion_ext kernel (resets)");
        ++g_launches;
        return SVN_OK;
    }
    a.ext_ring = nullptr;
    const size_t rows = static_cast<size_t>(M) * (m->n_mb ? m->n_mb : 1) * m->N;
    SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&ext), rows * 32), "cudaMallocAsync(motion ext)");
    svn_status s = encode_blob_map(&a.tmap_xq, ext, 32, rows, static_cast<uint32_t>(m->N == 256 ? m->N / 2 : m->N / 4));
    if (s != SVN_OK) return s;
    SVN_CUDA(launch_motion_ext(a, m->d_wq_bf, m->d_mbbase_bf, m->d_wxslots_bf, ext, keys, counters, n_keys, sched, st),
             "motion_ext kernel");
    ++g_launches;
    return SVN_OK;
}

// Shared body of the dense query (full result or keys-only partial).
svn_status query_dense(const svn_model* m, svn_precision prec, const float* points, int64_t P, int64_t index_offset,
                       const float* q01, int64_t M, double margin, float* min_out, int32_t* argmin_out,
                       uint8_t* free_out, float* per_point, uint64_t* keys_partial, cudaStream_t st) {
    NvtxRange nvtx("svn query (K0 + fused K1)");
    if (!m) return fail(SVN_ERR_INVALID_ARGUMENT, "query: null model");
    if (P < 1) return fail(SVN_ERR_INVALID_ARGUMENT, "predict_min_distance: empty point cloud");
    if (M < 1) return fail(SVN_ERR_INVALID_ARGUMENT, "query: no motions");
    {
        // TMA row coordinates of the per-motion extension stream are int32: beyond ~1e9 rows
        // (about a million motions at width 512) the query runs as consecutive motion chunks
        static const int64_t override_max = [] {
            const char* e = std::getenv("SVN_MAX_MOTIONS_PER_LAUNCH");  // test hook
            return e ? std::atoll(e) : 0ll;
        }();
        const int64_t rows_per_motion = static_cast<int64_t>(m->n_mb ? m->n_mb : 1) * m->N * 2;
        int64_t max_m = (static_cast<int64_t>(INT32_MAX) / 2) / rows_per_motion;
        if (override_max > 0) max_m = override_max;
        if (max_m < 1) max_m = 1;
        if (M > max_m) {
            const int64_t nq = 2 * static_cast<int64_t>(m->dof);
            for (int64_t b0 = 0; b0 < M; b0 += max_m) {
                const int64_t n = std::min(max_m, M - b0);
                const svn_status s = query_dense(m, prec, points, P, index_offset, q01 + b0 * nq, n, margin,
                                                 min_out ? min_out + b0 : nullptr, argmin_out ? argmin_out + b0 : nullptr,
                                                 free_out ? free_out + b0 : nullptr,
                                                 per_point ? per_point + b0 * P : nullptr,
                                                 keys_partial ? keys_partial + b0 : nullptr, st);
                if (s != SVN_OK) return s;
            }
            return SVN_OK;
        }
    }
    if (P + index_offset > 0xFFFFFFFFll) return fail(SVN_ERR_UNSUPPORTED, "query: more than 2^32 points");
    svn_status s = check_prec(m, prec);
    if (s != SVN_OK) return s;
    DeviceGuard guard(m->device);
    ensure_pool(m->device);
    const Kind kind0 = kernel_kind(m, prec);
    FusedArgs a = kind0 == Kind::SPLIT  ? m->base_split
                  : kind0 == Kind::BF16 ? (prec == SVN_PREC_FP16 ? m->base_f16 : m->base_bf16)
                                        : m->base;
    // fp32 on the SIMT kernel runs in the oracle's order (no q-fold): at width 512 that costs
    // nothing measurable (c3/c4: 12.0/16.8 M q/s either way) and makes it bit-identical
    const bool exact = kind0 == Kind::SIMT;
    a.exact = exact ? 1 : 0;
    a.points = points;
    a.point_stride = 3;
    a.P = P;
    a.q01 = q01;
    a.M = M;
    const Kind kind = kernel_kind(m, prec);
    const int TM0 = tile_rows(kind, m->N);
    // a shard takes the tile shape of the batch it is a shard of (same bits whatever the split)
    const bool shard = g_whole_M > 0 && g_whole_P > 0 && kind != Kind::SIMT;
    const int TM = tile_rows_for(kind, m->N, shard ? g_whole_M * ((g_whole_P + TM0 - 1) / TM0) : M * ((P + TM0 - 1) / TM0),
                                 m->num_sms);
    a.tile_rows = TM;
    a.tiles_per_motion = (P + TM - 1) / TM;
    a.n_tiles = a.tiles_per_motion * M;
    a.tiles = nullptr;
    a.margin = margin;
    a.per_point = per_point;
    a.index_offset = index_offset;
    Scratch sc(st);
    float* mb = nullptr;
    const int n_mb = exact ? 0 : m->n_mb;
    if (kind == Kind::SIMT)
        SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&mb),
                          sizeof(float) * static_cast<size_t>(M) * (n_mb ? n_mb : 1) * m->N),
                 "cudaMallocAsync(motion_bias)");
    a.motion_bias = mb;
    a.n_mb = m->n_mb;  // slot stride stays the model's (exact mode never reads it)
    unsigned long long* keys = nullptr;
    unsigned int* counters = nullptr;
    if (keys_partial) {
        keys = reinterpret_cast<unsigned long long*>(keys_partial);
    } else {
        SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&keys), sizeof(unsigned long long) * M), "cudaMallocAsync(keys)");
        SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&counters), sizeof(unsigned int) * M), "cudaMallocAsync(counters)");
    }
    a.keys = keys;
    a.counters = counters;
    a.min_out = min_out;
    a.argmin_out = argmin_out;
    a.free_out = free_out;
    SVN_TRACE(2);
    if (kind != Kind::SIMT) {
        s = motion_ext(m, a, M, keys_partial ? nullptr : keys, counters, keys_partial ? 0 : M, sc, st,
                       kind == Kind::SPLIT);
        if (s != SVN_OK) return s;
    } else {
        FusedArgs k0 = a;
        k0.n_mb = n_mb;
        SVN_CUDA(launch_motion_bias(k0, m->d_wq, m->d_mbbase, mb, keys_partial ? nullptr : keys, counters,
                                    keys_partial ? 0 : M, st),
                 "motion_bias kernel");
        ++g_launches;
    }
    SVN_TRACE(3);
    SVN_CUDA(launch_k1(a, kind, m->num_sms, st), "fused MLP kernel");
    SVN_TRACE(4);
    return SVN_OK;
}

// One non-blocking stream per (thread, device), destroyed when the thread exits (callers such
// as the reference's parallel_for workers come and go).
struct ThreadStreams {
    cudaStream_t s[64] = {};
    ~ThreadStreams() {
        for (int d = 0; d < 64; ++d)
            if (s[d]) {
                int prev = 0;
                cudaGetDevice(&prev);
                cudaSetDevice(d);
                cudaStreamDestroy(s[d]);
                cudaSetDevice(prev);
            }
    }
};

cudaStream_t thread_stream(int device) {
    thread_local ThreadStreams ts;
    if (device < 0 || device >= 64) return nullptr;
    if (!ts.s[device]) cudaStreamCreateWithFlags(&ts.s[device], cudaStreamNonBlocking);
    return ts.s[device];
}

// A second stream per (thread, device) for the host->device copies of a large cloud, and a few
// events to hand its chunks to the compute stream (query_min_host's pipelined path).
struct ThreadCopy {
    static constexpr int kEvents = 8;
    cudaStream_t s[64] = {};
    cudaEvent_t ev[64][kEvents] = {};
    ~ThreadCopy() {
        for (int d = 0; d < 64; ++d)
            if (s[d]) {
                int prev = 0;
                cudaGetDevice(&prev);
                cudaSetDevice(d);
                for (cudaEvent_t e : ev[d])
                    if (e) cudaEventDestroy(e);
                cudaStreamDestroy(s[d]);
                cudaSetDevice(prev);
            }
    }
};

ThreadCopy* thread_copy(int device) {
    thread_local ThreadCopy tc;
    if (device < 0 || device >= 64) return nullptr;
    if (!tc.s[device]) {
        if (cudaStreamCreateWithFlags(&tc.s[device], cudaStreamNonBlocking) != cudaSuccess) return nullptr;
        for (cudaEvent_t& e : tc.ev[device])
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    }
    return &tc;
}

}  // namespace abi
}  // namespace svn

namespace svn {
namespace abi {

// forward_eval (nn.cpp:95-130).  Consecutive rows with identical (q0, q1) form one
// motion segment; each segment is cut into tiles of one motion.
svn_status forward_rows(const svn_model* m, svn_precision prec, const float* raw_host, const float* raw_dev,
                               int64_t B, int64_t cols, float* out_dev, cudaStream_t st) {
    NvtxRange nvtx("svn forward_eval rows");
    if (!m) return fail(SVN_ERR_INVALID_ARGUMENT, "forward: null model");
    if (cols != m->in) return fail(SVN_ERR_INVALID_ARGUMENT, "forward: input width mismatch");
    if (B < 1) return fail(SVN_ERR_INVALID_ARGUMENT, "forward: batch must be non-empty");
    svn_status s = check_prec(m, prec);
    if (s != SVN_OK) return s;
    {
        // every row can be its own motion: keep the per-motion extension stream inside the
        // int32 TMA row range by running large batches as row chunks (rows are independent)
        static const int64_t override_max = [] {
            const char* e = std::getenv("SVN_MAX_MOTIONS_PER_LAUNCH");  // test hook
            return e ? std::atoll(e) : 0ll;
        }();
        const int64_t rows_per_motion = static_cast<int64_t>(m->n_mb ? m->n_mb : 1) * m->N * 2;
        int64_t max_b = (static_cast<int64_t>(INT32_MAX) / 2) / rows_per_motion;
        if (override_max > 0) max_b = override_max;
        if (max_b < 1) max_b = 1;
        if (B > max_b) {
            for (int64_t b0 = 0; b0 < B; b0 += max_b) {
                const int64_t n = std::min(max_b, B - b0);
                s = forward_rows(m, prec, raw_host + b0 * cols, raw_dev + b0 * cols, n, cols, out_dev + b0, st);
                if (s != SVN_OK) return s;
            }
            return SVN_OK;
        }
    }
    Kind kind = kernel_kind(m, prec);
    const int nq = 2 * m->dof;
    if (kind != Kind::SIMT && !(kind == Kind::BF16 && m->N == 512 && m->has_mixed)) {
        // rows of mostly distinct motions (segments shorter than 32 rows on average) would cost
        // the folded tensor-core kernels one tile per segment; without a per-row q-part variant
        // (width-512 bf16 has one, below) they run on the FP32 path, which reads each row's q and
        // is exact — inside every stated bound, and faster than one tile per row
        int64_t segs = 1;
        for (int64_t r = 1; r < B && segs * 32 <= B; ++r)
            segs += std::memcmp(raw_host + r * cols + 3, raw_host + (r - 1) * cols + 3, sizeof(float) * nq) != 0;
        if (segs * 32 > B) kind = Kind::SIMT;
    }
    const int TM0 = tile_rows(kind, m->N);
    const int TM = tile_rows_for(kind, m->N, (B + TM0 - 1) / TM0, m->num_sms);
    if (kind == Kind::SIMT) {
        // the FP32 path does not fold q (exact order): every row reads its own q0|q1 from the raw
        // batch, so tiles are cut over the rows regardless of motion — a batch whose rows all
        // differ in motion (eval_mae, bench.cpp:80-88; training validation, nn.cpp:370) runs
        // full tiles instead of one tile per row
        std::vector<TileDesc> tiles;
        for (int64_t t0 = 0; t0 < B; t0 += TM)
            tiles.push_back(TileDesc{t0, t0, 0, static_cast<int32_t>(std::min<int64_t>(TM, B - t0))});
        FusedArgs a = m->base;
        a.exact = 1;
        a.row_q = 1;
        a.points = raw_dev;
        a.point_stride = cols;
        a.P = B;
        a.M = 1;
        a.q01 = raw_dev + 3;  // unused with row_q
        a.n_tiles = static_cast<int64_t>(tiles.size());
        a.tile_rows = TM;
        a.tiles_per_motion = 1;
        a.per_point = out_dev;
        a.keys = nullptr;
        a.counters = nullptr;
        a.motion_bias = nullptr;
        Scratch sc(st);
        TileDesc* dt = nullptr;
        SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&dt), sizeof(TileDesc) * tiles.size()), "cudaMallocAsync");
        SVN_CUDA(cudaMemcpyAsync(dt, tiles.data(), sizeof(TileDesc) * tiles.size(), cudaMemcpyHostToDevice, st),
                 "H2D tiles");
        a.tiles = dt;
        SVN_CUDA(launch_k1(a, kind, m->num_sms, st), "fused MLP kernel");
        SVN_CUDA(cudaStreamSynchronize(st), "forward kernels");  // the host tile vector feeds an async copy
        return SVN_OK;
    }
    std::vector<float> qseg;
    std::vector<TileDesc> tiles;
    int64_t seg_start = 0;
    int32_t nseg = 0;
    for (int64_t r = 1; r <= B; ++r) {
        const bool cut = (r == B) || std::memcmp(raw_host + r * cols + 3, raw_host + (r - 1) * cols + 3,
                                                 sizeof(float) * nq) != 0;
        if (!cut) continue;
        qseg.insert(qseg.end(), raw_host + seg_start * cols + 3, raw_host + seg_start * cols + 3 + nq);
        for (int64_t t0 = seg_start; t0 < r; t0 += TM) {
            const int64_t n = (r - t0) < TM ? (r - t0) : TM;
            tiles.push_back(TileDesc{t0, t0, nseg, static_cast<int32_t>(n)});
        }
        ++nseg;
        seg_start = r;
    }
    if (kind == Kind::BF16 && m->N == 512 && m->has_mixed && static_cast<int64_t>(nseg) * 32 > B) {
        // rows of mostly distinct motions (segments shorter than 32 rows on average): instead of
        // one tile per segment, 128-row tiles over the rows with every concat layer's q-part
        // computed per row by the tensor core (FusedArgs::mixed, kernels_bf16_pair.cu)
        tiles.clear();
        for (int64_t t0 = 0; t0 < B; t0 += 128)
            tiles.push_back(TileDesc{t0, t0, 0, static_cast<int32_t>(std::min<int64_t>(128, B - t0))});
        FusedArgs a = prec == SVN_PREC_FP16 ? m->base_f16 : m->base_bf16;
        a.mixed = 1;
        a.points = raw_dev;
        a.point_stride = cols;
        a.q01 = raw_dev + 3;  // K0 reads no motion in this mode
        a.P = B;
        a.M = 1;
        a.n_tiles = static_cast<int64_t>(tiles.size());
        a.tile_rows = 128;
        a.tiles_per_motion = 1;
        a.per_point = out_dev;
        a.keys = nullptr;
        a.counters = nullptr;
        a.ext_ring = nullptr;
        a.tile_group = 1;
        Scratch sc(st);
        TileDesc* dt = nullptr;
        unsigned int* sched = nullptr;
        SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&dt), sizeof(TileDesc) * tiles.size()), "cudaMallocAsync");
        SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&sched), sizeof(unsigned int)), "cudaMallocAsync");
        SVN_CUDA(cudaMemcpyAsync(dt, tiles.data(), sizeof(TileDesc) * tiles.size(), cudaMemcpyHostToDevice, st),
                 "H2D tiles");
        a.tiles = dt;
        a.sched = sched;
        SVN_CUDA(launch_motion_ext(a, m->d_wq_bf, m->d_mbbase_bf, m->d_wxslots_bf, nullptr, nullptr, nullptr, 0, sched,
                                   st),
                 "motion_ext kernel (tile counter reset)");
        ++g_launches;
        SVN_CUDA(launch_k1(a, kind, m->num_sms, st), "fused MLP kernel");
        SVN_CUDA(cudaStreamSynchronize(st), "forward kernels");
        return SVN_OK;
    }
    FusedArgs a = kind == Kind::SPLIT  ? m->base_split
                  : kind == Kind::BF16 ? (prec == SVN_PREC_FP16 ? m->base_f16 : m->base_bf16)
                                       : m->base;
    a.exact = kind == Kind::SIMT ? 1 : 0;
    a.points = raw_dev;
    a.point_stride = cols;
    a.P = B;
    a.M = nseg;
    a.n_tiles = static_cast<int64_t>(tiles.size());
    a.tile_rows = TM;
    a.tiles_per_motion = 1;
    a.per_point = out_dev;
    a.keys = nullptr;
    a.counters = nullptr;
    Scratch sc(st);
    float *dq = nullptr, *mb = nullptr;
    TileDesc* dt = nullptr;
    SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&dq), sizeof(float) * qseg.size()), "cudaMallocAsync");
    SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&dt), sizeof(TileDesc) * tiles.size()), "cudaMallocAsync");
    SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&mb), sizeof(float) * static_cast<size_t>(nseg) * (m->n_mb ? m->n_mb : 1) * m->N),
             "cudaMallocAsync");
    SVN_CUDA(cudaMemcpyAsync(dq, qseg.data(), sizeof(float) * qseg.size(), cudaMemcpyHostToDevice, st), "H2D q");
    SVN_CUDA(cudaMemcpyAsync(dt, tiles.data(), sizeof(TileDesc) * tiles.size(), cudaMemcpyHostToDevice, st), "H2D tiles");
    a.q01 = dq;
    a.tiles = dt;
    a.motion_bias = mb;
    if (kind != Kind::SIMT) {
        s = motion_ext(m, a, nseg, nullptr, nullptr, 0, sc, st, kind == Kind::SPLIT);
        if (s != SVN_OK) return s;
    } else {
        FusedArgs k0 = a;
        k0.n_mb = a.exact ? 0 : m->n_mb;
        SVN_CUDA(launch_motion_bias(k0, m->d_wq, m->d_mbbase, mb, nullptr, nullptr, 0, st), "motion_bias kernel");
        ++g_launches;
    }
    SVN_CUDA(launch_k1(a, kind, m->num_sms, st), "fused MLP kernel");
    // keep the host tile/q vectors alive until the async copies have consumed them
    SVN_CUDA(cudaStreamSynchronize(st), "forward kernels");
    return SVN_OK;
}


constexpr int64_t kSmallStagingPoints = 8192;  // above it the DMA copy is faster (20000 points: +9 us)

bool small_staging_enabled() {  // SVN_SMALL_STAGING=0: DMA copies for every call (A/B hook)
    static const bool on = [] {
        const char* e = std::getenv("SVN_SMALL_STAGING");
        return !(e && e[0] == '0');
    }();
    return on;
}

// svn_query_min / svn_predict_min_distance: inputs from host memory, outputs to host memory.
// fill(pts, q, p0, n) writes points p0..p0+n-1 (when pts != null) and the motions (when q != null)
// as floats into the pinned staging block; points/q01 are
// the caller's float arrays (null for predict_min_distance, whose double inputs are converted
// by fill), sent to the device directly when they are already pinned.
// Small staged calls as one CUDA graph (SVN_GRAPH=0 turns it off): the stage-in kernel, K0
// and the fused kernel (behind its programmatic edge), with scratch from the thread's arena and
// inputs / outputs in the pinned staging block, are captured once per (thread, model,
// precision, P, M, margin, staging block, arena block) and replayed with one graph launch
// instead of three kernel launches.
struct GraphEntry {
    const svn_model* m;
    uint64_t serial;
    int prec;
    int64_t P, M;
    double margin;
    const uint8_t *host, *dev, *arena;
    cudaGraphExec_t exec;
    int64_t launches;
    uint64_t used;
};

struct GraphCache {
    std::vector<GraphEntry> e;
    uint64_t tick = 0;
    ~GraphCache() {
        for (GraphEntry& x : e)
            if (x.exec) cudaGraphExecDestroy(x.exec);
    }
};

bool graphs_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SVN_GRAPH");
        return !(e && e[0] == '0');
    }();
    return on;
}

// true: the call ran (launched) as a graph; false: use the stream path (a failed capture only
// loses the fast path — the stream path reports any real error)
bool small_graph(const svn_model* m, svn_precision prec, int64_t P, int64_t M, double margin, Staging& sg,
                 Arena& arena, size_t o_q, size_t o_min, size_t o_arg, size_t o_free, cudaStream_t st) {
    thread_local GraphCache gc;
    GraphEntry* hit = nullptr;
    for (GraphEntry& x : gc.e)
        if (x.m == m && x.serial == m->serial && x.prec == static_cast<int>(prec) && x.P == P && x.M == M &&
            x.margin == margin && x.host == sg.host && x.dev == sg.dev && x.arena == arena.base) {
            hit = &x;
            break;
        }
    if (!hit) {
        if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        const int64_t l0 = g_launches;
        bool ok = launch_stage_in(sg.host, sg.dev, o_min, st) == cudaSuccess;
        bool fallback_alloc = false;
        if (ok) {
            ArenaScope as(&arena);
            Scratch sc(st);
            ok = query_dense(m, prec, reinterpret_cast<const float*>(sg.dev), P, 0,
                             reinterpret_cast<const float*>(sg.dev + o_q), M, margin,
                             reinterpret_cast<float*>(sg.host + o_min), reinterpret_cast<int32_t*>(sg.host + o_arg),
                             sg.host + o_free, nullptr, nullptr, st) == SVN_OK;
            fallback_alloc = !sc.ptrs.empty();
        }
        cudaGraph_t g = nullptr;
        const cudaError_t ee = cudaStreamEndCapture(st, &g);
        const int64_t launches = g_launches - l0 + 1;
        g_launches = l0;
        cudaGraphExec_t ex = nullptr;
        if (!ok || fallback_alloc || ee != cudaSuccess || !g || cudaGraphInstantiate(&ex, g, 0) != cudaSuccess) {
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
            return false;
        }
        cudaGraphDestroy(g);
        if (gc.e.size() >= 8) {
            auto lru = std::min_element(gc.e.begin(), gc.e.end(),
                                        [](const GraphEntry& x, const GraphEntry& y) { return x.used < y.used; });
            cudaGraphExecDestroy(lru->exec);
            gc.e.erase(lru);
        }
        gc.e.push_back({m, m->serial, static_cast<int>(prec), P, M, margin, sg.host, sg.dev, arena.base, ex, launches, 0});
        hit = &gc.e.back();
    }
    hit->used = ++gc.tick;
    if (cudaGraphLaunch(hit->exec, st) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    g_launches += hit->launches;
    return true;
}

// nn.cpp:469-471's double -> float cast of the cloud, vectorisable (no aliasing)
static void cvt_f64_f32(float* __restrict__ d, const double* __restrict__ src, int64_t n) {
    for (int64_t i = 0; i < n; ++i) d[i] = static_cast<float>(src[i]);
}

template <class Fill>
svn_status query_min_host(const svn_model* m, svn_precision prec, int64_t P, int64_t M, double margin,
                          const float* points, const float* q01, Fill fill, float* min_out, int32_t* argmin_out,
                          uint8_t* free_out, float* per_point) {
    if (!m) return fail(SVN_ERR_INVALID_ARGUMENT, "query: null model");
    if (P < 1) return fail(SVN_ERR_INVALID_ARGUMENT, "predict_min_distance: empty point cloud");
    if (M < 1) return fail(SVN_ERR_INVALID_ARGUMENT, "query: no motions");
    if (!min_out || !argmin_out || !free_out) return fail(SVN_ERR_INVALID_ARGUMENT, "query: null buffer");
    DeviceGuard guard(m->device);
    ensure_pool(m->device);
    cudaStream_t st = thread_stream(m->device);
    const int nq = 2 * m->dof;
    // staged layout: [points | q01] in, [min | argmin | free] out
    const size_t o_q = align256(sizeof(float) * 3 * P), o_min = align256(o_q + sizeof(float) * nq * M);
    const size_t o_arg = align256(o_min + sizeof(float) * M), o_free = align256(o_arg + sizeof(int32_t) * M);
    const size_t total = align256(o_free + M);
    Staging& sg = thread_staging(m->device);
    SVN_CUDA(sg.reserve(m->device, total), "staging buffers");
    // inputs already in pinned memory go to the device directly; pageable ones through the
    // pinned staging block (one host copy, then one H2D).  (cudaPointerGetAttributes is only
    // asked about caller arrays: on pageable memory it costs several microseconds.)
    auto pinned = [](const void* p) {
        cudaPointerAttributes at{};
        return p && cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeHost;
    };
    g_trace_on = HostTrace::on();
    if (g_trace_on) g_trace.start();
    const bool direct = pinned(points) && pinned(q01);
    SVN_TRACE(8);
    Arena& arena = thread_arena(m->device);
    // A large cloud (>= 2^21 points, 24 MB): the points travel in chunks on a
    // second stream while the compute stream folds the chunks already on the device into the
    // per-motion keys (the point-sharding identity: atomicMin over (delta, index) keys, bit-identical
    // to one launch) — pageable callers' staging copy, the H2D and the kernels overlap instead of
    // running one after the other.  SVN_PIPELINE=0 turns it off (A/B hook).
    static const bool pipeline_on = [] {
        const char* e = std::getenv("SVN_PIPELINE");
        return !(e && e[0] == '0');
    }();
    static const int fill_threads = [] {
        const char* e = std::getenv("SVN_FILL_THREADS");
        const int v = e ? std::atoi(e) : 4;
        return v < 1 ? 1 : (v > 16 ? 16 : v);
    }();
    constexpr int64_t kChunkPoints = int64_t(1) << 20;
    ThreadCopy* tc = nullptr;
    if (pipeline_on && !per_point && P >= 2 * kChunkPoints && !g_timing && !prof_enabled())
        tc = thread_copy(m->device);
    if (tc) {
        cudaStream_t cs = tc->s[m->device];
        ArenaScope as(&arena);
        Scratch sc(st);
        unsigned long long* keys = nullptr;
        SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&keys), sizeof(unsigned long long) * M), "cudaMallocAsync(keys)");
        if (!direct) fill(nullptr, reinterpret_cast<float*>(sg.host + o_q), 0, 0);
        SVN_CUDA(cudaMemcpyAsync(sg.dev + o_q, direct ? reinterpret_cast<const uint8_t*>(q01) : sg.host + o_q,
                                 sizeof(float) * nq * M, cudaMemcpyHostToDevice, st),
                 "H2D motions");
        SVN_CUDA(launch_keys_init(keys, M, st), "keys_init kernel");
        ++g_launches;
        int k = 0;
        for (int64_t p0 = 0; p0 < P; p0 += kChunkPoints, ++k) {
            const int64_t n = std::min(kChunkPoints, P - p0);
            const size_t off = sizeof(float) * 3 * static_cast<size_t>(p0), bytes = sizeof(float) * 3 * static_cast<size_t>(n);
            const uint8_t* src = direct ? reinterpret_cast<const uint8_t*>(points) + off : nullptr;
            if (!direct) {  // pageable floats or the reference's double cloud: through the chunk's own
                // part of the pinned block, the copy / double->float cast of a chunk split over a
                // few threads (SVN_FILL_THREADS, default 4: one thread casts 2^24 points in ~50 ms,
                // longer than the GPU needs for them)
                float* dst = reinterpret_cast<float*>(sg.host + off);
                const int T = static_cast<int>(std::min<int64_t>(fill_threads, n / 65536 + 1));
                if (T <= 1) {
                    fill(dst, nullptr, p0, n);
                } else {
                    std::vector<std::thread> pool;
                    const int64_t per = (n + T - 1) / T;
                    for (int t = 1; t < T; ++t) {
                        const int64_t a0 = std::min<int64_t>(n, t * per), a1 = std::min<int64_t>(n, (t + 1) * per);
                        if (a1 > a0) pool.emplace_back([&, a0, a1] { fill(dst + 3 * a0, nullptr, p0 + a0, a1 - a0); });
                    }
                    fill(dst, nullptr, p0, std::min<int64_t>(n, per));
                    for (std::thread& th : pool) th.join();
                }
                src = sg.host + off;
            }
            cudaEvent_t ev = tc->ev[m->device][k % ThreadCopy::kEvents];
            SVN_CUDA(cudaMemcpyAsync(sg.dev + off, src, bytes, cudaMemcpyHostToDevice, cs), "H2D point chunk");
            SVN_CUDA(cudaEventRecord(ev, cs), "cudaEventRecord");
            SVN_CUDA(cudaStreamWaitEvent(st, ev, 0), "cudaStreamWaitEvent");
            const svn_status s = query_dense(m, prec, reinterpret_cast<const float*>(sg.dev + off), n, p0,
                                             reinterpret_cast<const float*>(sg.dev + o_q), M, margin, nullptr, nullptr,
                                             nullptr, nullptr, reinterpret_cast<uint64_t*>(keys), st);
            if (s != SVN_OK) {
                cudaStreamSynchronize(cs);
                cudaStreamSynchronize(st);
                return s;
            }
        }
        SVN_CUDA(launch_keys_finalize(keys, M, margin, reinterpret_cast<float*>(sg.dev + o_min),
                                      reinterpret_cast<int32_t*>(sg.dev + o_arg), sg.dev + o_free, st),
                 "keys_finalize kernel");
        ++g_launches;
        SVN_CUDA(cudaMemcpyAsync(sg.host + o_min, sg.dev + o_min, total - o_min, cudaMemcpyDeviceToHost, st),
                 "D2H min/argmin/free");
        SVN_CUDA(cudaStreamSynchronize(st), "query kernels");
        SVN_CUDA(arena.grow_to_need(), "scratch arena");
        std::memcpy(min_out, sg.host + o_min, sizeof(float) * M);
        std::memcpy(argmin_out, sg.host + o_arg, sizeof(int32_t) * M);
        std::memcpy(free_out, sg.host + o_free, M);
        g_trace_on = false;
        return SVN_OK;
    }
    if (!direct) fill(reinterpret_cast<float*>(sg.host), reinterpret_cast<float*>(sg.host + o_q), 0, P);
    SVN_TRACE(0);
    const bool small = !direct && !per_point && P <= kSmallStagingPoints && M <= 64 && small_staging_enabled();
    if (small && arena.cap > 0 && graphs_enabled() && !g_timing && !prof_enabled() &&
        small_graph(m, prec, P, M, margin, sg, arena, o_q, o_min, o_arg, o_free, st)) {
        SVN_TRACE(4);
    } else {
        ArenaScope as(&arena);
        Scratch sc(st);
        float* dpp = nullptr;
        if (per_point)
            SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&dpp), sizeof(float) * P * M), "cudaMallocAsync");
        // small staged calls (the reference's per-motion predict_min_distance): a kernel pulls the
        // inputs out of the pinned block and the fused finaliser writes (min, argmin, free)
        // straight into it — no DMA copy on the critical path (each costs ~5-10 us of setup)
        if (direct) {
            SVN_CUDA(cudaMemcpyAsync(sg.dev, points, sizeof(float) * 3 * P, cudaMemcpyHostToDevice, st), "H2D points");
            SVN_CUDA(cudaMemcpyAsync(sg.dev + o_q, q01, sizeof(float) * nq * M, cudaMemcpyHostToDevice, st),
                     "H2D motions");
        } else if (small) {
            SVN_CUDA(launch_stage_in(sg.host, sg.dev, o_min, st), "stage_in kernel");
            ++g_launches;
        } else {
            SVN_CUDA(cudaMemcpyAsync(sg.dev, sg.host, o_min, cudaMemcpyHostToDevice, st), "H2D points + motions");
        }
        SVN_TRACE(1);
        uint8_t* const out = small ? sg.host : sg.dev;
        const svn_status s = query_dense(m, prec, reinterpret_cast<const float*>(sg.dev), P, 0,
                                         reinterpret_cast<const float*>(sg.dev + o_q), M, margin,
                                         reinterpret_cast<float*>(out + o_min), reinterpret_cast<int32_t*>(out + o_arg),
                                         out + o_free, dpp, nullptr, st);
        if (s != SVN_OK) return s;
        if (!small)
            SVN_CUDA(cudaMemcpyAsync(sg.host + o_min, sg.dev + o_min, total - o_min, cudaMemcpyDeviceToHost, st),
                     "D2H min/argmin/free");
        if (per_point)
            SVN_CUDA(cudaMemcpyAsync(per_point, dpp, sizeof(float) * P * M, cudaMemcpyDeviceToHost, st), "D2H delta");
        SVN_TRACE(5);
    }
    SVN_CUDA(cudaStreamSynchronize(st), "query kernels");
    SVN_TRACE(6);
    SVN_CUDA(arena.grow_to_need(), "scratch arena");
    std::memcpy(min_out, sg.host + o_min, sizeof(float) * M);
    std::memcpy(argmin_out, sg.host + o_arg, sizeof(int32_t) * M);
    std::memcpy(free_out, sg.host + o_free, M);
    if (g_trace_on) {
        g_trace.lap(7);
        g_trace.done();
        g_trace_on = false;
    }
    return SVN_OK;
}

}  // namespace abi
}  // namespace svn

extern "C" {

SVN_API svn_status svn_query_min_device(const svn_model* m, svn_precision prec, const float* points, int64_t P,
                                        const float* q01, int64_t M, double margin, float* min_out,
                                        int32_t* argmin_out, uint8_t* free_out, float* per_point, void* stream) {
    try {
        if (!min_out || !argmin_out || !free_out) return fail(SVN_ERR_INVALID_ARGUMENT, "query: null output");
        return query_dense(m, prec, points, P, 0, q01, M, margin, min_out, argmin_out, free_out, per_point, nullptr,
                           static_cast<cudaStream_t>(stream));
    } catch (...) {
        return host_exception();
    }
}

SVN_API void svn_set_whole_batch(int64_t M_total, int64_t P_total) {
    g_whole_M = M_total > 0 && P_total > 0 ? M_total : 0;
    g_whole_P = M_total > 0 && P_total > 0 ? P_total : 0;
}

SVN_API svn_status svn_keys_init_device(uint64_t* keys, int64_t M, void* stream) {
    try {
        SVN_CUDA(launch_keys_init(reinterpret_cast<unsigned long long*>(keys), M, static_cast<cudaStream_t>(stream)),
                 "keys_init kernel");
        ++g_launches;
        return SVN_OK;
    } catch (...) {
        return host_exception();
    }
}

SVN_API svn_status svn_query_min_keys_device(const svn_model* m, svn_precision prec, const float* points, int64_t P,
                                             int64_t index_offset, const float* q01, int64_t M, uint64_t* keys,
                                             void* stream) {
    try {
        if (!keys) return fail(SVN_ERR_INVALID_ARGUMENT, "query: null keys");
        return query_dense(m, prec, points, P, index_offset, q01, M, 0.0, nullptr, nullptr, nullptr, nullptr, keys,
                           static_cast<cudaStream_t>(stream));
    } catch (...) {
        return host_exception();
    }
}

SVN_API svn_status svn_keys_finalize_device(const uint64_t* keys, int64_t M, double margin, float* min_out,
                                            int32_t* argmin_out, uint8_t* free_out, void* stream) {
    try {
        SVN_CUDA(launch_keys_finalize(reinterpret_cast<const unsigned long long*>(keys), M, margin, min_out, argmin_out,
                                      free_out, static_cast<cudaStream_t>(stream)),
                 "keys_finalize kernel");
        ++g_launches;
        return SVN_OK;
    } catch (...) {
        return host_exception();
    }
}

SVN_API svn_status svn_query_min(const svn_model* m, svn_precision prec, const float* points, int64_t P,
                                 const float* q01, int64_t M, double margin, float* min_out, int32_t* argmin_out,
                                 uint8_t* free_out, float* per_point) {
    try {
        if (!points || !q01) return fail(SVN_ERR_INVALID_ARGUMENT, "query: null buffer");
        const int nq = m ? 2 * m->dof : 0;
        return query_min_host(m, prec, P, M, margin, points, q01,
                              [&](float* hp, float* hq, int64_t p0, int64_t n) {
                                  if (hp) std::memcpy(hp, points + 3 * p0, sizeof(float) * 3 * n);
                                  if (hq) std::memcpy(hq, q01, sizeof(float) * nq * M);
                              },
                              min_out, argmin_out, free_out, per_point);
    } catch (...) {
        return host_exception();
    }
}

// Margin classification that is exact for every motion at close to the coarse path's cost: the
// whole batch on a fast tensor-core precision, then only the motions whose min lies within that
// precision's stated band of the margin (or is not finite: an fp16 range report) again on
// fp32_split, and what is still within fp32_split's band of the margin on the FP32 path, whose
// class is the reference's bit for bit (collision.cpp:68 on nn.cpp:460-480's result).
SVN_API svn_status svn_query_min_cascade(const svn_model* m, svn_precision coarse, double band_coarse,
                                         double band_split, const float* points, int64_t P, const float* q01,
                                         int64_t M, double margin, float* min_out, int32_t* argmin_out,
                                         uint8_t* free_out, int64_t* stage_motions) {
    try {
        if (!m) return fail(SVN_ERR_INVALID_ARGUMENT, "query: null model");
        if (!(band_coarse >= 0.0) || !(band_split >= 0.0))
            return fail(SVN_ERR_INVALID_ARGUMENT, "cascade: bands must be non-negative");
        if (kernel_kind(m, coarse) == Kind::SIMT)
            return fail(SVN_ERR_INVALID_ARGUMENT, "cascade: the coarse stage must be a tensor-core precision");
        svn_status s = svn_query_min(m, coarse, points, P, q01, M, margin, min_out, argmin_out, free_out, nullptr);
        if (s != SVN_OK) return s;
        if (stage_motions) stage_motions[0] = M, stage_motions[1] = 0, stage_motions[2] = 0;
        const int nq = 2 * m->dof;
        std::vector<int64_t> idx;
        auto near_margin = [&](int64_t i, double band) {
            const double v = static_cast<double>(min_out[i]);
            return !std::isfinite(v) || std::fabs(v - margin) <= band;  // NaN / -inf: a range report, look again
        };
        for (int64_t i = 0; i < M; ++i)
            if (near_margin(i, band_coarse)) idx.push_back(i);
        // one finer stage over the motions in idx, results scattered back
        auto refine = [&](svn_precision prec) -> svn_status {
            const int64_t n = static_cast<int64_t>(idx.size());
            std::vector<float> q(static_cast<size_t>(n) * nq), mn(static_cast<size_t>(n));
            std::vector<int32_t> am(static_cast<size_t>(n));
            std::vector<uint8_t> fr(static_cast<size_t>(n));
            for (int64_t k = 0; k < n; ++k)
                std::memcpy(q.data() + k * nq, q01 + idx[static_cast<size_t>(k)] * nq, sizeof(float) * nq);
            const svn_status r = svn_query_min(m, prec, points, P, q.data(), n, margin, mn.data(), am.data(), fr.data(), nullptr);
            if (r != SVN_OK) return r;
            for (int64_t k = 0; k < n; ++k) {
                const int64_t i = idx[static_cast<size_t>(k)];
                min_out[i] = mn[static_cast<size_t>(k)];
                argmin_out[i] = am[static_cast<size_t>(k)];
                free_out[i] = fr[static_cast<size_t>(k)];
            }
            return SVN_OK;
        };
        if (!idx.empty() && m->has_split && coarse != SVN_PREC_FP32_SPLIT) {
            if ((s = refine(SVN_PREC_FP32_SPLIT)) != SVN_OK) return s;
            if (stage_motions) stage_motions[1] = static_cast<int64_t>(idx.size());
            std::vector<int64_t> rest;
            for (int64_t i : idx)
                if (near_margin(i, band_split)) rest.push_back(i);
            idx.swap(rest);
        }
        if (!idx.empty()) {
            if ((s = refine(SVN_PREC_FP32_EXACT)) != SVN_OK) return s;
            if (stage_motions) stage_motions[2] = static_cast<int64_t>(idx.size());
        }
        return SVN_OK;
    } catch (...) {
        return host_exception();
    }
}

SVN_API svn_status svn_forward_eval(const svn_model* m, svn_precision prec, const float* raw, int64_t B, int64_t cols,
                                    float* out) {
    try {
        if (!m) return fail(SVN_ERR_INVALID_ARGUMENT, "forward: null model");
        if (cols != m->in) return fail(SVN_ERR_INVALID_ARGUMENT, "forward: input width mismatch");
        if (B < 1) return fail(SVN_ERR_INVALID_ARGUMENT, "forward: batch must be non-empty");
        if (!raw || !out) return fail(SVN_ERR_INVALID_ARGUMENT, "forward: null buffer");
        DeviceGuard guard(m->device);
        ensure_pool(m->device);
        cudaStream_t st = thread_stream(m->device);
        float *draw = nullptr, *dout = nullptr;
        {
            Scratch sc(st);
            SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&draw), sizeof(float) * B * cols), "cudaMallocAsync");
            SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&dout), sizeof(float) * B), "cudaMallocAsync");
            SVN_CUDA(cudaMemcpyAsync(draw, raw, sizeof(float) * B * cols, cudaMemcpyHostToDevice, st), "H2D raw");
            svn_status s = forward_rows(m, prec, raw, draw, B, cols, dout, st);
            if (s != SVN_OK) return s;
            SVN_CUDA(cudaMemcpyAsync(out, dout, sizeof(float) * B, cudaMemcpyDeviceToHost, st), "D2H out");
        }
        SVN_CUDA(cudaStreamSynchronize(st), "forward");
        return SVN_OK;
    } catch (...) {
        return host_exception();
    }
}

SVN_API svn_status svn_forward_eval_device(const svn_model* m, svn_precision prec, const float* raw, int64_t B,
                                           int64_t cols, float* out, void* stream) {
    try {
        if (!m) return fail(SVN_ERR_INVALID_ARGUMENT, "forward: null model");
        if (cols != m->in) return fail(SVN_ERR_INVALID_ARGUMENT, "forward: input width mismatch");
        if (B < 1) return fail(SVN_ERR_INVALID_ARGUMENT, "forward: batch must be non-empty");
        DeviceGuard guard(m->device);
        ensure_pool(m->device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        // segmenting needs the q columns on the host
        std::vector<float> host(static_cast<size_t>(B * cols));
        SVN_CUDA(cudaMemcpyAsync(host.data(), raw, sizeof(float) * B * cols, cudaMemcpyDeviceToHost, st), "D2H raw");
        SVN_CUDA(cudaStreamSynchronize(st), "D2H raw");
        return forward_rows(m, prec, host.data(), raw, B, cols, out, st);
    } catch (...) {
        return host_exception();
    }
}

SVN_API svn_status svn_predict_min_distance(const svn_model* m, svn_precision prec, const double* cloud, int64_t P,
                                            const double* q0, const double* q1, int32_t dof, double* min_out,
                                            int32_t* argmin_out) {
    try {
        if (!m) return fail(SVN_ERR_INVALID_ARGUMENT, "predict_min_distance: null model");
        if (P < 1) return fail(SVN_ERR_INVALID_ARGUMENT, "predict_min_distance: empty point cloud");
        if (3 + 2 * dof != m->in) return fail(SVN_ERR_INVALID_ARGUMENT, "predict_min_distance: motion dof does not match model");
        if (!cloud || !q0 || !q1 || !min_out || !argmin_out)
            return fail(SVN_ERR_INVALID_ARGUMENT, "predict_min_distance: null buffer");
        // nn.cpp:469-473: every coordinate and joint value is cast to float (straight into the
        // pinned staging block)
        float mn = 0.f;
        int32_t idx = 0;
        uint8_t fr = 0;
        svn_status s = query_min_host(m, prec, P, 1, 0.0, nullptr, nullptr,
                                      [&](float* hp, float* hq, int64_t p0, int64_t n) {
                                          if (hp) cvt_f64_f32(hp, cloud + 3 * p0, 3 * n);
                                          if (hq) {
                                              for (int i = 0; i < dof; ++i) hq[i] = static_cast<float>(q0[i]);
                                              for (int i = 0; i < dof; ++i) hq[dof + i] = static_cast<float>(q1[i]);
                                          }
                                      },
                                      &mn, &idx, &fr, nullptr);
        if (s != SVN_OK) return s;
        *min_out = static_cast<double>(mn);
        *argmin_out = idx;
        return SVN_OK;
    } catch (...) {
        return host_exception();
    }
}

SVN_API svn_status svn_eval_grid(const svn_model* m, svn_precision prec, const double* origin, double voxel_size,
                                 const int32_t* dims, const double* q0, const double* q1, int32_t dof, float* values) {
    try {
        if (!m) return fail(SVN_ERR_INVALID_ARGUMENT, "reconstruct: null model");
        if (!origin || !dims || !q0 || !q1 || !values) return fail(SVN_ERR_INVALID_ARGUMENT, "reconstruct: null buffer");
        if (3 + 2 * dof != m->in)
            return fail(SVN_ERR_INVALID_ARGUMENT, "reconstruct: q0/q1 must have one angle per joint");
        if (dims[0] < 1 || dims[1] < 1 || dims[2] < 1 || !(voxel_size > 0))
            return fail(SVN_ERR_INVALID_ARGUMENT, "reconstruct: empty grid");
        const int64_t P = static_cast<int64_t>(dims[0]) * dims[1] * dims[2];
        DeviceGuard guard(m->device);
        ensure_pool(m->device);
        cudaStream_t st = thread_stream(m->device);
        std::vector<float> q(static_cast<size_t>(2 * dof));
        for (int i = 0; i < dof; ++i) q[i] = static_cast<float>(q0[i]);
        for (int i = 0; i < dof; ++i) q[dof + i] = static_cast<float>(q1[i]);
        {
            Scratch sc(st);
            float *dp = nullptr, *dq = nullptr, *dmin = nullptr, *dvals = nullptr;
            int32_t* darg = nullptr;
            uint8_t* dfree = nullptr;
            SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&dp), sizeof(float) * 3 * P), "cudaMallocAsync");
            SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&dq), sizeof(float) * q.size()), "cudaMallocAsync");
            SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&dmin), sizeof(float)), "cudaMallocAsync");
            SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&darg), sizeof(int32_t)), "cudaMallocAsync");
            SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&dfree), 1), "cudaMallocAsync");
            SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&dvals), sizeof(float) * P), "cudaMallocAsync");
            SVN_CUDA(cudaMemcpyAsync(dq, q.data(), sizeof(float) * q.size(), cudaMemcpyHostToDevice, st), "H2D q");
            SVN_CUDA(launch_grid_points(origin, voxel_size, dims, dp, st), "grid_points kernel");
            ++g_launches;
            svn_status s = query_dense(m, prec, dp, P, 0, dq, 1, 0.0, dmin, darg, dfree, dvals, nullptr, st);
            if (s != SVN_OK) return s;
            SVN_CUDA(cudaMemcpyAsync(values, dvals, sizeof(float) * P, cudaMemcpyDeviceToHost, st), "D2H values");
            SVN_CUDA(cudaStreamSynchronize(st), "eval_grid");
        }
        return SVN_OK;
    } catch (...) {
        return host_exception();
    }
}


}  // extern "C"
