// abi_gcc.cu — C-ABI: the GPU geometric checker and the whole of Alg. 1 (gcc_nn_search).
#include "abi_internal.cuh"

using namespace svn;
using namespace svn::abi;

namespace svn {
namespace abi {

svn_status gcc_args(const svn_robot_desc* r, int32_t steps, GccArgs& a) {
    if (!r || !r->joints || !r->capsules) return fail(SVN_ERR_INVALID_ARGUMENT, "robot: null descriptor");
    if (r->dof < 1 || r->dof > kGccMaxDof) return fail(SVN_ERR_INVALID_ARGUMENT, "robot: dof must be >= 1");
    if (r->n_capsules < 1 || r->n_capsules > kGccMaxCaps)
        return fail(SVN_ERR_INVALID_ARGUMENT, "robot: every link needs at least one capsule");
    if (steps < 2) return fail(SVN_ERR_INVALID_ARGUMENT, "discretize: steps must be >= 2");
    a = GccArgs{};
    a.dof = r->dof;
    a.ncap = r->n_capsules;
    a.steps = steps;
    for (int k = 0; k < 12; ++k) a.base[k] = r->base_pose ? r->base_pose[k] : ((k % 4) == (k / 4) ? 1.0 : 0.0);
    for (int j = 0; j < r->dof; ++j)
        for (int k = 0; k < 3; ++k) {
            a.joints[j].axis[k] = r->joints[j].axis[k];
            a.joints[j].offset[k] = r->joints[j].offset[k];
        }
    int prev = -1;
    for (int c = 0; c < r->n_capsules; ++c) {
        const svn_capsule& cap = r->capsules[c];
        if (cap.link < prev || cap.link >= r->dof || !(cap.radius > 0))
            return fail(SVN_ERR_INVALID_ARGUMENT, "robot: link capsule invalid");
        prev = cap.link;
        a.caps[c].link = cap.link;
        for (int k = 0; k < 3; ++k) {
            a.caps[c].a[k] = cap.a[k];
            a.caps[c].b[k] = cap.b[k];
        }
        a.caps[c].radius = cap.radius;
    }
    if (gcc_smem_bytes(steps, r->n_capsules) > 220 * 1024)
        return fail(SVN_ERR_UNSUPPORTED, "gcc: steps x capsules exceeds shared memory");
    return SVN_OK;
}

// The checker on device buffers; early_exit = gcc_clearance semantics (a motion stops as soon
// as one point is within the margin; its distance is then a partial minimum <= margin).
svn_status gcc_run(const svn_robot_desc* robot, const double* points, int64_t P, const double* q01, int64_t M,
                          int32_t steps, double margin, bool early_exit, double* dist_out, uint8_t* free_out,
                          cudaStream_t st) {
    NvtxRange nvtx(early_exit ? "svn gcc (clearance)" : "svn gcc (min distance)");
    if (P < 1) return fail(SVN_ERR_INVALID_ARGUMENT, "gcc_min_distance: empty point cloud");
    if (M < 1) return SVN_OK;
    GccArgs a;
    svn_status s = gcc_args(robot, steps, a);
    if (s != SVN_OK) return s;
    Scratch sc(st);
    SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&a.keys), sizeof(unsigned long long) * M), "cudaMallocAsync");
    a.points = points;
    a.P = P;
    a.q01 = q01;
    a.M = M;
    a.points_per_chunk = 2048;  // 512..32768 measured within 4 % at c3 size: the scan dominates
    a.chunks = (P + a.points_per_chunk - 1) / a.points_per_chunk;
    a.early_exit = early_exit ? 1 : 0;
    a.margin = margin;
    if (early_exit) {
        SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&a.hit), sizeof(unsigned int) * M), "cudaMallocAsync");
        SVN_CUDA(cudaMemsetAsync(a.hit, 0, sizeof(unsigned int) * M, st), "memset hit");
    }
    SVN_CUDA(launch_gcc(a, margin, dist_out, free_out, st), "gcc kernel");
    g_launches += 3;
    return SVN_OK;
}

// Host buffers in and out, on the calling thread's stream.
svn_status gcc_host(const svn_robot_desc* robot, const double* points, int64_t P, const double* q01, int64_t M,
                           int32_t steps, double margin, bool early_exit, int32_t device, double* dist_out,
                           uint8_t* free_out) {
    if (P < 1) return fail(SVN_ERR_INVALID_ARGUMENT, "gcc_min_distance: empty point cloud");
    if (M < 1) return SVN_OK;
    if (!robot || !points || !q01 || !dist_out || !free_out)
        return fail(SVN_ERR_INVALID_ARGUMENT, "gcc_min_distance: null buffer");
    DeviceGuard guard(device);
    ensure_pool(device);
    cudaStream_t st = thread_stream(device);
    const int64_t nq = 2 * static_cast<int64_t>(robot->dof);
    {
        Scratch sc(st);
        double *dp = nullptr, *dq = nullptr, *dd = nullptr;
        uint8_t* df = nullptr;
        SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&dp), sizeof(double) * 3 * P), "cudaMallocAsync");
        SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&dq), sizeof(double) * nq * M), "cudaMallocAsync");
        SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&dd), sizeof(double) * M), "cudaMallocAsync");
        SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&df), M), "cudaMallocAsync");
        SVN_CUDA(cudaMemcpyAsync(dp, points, sizeof(double) * 3 * P, cudaMemcpyHostToDevice, st), "H2D points");
        SVN_CUDA(cudaMemcpyAsync(dq, q01, sizeof(double) * nq * M, cudaMemcpyHostToDevice, st), "H2D motions");
        svn_status s = gcc_run(robot, dp, P, dq, M, steps, margin, early_exit, dd, df, st);
        if (s != SVN_OK) return s;
        SVN_CUDA(cudaMemcpyAsync(dist_out, dd, sizeof(double) * M, cudaMemcpyDeviceToHost, st), "D2H dist");
        SVN_CUDA(cudaMemcpyAsync(free_out, df, M, cudaMemcpyDeviceToHost, st), "D2H free");
    }
    SVN_CUDA(cudaStreamSynchronize(st), "gcc");
    return SVN_OK;
}

}  // namespace abi
}  // namespace svn

extern "C" {
SVN_API svn_status svn_gcc_min_distance_device(const svn_robot_desc* robot, const double* points, int64_t P,
                                               const double* q01, int64_t M, int32_t steps, double margin,
                                               double* dist_out, uint8_t* free_out, void* stream) {
    try {
        return gcc_run(robot, points, P, q01, M, steps, margin, false, dist_out, free_out,
                       static_cast<cudaStream_t>(stream));
    } catch (...) {
        return host_exception();
    }
}

SVN_API svn_status svn_gcc_min_distance(const svn_robot_desc* robot, const double* points, int64_t P,
                                        const double* q01, int64_t M, int32_t steps, double margin, int32_t device,
                                        double* dist_out, uint8_t* free_out) {
    try {
        return gcc_host(robot, points, P, q01, M, steps, margin, false, device, dist_out, free_out);
    } catch (...) {
        return host_exception();
    }
}

// Alg. 1 (collision.cpp:55-107) with both callables on the GPU; see the header.
SVN_API svn_status svn_gcc_nn_search(const svn_model* m, svn_precision prec, const svn_robot_desc* robot,
                                     const double* cloud, int64_t P, const double* q01, int64_t M, int32_t steps,
                                     double margin, int32_t batch, svn_search_result* out) {
    try {
        NvtxRange nvtx("svn gcc_nn_search (Alg. 1)");
        using clk = std::chrono::steady_clock;
        auto secs = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); };
        if (!m || !robot || !out) return fail(SVN_ERR_INVALID_ARGUMENT, "gcc_nn_search: null argument");
        if (P < 1) return fail(SVN_ERR_INVALID_ARGUMENT, "predict_min_distance: empty point cloud");
        if (robot->dof != m->dof) return fail(SVN_ERR_INVALID_ARGUMENT, "predict_min_distance: motion dof does not match model");
        if (M < 1 || !cloud || !q01) {
            *out = svn_search_result{0, -1, 0.0, 0, 0, 0.0, 0.0, 0.0};
            if (M < 1) return SVN_OK;
            return fail(SVN_ERR_INVALID_ARGUMENT, "gcc_nn_search: null buffer");
        }
        const int nq = 2 * m->dof;
        const int64_t B = batch > 0 ? batch : 64;
        svn_search_result r{0, -1, 0.0, 0, 0, 0.0, 0.0, 0.0};
        const auto t_start = clk::now();

        // every proxy at once: predict_min_distance casts points and q to float (nn.cpp:466-474)
        std::vector<float> pf(static_cast<size_t>(3 * P)), qf(static_cast<size_t>(nq * M));
        for (int64_t i = 0; i < 3 * P; ++i) pf[static_cast<size_t>(i)] = static_cast<float>(cloud[i]);
        for (int64_t i = 0; i < nq * M; ++i) qf[static_cast<size_t>(i)] = static_cast<float>(q01[i]);
        std::vector<float> mn(static_cast<size_t>(M));
        std::vector<int32_t> am(static_cast<size_t>(M));
        std::vector<uint8_t> fr(static_cast<size_t>(M));
        svn_status s = svn_query_min(m, prec, pf.data(), P, qf.data(), M, margin, mn.data(), am.data(), fr.data(), nullptr);
        if (s != SVN_OK) return s;
        const auto t_proxy = clk::now();
        r.proxy_seconds = secs(t_start, t_proxy);

        // the sequential algorithm's checker order
        std::vector<int64_t> order;
        order.reserve(static_cast<size_t>(M));
        for (int64_t j = 0; j < M; ++j)
            if (static_cast<double>(mn[static_cast<size_t>(j)]) > margin) order.push_back(j);
        const int64_t n_first = static_cast<int64_t>(order.size());
        std::vector<int64_t> rest;
        for (int64_t j = 0; j < M; ++j)
            if (!(static_cast<double>(mn[static_cast<size_t>(j)]) > margin)) rest.push_back(j);
        std::stable_sort(rest.begin(), rest.end(), [&](int64_t a, int64_t b) {
            return static_cast<double>(mn[static_cast<size_t>(a)]) > static_cast<double>(mn[static_cast<size_t>(b)]);
        });
        order.insert(order.end(), rest.begin(), rest.end());

        // checker in that order, batch by batch, until the first free motion
        std::vector<double> qb(static_cast<size_t>(B * nq)), db(static_cast<size_t>(B));
        std::vector<uint8_t> fb(static_cast<size_t>(B));
        for (int64_t pos = 0; pos < M && !r.found; pos += B) {
            const int64_t nb = std::min<int64_t>(B, M - pos);
            for (int64_t i = 0; i < nb; ++i)
                std::memcpy(qb.data() + i * nq, q01 + order[static_cast<size_t>(pos + i)] * nq, sizeof(double) * nq);
            // gcc_clearance semantics: a colliding motion stops at its first point within the margin
            s = gcc_host(robot, cloud, P, qb.data(), nb, steps, margin, true, m->device, db.data(), fb.data());
            if (s != SVN_OK) return s;
            for (int64_t i = 0; i < nb; ++i) {
                if (!fb[static_cast<size_t>(i)]) continue;
                const int64_t k = pos + i;  // position in the visiting order
                r.found = 1;
                r.motion_index = static_cast<int32_t>(order[static_cast<size_t>(k)]);
                r.certified_distance = db[static_cast<size_t>(i)];
                r.exact_checks = k + 1;
                r.nn_checks = k < n_first ? static_cast<int64_t>(r.motion_index) + 1 : M;
                break;
            }
        }
        if (!r.found) {
            r.exact_checks = M;
            r.nn_checks = M;
        }
        const auto t_end = clk::now();
        r.exact_seconds = secs(t_proxy, t_end);
        r.total_seconds = secs(t_start, t_end);
        *out = r;
        return SVN_OK;
    } catch (...) {
        return host_exception();
    }
}


}  // extern "C"
