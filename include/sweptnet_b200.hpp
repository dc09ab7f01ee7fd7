// sweptnet_b200.hpp — header-only C++ host API over the C-ABI (include/sweptnet_b200.h).
//
// Mirrors the reference's inference interface (/root/reference/proj/include/sweptnet/nn.hpp
// and collision.hpp) with std containers instead of Eigen, so it compiles anywhere the
// C-ABI library does:
//   init_model            nn.hpp:80-81     -> Model::init
//   load_checkpoint       nn.hpp:168       -> Model::load_checkpoint
//   forward_eval<float>   nn.hpp:92-93     -> forward_eval
//   predict_min_distance  nn.hpp:162-163   -> predict_min_distance
//   ProxyEvaluator        collision.hpp:45 -> batched_proxy (one GPU call for all motions)
// Errors are rethrown with the reference's exception types and messages:
// std::invalid_argument for argument errors (nn.cpp:98-99, 462, 465), and IoError /
// FormatError / TruncationError / VersionError (errors.hpp:8-27) for checkpoints.
#pragma once

#include <array>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sweptnet_b200.h"

namespace sweptnet_b200 {

struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct FormatError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct TruncationError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct VersionError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(svn_status s) {
    if (s == SVN_OK) return;
    const std::string msg = svn_last_error();
    switch (s) {
        case SVN_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case SVN_ERR_IO: throw IoError(msg);
        case SVN_ERR_FORMAT: throw FormatError(msg);
        case SVN_ERR_TRUNCATION: throw TruncationError(msg);
        case SVN_ERR_VERSION: throw VersionError(msg);
        default: throw std::runtime_error(msg);
    }
}

using Vec3 = std::array<double, 3>;

// Motion (sweptvol.hpp:14-18): start and goal joint configurations.
struct Motion {
    std::vector<double> q0, q1;
};

enum class Precision {
    BF16 = SVN_PREC_BF16,
    FP32 = SVN_PREC_FP32,
    FP32_EXACT = SVN_PREC_FP32_EXACT,
    FP32_SPLIT = SVN_PREC_FP32_SPLIT,
    FP16 = SVN_PREC_FP16
};

// A layer program; fig2() is the reference network (nn.hpp:11-15).
struct Program {
    int width = 0, dof = 0;
    std::vector<svn_layer> layers;
    svn_model_desc desc() const { return svn_model_desc{static_cast<int32_t>(layers.size()), width, dof, layers.data()}; }
    static Program fig2(int n_blocks, int width, int dof) {
        Program p{width, dof, {}};
        p.layers.push_back(svn_layer{1, 0, 0, 0});
        for (int i = 0; i < n_blocks; ++i) p.layers.push_back(svn_layer{1, 1, 1, 1});
        return p;
    }
    static Program plain(int hidden, int width, int dof) {
        Program p{width, dof, {}};
        p.layers.push_back(svn_layer{1, 1, 0, 0});
        for (int i = 1; i < hidden; ++i) p.layers.push_back(svn_layer{0, 1, 0, 0});
        return p;
    }
    static Program deepsdf(int hidden, int width, int dof, int skip_at = 4) {
        Program p{width, dof, {}};
        p.layers.push_back(svn_layer{1, 1, 0, 0});
        for (int i = 1; i < hidden; ++i) p.layers.push_back(svn_layer{i == skip_at ? 1 : 0, 1, 0, 0});
        return p;
    }
};

class Model {
public:
    Model(const Program& prog, const std::vector<float>& params, int device = 0) : prog_(prog) {
        const svn_model_desc d = prog_.desc();
        svn_model* h = nullptr;
        check(svn_model_create(&d, params.data(), static_cast<int64_t>(params.size()), device, &h));
        h_.reset(h, svn_model_destroy);
    }
    // init_model (nn.cpp:57-93); bound_mode 0 = +-1/sqrt(fan_in), 1 = He-uniform.
    static Model init(const Program& prog, uint64_t seed, int bound_mode = 0, int device = 0) {
        const svn_model_desc d = prog.desc();
        std::vector<float> p(static_cast<size_t>(svn_param_count(&d)));
        check(svn_init_params(&d, seed, bound_mode, p.data()));
        return Model(prog, p, device);
    }
    static Model load_checkpoint(const std::string& path, int device = 0) {
        svn_model* h = nullptr;
        check(svn_model_load_checkpoint(path.c_str(), device, &h));
        Model m;
        m.h_.reset(h, svn_model_destroy);
        int32_t width = 0, dof = 0, n = 0;
        check(svn_model_get_program(h, &width, &dof, &n, nullptr, 0));
        m.prog_ = Program{width, dof, std::vector<svn_layer>(static_cast<size_t>(n))};
        check(svn_model_get_program(h, &width, &dof, &n, m.prog_.layers.data(), n));
        return m;
    }
    const svn_model* handle() const { return h_.get(); }
    int dof() const { return prog_.dof; }
    const Program& program() const { return prog_; }

private:
    Model() = default;
    Program prog_;
    std::shared_ptr<svn_model> h_;
};

// forward_eval<float> (nn.cpp:95-130): raw row-major [rows x (3 + 2*dof)].
inline std::vector<float> forward_eval(const Model& m, const std::vector<float>& raw, long rows, long cols,
                                       Precision prec = Precision::FP32_EXACT) {
    std::vector<float> out(static_cast<size_t>(rows > 0 ? rows : 0));
    check(svn_forward_eval(m.handle(), static_cast<svn_precision>(prec), raw.data(), rows, cols, out.data()));
    return out;
}

// predict_min_distance (nn.cpp:460-480): (double(min delta), argmin point index).
inline std::pair<double, int> predict_min_distance(const Model& m, const std::vector<Vec3>& cloud, const Motion& mo,
                                                   Precision prec = Precision::FP32_EXACT) {
    if (mo.q0.size() != mo.q1.size()) throw std::invalid_argument("predict_min_distance: motion dof does not match model");
    double mn = 0.0;
    int32_t idx = 0;
    check(svn_predict_min_distance(m.handle(), static_cast<svn_precision>(prec),
                                   cloud.empty() ? nullptr : cloud.front().data(), static_cast<int64_t>(cloud.size()),
                                   mo.q0.data(), mo.q1.data(), static_cast<int32_t>(mo.q0.size()), &mn, &idx));
    return {mn, idx};
}

// Batched proxy for gcc_nn_search_impl (collision.cpp:55-107): every motion of a scene in
// one GPU call; proxy(j) then returns the cached predict_min_distance(...).first.
inline std::function<double(int)> batched_proxy(const Model& m, const std::vector<Vec3>& cloud,
                                                const std::vector<Motion>& motions,
                                                Precision prec = Precision::BF16) {
    if (cloud.empty()) throw std::invalid_argument("predict_min_distance: empty point cloud");
    std::vector<float> pts;
    pts.reserve(cloud.size() * 3);
    for (const Vec3& p : cloud)
        for (double c : p) pts.push_back(static_cast<float>(c));
    const size_t dof = motions.empty() ? 0 : motions.front().q0.size();
    std::vector<float> q;
    for (const Motion& mo : motions) {
        if (mo.q0.size() != dof || mo.q1.size() != dof)
            throw std::invalid_argument("predict_min_distance: motion dof does not match model");
        for (double v : mo.q0) q.push_back(static_cast<float>(v));
        for (double v : mo.q1) q.push_back(static_cast<float>(v));
    }
    const size_t M = motions.size();
    auto mins = std::make_shared<std::vector<float>>(M);
    if (M) {
        std::vector<int32_t> am(M);
        std::vector<uint8_t> fr(M);
        check(svn_query_min(m.handle(), static_cast<svn_precision>(prec), pts.data(), static_cast<int64_t>(cloud.size()),
                            q.data(), static_cast<int64_t>(M), 0.0, mins->data(), am.data(), fr.data(), nullptr));
    }
    return [mins](int j) { return static_cast<double>((*mins)[static_cast<size_t>(j)]); };
}

// The classification step of the callers (collision.cpp:68, bench.cpp:108) for a batch of motions,
// exact for every motion (svn_query_min_cascade): `coarse` (FP16 or BF16) for the batch, FP32_SPLIT
// for the motions within band_coarse of the margin, the FP32 path for those within band_split.
struct CascadeResult {
    std::vector<float> min;
    std::vector<int32_t> argmin;
    std::vector<uint8_t> free;   // == the reference's double(min) > margin, motion by motion
    int64_t stage_motions[3];    // motions evaluated on {coarse, FP32_SPLIT, FP32}
};
inline CascadeResult classify_motions(const Model& m, const std::vector<float>& points_xyz,
                                      const std::vector<float>& q01, double margin, double band_coarse,
                                      double band_split, Precision coarse = Precision::FP16) {
    const int64_t P = static_cast<int64_t>(points_xyz.size() / 3);
    const int64_t M = m.dof() > 0 ? static_cast<int64_t>(q01.size()) / (2 * m.dof()) : 0;
    CascadeResult r;
    r.min.resize(static_cast<size_t>(M));
    r.argmin.resize(static_cast<size_t>(M));
    r.free.resize(static_cast<size_t>(M));
    check(svn_query_min_cascade(m.handle(), static_cast<svn_precision>(coarse), band_coarse, band_split,
                                points_xyz.data(), P, q01.data(), M, margin, r.min.data(), r.argmin.data(),
                                r.free.data(), r.stage_motions));
    return r;
}

// The calls made while a WholeBatch is alive are shards (motion ranges or point chunks) of one
// batch of that shape and take its tile shape: the same bits whatever the split, in every
// precision (svn_set_whole_batch; thread-local).  MultiModel does this itself.
struct WholeBatch {
    WholeBatch(int64_t motions, int64_t points) { svn_set_whole_batch(motions, points); }
    ~WholeBatch() { svn_set_whole_batch(0, 0); }
    WholeBatch(const WholeBatch&) = delete;
    WholeBatch& operator=(const WholeBatch&) = delete;
};

// Several GPUs of this box from one process (svn_multi_*): one model copy and one worker
// thread per device.  query_min shards motions (no communication) or, for batches with
// fewer motions than devices, points (one NCCL u64 MIN all-reduce); bit-identical to Model.
enum class Shard { AUTO = SVN_SHARD_AUTO, MOTIONS = SVN_SHARD_MOTIONS, POINTS = SVN_SHARD_POINTS };

struct MinResult {
    std::vector<float> min;
    std::vector<int32_t> argmin;
    std::vector<uint8_t> free;
};

class MultiModel {
public:
    MultiModel(const Program& prog, const std::vector<float>& params, const std::vector<int32_t>& devices)
        : prog_(prog) {
        const svn_model_desc d = prog_.desc();
        svn_multi* h = nullptr;
        check(svn_multi_create(&d, params.data(), static_cast<int64_t>(params.size()), devices.data(),
                               static_cast<int32_t>(devices.size()), &h));
        h_.reset(h, svn_multi_destroy);
    }
    // points float [P x 3], q01 float [M x 2 dof] (q0 | q1), as svn_query_min.
    MinResult query_min(const std::vector<float>& points, const std::vector<float>& q01, double margin,
                        Precision prec = Precision::BF16, Shard shard = Shard::AUTO) const {
        const int64_t P = static_cast<int64_t>(points.size() / 3), M = static_cast<int64_t>(q01.size() / (2 * prog_.dof));
        MinResult r{std::vector<float>(static_cast<size_t>(M)), std::vector<int32_t>(static_cast<size_t>(M)),
                    std::vector<uint8_t>(static_cast<size_t>(M))};
        check(svn_query_min_multi(h_.get(), static_cast<svn_precision>(prec), points.data(), P, q01.data(), M, margin,
                                  static_cast<svn_shard_mode>(shard), r.min.data(), r.argmin.data(), r.free.data()));
        return r;
    }
    // Keep one scene's cloud resident on every device (svn_multi_set_scene); an empty vector
    // drops it.  query_min_scene then moves only the motions in and the results out.
    void set_scene(const std::vector<float>& points) {
        check(svn_multi_set_scene(h_.get(), points.empty() ? nullptr : points.data(), static_cast<int64_t>(points.size() / 3)));
        scene_points_ = static_cast<int64_t>(points.size() / 3);
    }
    MinResult query_min_scene(const std::vector<float>& q01, double margin, Precision prec = Precision::BF16,
                              Shard shard = Shard::AUTO) const {
        const int64_t M = static_cast<int64_t>(q01.size() / (2 * prog_.dof));
        MinResult r{std::vector<float>(static_cast<size_t>(M)), std::vector<int32_t>(static_cast<size_t>(M)),
                    std::vector<uint8_t>(static_cast<size_t>(M))};
        check(svn_query_min_multi(h_.get(), static_cast<svn_precision>(prec), nullptr, scene_points_, q01.data(), M,
                                  margin, static_cast<svn_shard_mode>(shard), r.min.data(), r.argmin.data(),
                                  r.free.data()));
        return r;
    }
    // query_min with the class equal to the FP32 path's for every motion (svn_query_min_cascade_multi):
    // bands = the stated bounds of `coarse` and of FP32_SPLIT; stage_motions as in the C entry.
    MinResult query_min_cascade(const std::vector<float>& points, const std::vector<float>& q01, double margin,
                                double band_coarse, double band_split, Precision coarse = Precision::FP16,
                                std::array<int64_t, 3>* stage_motions = nullptr) const {
        const int64_t P = static_cast<int64_t>(points.size() / 3), M = static_cast<int64_t>(q01.size() / (2 * prog_.dof));
        MinResult r{std::vector<float>(static_cast<size_t>(M)), std::vector<int32_t>(static_cast<size_t>(M)),
                    std::vector<uint8_t>(static_cast<size_t>(M))};
        check(svn_query_min_cascade_multi(h_.get(), static_cast<svn_precision>(coarse), band_coarse, band_split,
                                          points.data(), P, q01.data(), M, margin, r.min.data(), r.argmin.data(),
                                          r.free.data(), stage_motions ? stage_motions->data() : nullptr));
        return r;
    }
    int devices() const { return svn_multi_device_count(h_.get()); }

private:
    Program prog_;
    std::shared_ptr<svn_multi> h_;
    int64_t scene_points_ = 0;
};

}  // namespace sweptnet_b200
