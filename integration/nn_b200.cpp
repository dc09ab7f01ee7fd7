// src/nn_b200.cpp — the reference-side drop-in (add to proj/src, build with -DSWEPTNET_B200 and
// integration/sweptnet_b200.patch applied).  Replaces the bodies of forward_eval<float>
// (nn.hpp:92-93, nn.cpp:95-130) and predict_min_distance (nn.hpp:162-163, nn.cpp:460-480) with
// calls into the B200 C-ABI (include/sweptnet_b200.h); forward_eval<double> and everything else
// in nn.cpp keep their CPU bodies.  Errors come back as the reference's own exception types and
// texts (std::invalid_argument, nn.cpp:98-99,462,465).
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <unordered_map>
#include <vector>

#include "sweptnet/nn.hpp"
#include "sweptnet_b200.h"

namespace sweptnet {
namespace {

void check(svn_status s) {
    if (s == SVN_OK) return;
    if (s == SVN_ERR_INVALID_ARGUMENT) throw std::invalid_argument(svn_last_error());
    throw std::runtime_error(svn_last_error());
}

// SVCKPT01 body order (nn.cpp:507-520) == the svn parameter layout of the Fig. 2 program.
std::vector<float> flatten(const Mlp& m) {
    std::vector<float> p;
    auto put = [&](const float* d, long n) { p.insert(p.end(), d, d + n); };
    put(m.norm_shift.data(), m.norm_shift.size());
    put(m.norm_scale.data(), m.norm_scale.size());
    put(m.input_weight.data(), m.input_weight.size());  // column-major, as stored
    put(m.input_bias.data(), m.input_bias.size());
    for (const auto& b : m.blocks) {
        put(b.weight.data(), b.weight.size());
        put(b.bias.data(), b.bias.size());
        put(b.gamma.data(), b.gamma.size());
        put(b.beta.data(), b.beta.size());
        put(b.running_mean.data(), b.running_mean.size());
        put(b.running_var.data(), b.running_var.size());
    }
    put(m.output_weight.data(), m.output_weight.size());
    p.push_back(m.output_bias);
    return p;
}

// Cheap per-call identity of a model: its tensors' addresses and sizes plus a strided sample
// of every tensor's values (~1/64 of the words).  An eval-mode Mlp is immutable (nn.hpp:84-87);
// training rewrites every parameter per Adam step (nn.cpp:267-300), which the sample sees, and
// Eigen reallocates on resize, which the addresses see.  The full upload happens only when the
// fingerprint changes — not on every per-motion call of gcc_nn_search (collision.cpp:124).
uint64_t fingerprint(const Mlp& m) {
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](uint64_t v) { h = (h ^ v) * 1099511628211ull; };
    auto tensor = [&](const float* d, long n) {
        mix(reinterpret_cast<uintptr_t>(d));
        mix(static_cast<uint64_t>(n));
        for (long i = 0; i < n; i += 64) {
            uint32_t w;
            std::memcpy(&w, d + i, 4);
            mix(w);
        }
        if (n) {
            uint32_t w;
            std::memcpy(&w, d + n - 1, 4);
            mix(w);
        }
    };
    tensor(m.norm_shift.data(), m.norm_shift.size());
    tensor(m.norm_scale.data(), m.norm_scale.size());
    tensor(m.input_weight.data(), m.input_weight.size());
    tensor(m.input_bias.data(), m.input_bias.size());
    for (const auto& b : m.blocks) {
        tensor(b.weight.data(), b.weight.size());
        tensor(b.bias.data(), b.bias.size());
        tensor(b.gamma.data(), b.gamma.size());
        tensor(b.beta.data(), b.beta.size());
        tensor(b.running_mean.data(), b.running_mean.size());
        tensor(b.running_var.data(), b.running_var.size());
    }
    tensor(m.output_weight.data(), m.output_weight.size());
    tensor(&m.output_bias, 1);
    return h;
}

// The arithmetic of the drop-in, read once from SWEPTNET_B200_PRECISION: "fp32_exact" (default:
// the reference's float results bit for bit), "fp32_split" (fp32-grade on the tensor cores,
// within 1e-5 on the reference's Fig. 2 networks), "fp16" (tensor cores at the bf16 rate, a
// bound about 8 times tighter than bf16: 0.0032 on Fig. 2 5x512) or "bf16" (its stated bound).
svn_precision precision() {
    static const svn_precision p = [] {
        const char* e = std::getenv("SWEPTNET_B200_PRECISION");
        if (e && std::strcmp(e, "bf16") == 0) return SVN_PREC_BF16;
        if (e && std::strcmp(e, "fp16") == 0) return SVN_PREC_FP16;
        if (e && std::strcmp(e, "fp32_split") == 0) return SVN_PREC_FP32_SPLIT;
        return SVN_PREC_FP32_EXACT;
    }();
    return p;
}

const svn_model* device_model(const Mlp& m) {
    static std::mutex mu;  // callers are parallel_for workers (bench.cpp:156,193)
    static std::unordered_map<const Mlp*, std::pair<uint64_t, svn_model*>> cache;
    const uint64_t h = fingerprint(m);
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(&m);
    if (it != cache.end() && it->second.first == h) return it->second.second;
    const std::vector<float> p = flatten(m);
    std::vector<svn_layer> layers(static_cast<size_t>(m.n_blocks) + 1, svn_layer{1, 1, 1, 1});
    layers[0] = svn_layer{1, 0, 0, 0};
    const svn_model_desc d{m.n_blocks + 1, m.block_dim, m.dof(), layers.data()};
    svn_model* dm = nullptr;
    check(svn_model_create(&d, p.data(), static_cast<int64_t>(p.size()), 0, &dm));
    if (it != cache.end()) svn_model_destroy(it->second.second);
    cache[&m] = {h, dm};
    return dm;
}

}  // namespace

template <>
MlpT<float>::Vec forward_eval<float>(const MlpT<float>& model, const MlpT<float>::Mat& raw) {
    if (raw.cols() != model.input_dim) throw std::invalid_argument("forward: input width mismatch");
    if (raw.rows() < 1) throw std::invalid_argument("forward: batch must be non-empty");
    MlpT<float>::Vec out(raw.rows());
    check(svn_forward_eval(device_model(model), precision(), raw.data(), raw.rows(), raw.cols(),
                           out.data()));  // raw is RowMajor (nn.hpp:18)
    return out;
}

std::pair<double, int> predict_min_distance(const Mlp& model, const std::vector<Vec3>& cloud, const Motion& m) {
    if (cloud.empty()) throw std::invalid_argument("predict_min_distance: empty point cloud");
    double mn = 0;
    int32_t idx = 0;
    // std::vector<Vec3> is a contiguous double [P x 3] (Vec3 = Eigen::Vector3d, geometry.hpp:11)
    check(svn_predict_min_distance(device_model(model), precision(), cloud.front().data(),
                                   static_cast<int64_t>(cloud.size()), m.q0.data(), m.q1.data(),
                                   static_cast<int32_t>(m.q0.size()), &mn, &idx));
    return {mn, idx};
}

}  // namespace sweptnet
