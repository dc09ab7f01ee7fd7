// Compiles the C++ host API against the C-ABI library and runs the reference-shaped
// calls.  Built and run by tests/test_cpp_host_api.py (GPU); compiled-only on CPU.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <stdexcept>

#include "sweptnet_b200.hpp"

using namespace sweptnet_b200;

int main() {
    const Program prog = Program::fig2(3, 256, 6);
    Model m = Model::init(prog, 7, 0);
    std::vector<Vec3> cloud;
    for (int i = 0; i < 300; ++i) cloud.push_back({0.004 * i, -0.2 + 0.001 * i, 0.1});
    Motion mo{{0.1, -0.2, 0.3, 0.0, 0.5, -0.4}, {1.0, 0.5, -0.3, 0.2, 0.1, 0.0}};
    auto [mn, idx] = predict_min_distance(m, cloud, mo);
    std::vector<float> raw;
    for (const Vec3& p : cloud) {
        for (double c : p) raw.push_back(static_cast<float>(c));
        for (double v : mo.q0) raw.push_back(static_cast<float>(v));
        for (double v : mo.q1) raw.push_back(static_cast<float>(v));
    }
    const std::vector<float> d = forward_eval(m, raw, static_cast<long>(cloud.size()), 15);
    int best = 0;
    for (int i = 1; i < static_cast<int>(d.size()); ++i)
        if (d[i] < d[best]) best = i;
    auto proxy = batched_proxy(m, cloud, {mo, mo}, Precision::FP32_EXACT);
    // the tensor-core precisions through the same call: fp16 within its frozen bound of the exact
    // path (tests/golden/fp16_bounds.json: fig2_3x256 0.0019), bf16 within its own (0.013)
    const double mn16 = predict_min_distance(m, cloud, mo, Precision::FP16).first;
    const double mnbf = predict_min_distance(m, cloud, mo, Precision::BF16).first;
    const bool tc_ok = std::fabs(mn16 - mn) <= 0.0019 && std::fabs(mnbf - mn) <= 0.013;
    bool threw = false;
    try {
        predict_min_distance(m, {}, mo);
    } catch (const std::invalid_argument& e) {
        threw = std::string(e.what()) == "predict_min_distance: empty point cloud";
    }
    // the same motion batch spread over "two GPUs" (device 0 twice: one worker thread each)
    std::vector<float> pts, q01;
    for (const Vec3& p : cloud)
        for (double c : p) pts.push_back(static_cast<float>(c));
    for (int j = 0; j < 3; ++j) {
        for (double v : mo.q0) q01.push_back(static_cast<float>(v) + 0.1f * j);
        for (double v : mo.q1) q01.push_back(static_cast<float>(v));
    }
    const svn_model_desc dd = prog.desc();
    std::vector<float> params(static_cast<size_t>(svn_param_count(&dd)));
    check(svn_init_params(&dd, 7, 0, params.data()));
    MultiModel mg(prog, params, {0, 0});
    const MinResult r = mg.query_min(pts, q01, 0.02, Precision::FP32_EXACT, Shard::MOTIONS);
    // the same against the scene kept resident on both devices
    mg.set_scene(pts);
    const MinResult rs = mg.query_min_scene(q01, 0.02, Precision::FP32_EXACT, Shard::MOTIONS);
    const bool multi_ok = mg.devices() == 2 && r.min.size() == 3 && static_cast<double>(r.min[0]) == mn && r.argmin[0] == idx &&
                          rs.min == r.min && rs.argmin == r.argmin && rs.free == r.free;
    // the same parameters as an SVCKPT01 checkpoint (nn.cpp:482-520): the loaded Model knows its
    // program from the header (dof, width, Fig. 2 layers) and predicts the same bits
    const char* ck = "host_api_demo.svckpt";
    {
        FILE* f = std::fopen(ck, "wb");
        const uint32_t hdr[4] = {1u, 3u, 256u, 15u};
        std::fwrite("SVCKPT01", 1, 8, f);
        std::fwrite(hdr, sizeof(uint32_t), 4, f);
        std::fwrite(params.data(), sizeof(float), params.size(), f);
        std::fclose(f);
    }
    Model mc = Model::load_checkpoint(ck);
    std::remove(ck);
    auto [mn_c, idx_c] = predict_min_distance(mc, cloud, mo);
    const bool ckpt_ok = mc.dof() == 6 && mc.program().width == 256 && mc.program().layers.size() == 4 &&
                         mc.program().layers[0].act == 0 && mc.program().layers[3].residual == 1 && mn_c == mn &&
                         idx_c == idx;
    std::printf("min %.9g idx %d | forward argmin %d %.9g | proxy %.9g | empty-cloud error %d | multi %.9g %d | "
                "checkpoint dof %d ok %d | fp16 %.9g bf16 %.9g ok %d\n", mn, idx, best, static_cast<double>(d[best]),
                proxy(1), threw ? 1 : 0, static_cast<double>(r.min[0]), multi_ok ? 1 : 0, mc.dof(), ckpt_ok ? 1 : 0, mn16,
                mnbf, tc_ok ? 1 : 0);
    return (idx == best && mn == static_cast<double>(d[best]) && proxy(1) == mn && threw && multi_ok && ckpt_ok && tc_ok)
               ? 0
               : 1;
}
