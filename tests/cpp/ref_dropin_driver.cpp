// ref_dropin_driver.cpp — TEST: the reference with the B200 drop-in applied, called through the
// reference's OWN API.  Linked (oracle/ref/Makefile target `dropin`) from the reference's
// nn.cpp / robot.cpp / geometry.cpp patched by integration/sweptnet_b200.patch, the shim
// integration/nn_b200.cpp and libsweptnet_b200.so.  tests/test_gpu_dropin.py runs it on the GPU
// against the golden vectors of the unpatched reference (tests/golden/ref_fig2.npz).
//
//   ref_dropin_driver <ckpt> <raw.f32> <B> <cloud.f64> <P> <q01.f64> <out.bin> [threads]
// out.bin: forward_eval<float>[B], forward<float>(Eval)[B] (f32), forward_eval<double>[B] (f64),
//          predict_min_distance (f64 min, i32 index), then the same call from `threads`
//          concurrent threads (f64 min, i32 index each).  stdout: the reference's error texts.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <stdexcept>
#include <thread>
#include <vector>

#include "sweptnet/nn.hpp"

using namespace sweptnet;

template <class T>
std::vector<T> read_file(const char* path, size_t n) {
    std::vector<T> v(n);
    std::ifstream f(path, std::ios::binary);
    f.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(n * sizeof(T)));
    if (!f) throw std::runtime_error(std::string("short read: ") + path);
    return v;
}

MlpT<double> widen(const Mlp& m) {
    MlpT<double> d;
    d.n_blocks = m.n_blocks;
    d.block_dim = m.block_dim;
    d.input_dim = m.input_dim;
    d.norm_shift = m.norm_shift.cast<double>();
    d.norm_scale = m.norm_scale.cast<double>();
    d.input_weight = m.input_weight.cast<double>();
    d.input_bias = m.input_bias.cast<double>();
    d.blocks.resize(m.blocks.size());
    for (size_t i = 0; i < m.blocks.size(); ++i) {
        d.blocks[i].weight = m.blocks[i].weight.cast<double>();
        d.blocks[i].bias = m.blocks[i].bias.cast<double>();
        d.blocks[i].gamma = m.blocks[i].gamma.cast<double>();
        d.blocks[i].beta = m.blocks[i].beta.cast<double>();
        d.blocks[i].running_mean = m.blocks[i].running_mean.cast<double>();
        d.blocks[i].running_var = m.blocks[i].running_var.cast<double>();
    }
    d.output_weight = m.output_weight.cast<double>();
    d.output_bias = m.output_bias;
    return d;
}

int main(int argc, char** argv) {
    if (argc < 8) {
        std::fprintf(stderr, "usage: %s ckpt raw.f32 B cloud.f64 P q01.f64 out.bin [threads]\n", argv[0]);
        return 2;
    }
    try {
        Mlp model = load_checkpoint(argv[1]);  // nn.cpp:524-576 (CPU, unchanged)
        const long B = std::atol(argv[3]), P = std::atol(argv[5]);
        const int in = model.input_dim, dof = model.dof();
        const int threads = argc > 8 ? std::atoi(argv[8]) : 4;
        const auto raw_v = read_file<float>(argv[2], static_cast<size_t>(B * in));
        const auto cloud_v = read_file<double>(argv[4], static_cast<size_t>(P * 3));
        const auto q_v = read_file<double>(argv[6], static_cast<size_t>(2 * dof));

        Mlp::Mat raw(B, in);
        for (long r = 0; r < B; ++r)
            for (int c = 0; c < in; ++c) raw(r, c) = raw_v[static_cast<size_t>(r * in + c)];
        const Mlp::Vec y = forward_eval(model, raw);                 // -> the B200 C-ABI
        const Mlp::Vec y2 = forward(model, raw, Mode::Eval);         // nn.cpp:137 dispatch -> same
        MlpT<double>::Mat raw64 = raw.cast<double>();
        const MlpT<double>::Vec y64 = forward_eval(widen(model), raw64);  // CPU body (nn.cpp:588)

        std::vector<Vec3> cloud(static_cast<size_t>(P));
        for (long i = 0; i < P; ++i) cloud[static_cast<size_t>(i)] = Vec3(cloud_v[3 * i], cloud_v[3 * i + 1], cloud_v[3 * i + 2]);
        Motion mo;
        mo.q0.resize(dof);
        mo.q1.resize(dof);
        for (int j = 0; j < dof; ++j) {
            mo.q0[j] = q_v[static_cast<size_t>(j)];
            mo.q1[j] = q_v[static_cast<size_t>(dof + j)];
        }
        const auto pmd = predict_min_distance(model, cloud, mo);     // -> the B200 C-ABI

        // concurrent callers, as run_box_world's parallel_for workers (bench.cpp:156,193)
        std::vector<std::pair<double, int>> par(static_cast<size_t>(threads));
        std::vector<std::thread> ts;
        for (int t = 0; t < threads; ++t)
            ts.emplace_back([&, t] { par[static_cast<size_t>(t)] = predict_min_distance(model, cloud, mo); });
        for (auto& t : ts) t.join();

        std::ofstream out(argv[7], std::ios::binary);
        out.write(reinterpret_cast<const char*>(y.data()), static_cast<std::streamsize>(B * sizeof(float)));
        out.write(reinterpret_cast<const char*>(y2.data()), static_cast<std::streamsize>(B * sizeof(float)));
        out.write(reinterpret_cast<const char*>(y64.data()), static_cast<std::streamsize>(B * sizeof(double)));
        auto put_pmd = [&](const std::pair<double, int>& r) {
            const int32_t i = r.second;
            out.write(reinterpret_cast<const char*>(&r.first), sizeof(double));
            out.write(reinterpret_cast<const char*>(&i), sizeof(int32_t));
        };
        put_pmd(pmd);
        for (const auto& r : par) put_pmd(r);

        // the reference's argument errors, raised through the drop-in
        auto expect = [](const char* what, auto&& f) {
            try {
                f();
                std::printf("%s: no error\n", what);
            } catch (const std::invalid_argument& e) {
                std::printf("%s: invalid_argument: %s\n", what, e.what());
            }
        };
        expect("empty_cloud", [&] { predict_min_distance(model, std::vector<Vec3>{}, mo); });
        Motion bad;
        bad.q0.resize(dof + 1);
        bad.q1.resize(dof + 1);
        bad.q0.setZero();
        bad.q1.setZero();
        expect("dof_mismatch", [&] { predict_min_distance(model, cloud, bad); });
        expect("width_mismatch", [&] { forward_eval(model, Mlp::Mat(2, in + 1)); });
        std::printf("ok\n");
    } catch (const std::exception& e) {
        std::printf("FAILED: %s\n", e.what());
        return 1;
    }
    return 0;
}
