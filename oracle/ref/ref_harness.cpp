// ref_harness.cpp — TEST INFRASTRUCTURE ONLY.  A C entry layer over the reference's OWN
// inference code (/root/reference/proj/src/nn.cpp, robot.cpp, geometry.cpp compiled
// unmodified against oracle/ref/eigen_subset by oracle/ref/Makefile into oracle/_ref/).
// tests/ and tests/golden/make_ref_golden.py load it as the checker of the C oracle
// (oracle/sweptnet_oracle.c) and of the CUDA path, and bench.py's CPU legs (--impl reference,
// cpu_baseline) time it as the reference's own CPU path; nothing in the product links it.
//
// Every entry returns 0 on success or an error kind (1 IoError, 2 FormatError,
// 3 TruncationError, 4 VersionError, 5 std::invalid_argument, 6 other) with the reference's
// exception text in ref_last_error().  Models travel as SVCKPT01 files, read and written by
// the reference's own load_checkpoint / save_checkpoint (nn.cpp:499-576).
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "sweptnet/errors.hpp"
#include "sweptnet/nn.hpp"
#include "sweptnet/robot.hpp"

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        g_err.clear();
        return 0;
    } catch (const sweptnet::IoError& e) {
        g_err = e.what();
        return 1;
    } catch (const sweptnet::FormatError& e) {
        g_err = e.what();
        return 2;
    } catch (const sweptnet::TruncationError& e) {
        g_err = e.what();
        return 3;
    } catch (const sweptnet::VersionError& e) {
        g_err = e.what();
        return 4;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 5;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 6;
    }
}

sweptnet::MlpT<double> to_double(const sweptnet::Mlp& m) {
    sweptnet::MlpT<double> d;
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
}  // namespace

extern "C" {

__attribute__((visibility("default"))) const char* ref_last_error() { return g_err.c_str(); }

// init_model<float> (nn.cpp:57-93) written with save_checkpoint (nn.cpp:499-522).
__attribute__((visibility("default"))) int ref_init_save(int n_blocks, int block_dim, int dof, uint64_t seed,
                                                         const char* path) {
    return guarded([&] { sweptnet::save_checkpoint(path, sweptnet::init_model<float>(n_blocks, block_dim, dof, seed)); });
}

// param_count (nn.cpp:18-24) of init_model(n_blocks, block_dim, dof, 0).
__attribute__((visibility("default"))) long ref_param_count(int n_blocks, int block_dim, int dof) {
    long n = -1;
    guarded([&] { n = sweptnet::init_model<float>(n_blocks, block_dim, dof, 0).param_count(); });
    return n;
}

// load_checkpoint (nn.cpp:524-576) and forward_eval<float> (nn.cpp:95-130) on raw [B x cols] rows.
__attribute__((visibility("default"))) int ref_forward_eval(const char* ckpt, const float* raw, long B, long cols,
                                                            float* out) {
    return guarded([&] {
        const sweptnet::Mlp m = sweptnet::load_checkpoint(ckpt);
        sweptnet::Mlp::Mat x(B, cols);
        for (long r = 0; r < B; ++r)
            for (long c = 0; c < cols; ++c) x(r, c) = raw[r * cols + c];
        const sweptnet::Mlp::Vec y = sweptnet::forward_eval(m, x);
        for (long r = 0; r < B; ++r) out[r] = y[r];
    });
}

// forward_eval<double> (the reference's test-oracle instantiation, nn.cpp:588) on the
// checkpoint's parameters widened to double.
__attribute__((visibility("default"))) int ref_forward_eval_f64(const char* ckpt, const double* raw, long B, long cols,
                                                                double* out) {
    return guarded([&] {
        const sweptnet::MlpT<double> m = to_double(sweptnet::load_checkpoint(ckpt));
        sweptnet::MlpT<double>::Mat x(B, cols);
        for (long r = 0; r < B; ++r)
            for (long c = 0; c < cols; ++c) x(r, c) = raw[r * cols + c];
        const sweptnet::MlpT<double>::Vec y = sweptnet::forward_eval(m, x);
        for (long r = 0; r < B; ++r) out[r] = y[r];
    });
}

// predict_min_distance (nn.cpp:460-480): double cloud [P x 3], q0/q1 [dof].
__attribute__((visibility("default"))) int ref_predict_min_distance(const char* ckpt, const double* cloud, long P,
                                                                    const double* q0, const double* q1, int dof,
                                                                    double* min_out, int* idx_out) {
    return guarded([&] {
        const sweptnet::Mlp m = sweptnet::load_checkpoint(ckpt);
        std::vector<sweptnet::Vec3> pts(static_cast<size_t>(P));
        for (long i = 0; i < P; ++i) pts[static_cast<size_t>(i)] = sweptnet::Vec3(cloud[3 * i], cloud[3 * i + 1], cloud[3 * i + 2]);
        sweptnet::Motion mo;
        mo.q0.resize(dof);
        mo.q1.resize(dof);
        for (int j = 0; j < dof; ++j) {
            mo.q0[j] = q0[j];
            mo.q1[j] = q1[j];
        }
        const auto r = sweptnet::predict_min_distance(m, pts, mo);
        *min_out = r.first;
        *idx_out = r.second;
    });
}

// make_normalizer (nn.cpp:314-338) for default_robot(dof) (robot.cpp:115-131) and a training
// split whose positions are x [n x 3] (the joint parts of the samples do not enter it).
__attribute__((visibility("default"))) int ref_make_normalizer(int dof, const float* x, long n, float* shift,
                                                               float* scale) {
    return guarded([&] {
        const sweptnet::RobotModel robot = sweptnet::default_robot(dof);
        std::vector<sweptnet::TrainingSample> split(static_cast<size_t>(n));
        for (long i = 0; i < n; ++i) {
            auto& s = split[static_cast<size_t>(i)];
            s.x = Eigen::Vector3f(x[3 * i], x[3 * i + 1], x[3 * i + 2]);
            s.q0.setZero(dof);
            s.q1.setZero(dof);
        }
        Eigen::VectorXf sh, sc;
        sweptnet::make_normalizer(robot, split, sh, sc);
        for (int k = 0; k < 3 + 2 * dof; ++k) {
            shift[k] = sh[k];
            scale[k] = sc[k];
        }
    });
}

// The reference's per-motion call pattern, timed (bench.py --impl reference and its cpu_baseline
// leg): one model, one cloud, M motions, each a predict_min_distance call (nn.cpp:460-480) issued
// from `threads` worker threads that claim motions from a shared counter — run_box_world's
// parallel_for over motions (bench.cpp:156,193).  `seconds` covers the calls only (model load and
// cloud conversion are outside, as they are per scene in the reference).
__attribute__((visibility("default"))) int ref_time_predict_min_distance(const char* ckpt, const double* cloud, long P,
                                                                         const double* q01, long M, int dof,
                                                                         int threads, double* min_out, int* idx_out,
                                                                         double* seconds) {
    return guarded([&] {
        const sweptnet::Mlp m = sweptnet::load_checkpoint(ckpt);
        std::vector<sweptnet::Vec3> pts(static_cast<size_t>(P));
        for (long i = 0; i < P; ++i) pts[static_cast<size_t>(i)] = sweptnet::Vec3(cloud[3 * i], cloud[3 * i + 1], cloud[3 * i + 2]);
        std::vector<sweptnet::Motion> motions(static_cast<size_t>(M));
        for (long j = 0; j < M; ++j) {
            sweptnet::Motion& mo = motions[static_cast<size_t>(j)];
            mo.q0.resize(dof);
            mo.q1.resize(dof);
            for (int k = 0; k < dof; ++k) {
                mo.q0[k] = q01[j * 2 * dof + k];
                mo.q1[k] = q01[j * 2 * dof + dof + k];
            }
        }
        std::atomic<long> next{0};
        std::string first_error;
        std::atomic<bool> failed{false};
        auto work = [&] {
            try {
                for (long j = next.fetch_add(1); j < M; j = next.fetch_add(1)) {
                    const auto r = sweptnet::predict_min_distance(m, pts, motions[static_cast<size_t>(j)]);
                    min_out[j] = r.first;
                    idx_out[j] = r.second;
                }
            } catch (const std::exception& e) {
                if (!failed.exchange(true)) first_error = e.what();
            }
        };
        const int T = threads < 1 ? 1 : threads;
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int t = 1; t < T; ++t) pool.emplace_back(work);
        work();
        for (std::thread& t : pool) t.join();
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (failed) throw std::runtime_error(first_error);
    });
}

// load_checkpoint alone: the error kind and text of a malformed file.
__attribute__((visibility("default"))) int ref_load_checkpoint(const char* ckpt, int* n_blocks, int* block_dim,
                                                               int* input_dim) {
    return guarded([&] {
        const sweptnet::Mlp m = sweptnet::load_checkpoint(ckpt);
        *n_blocks = m.n_blocks;
        *block_dim = m.block_dim;
        *input_dim = m.input_dim;
    });
}

// Rng::uniform(lo, hi) (rng.hpp:21-23) stream as compiled in the reference's own header.
__attribute__((visibility("default"))) void ref_uniform_stream(uint64_t seed, long n, double lo, double hi,
                                                               double* out) {
    sweptnet::Rng rng(seed);
    for (long i = 0; i < n; ++i) out[i] = rng.uniform(lo, hi);
}
}
