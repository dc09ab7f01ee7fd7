// Per-call latency of the drop-in predict_min_distance from C++ (no Python in the loop):
// median wall time of 300 calls per (network, points, precision), and the fused kernel's own
// CUDA-event time (svn_kernel_timing_*) over another 300 calls.
// g++ -std=c++17 -O2 -Iinclude scripts/latency_cpp.cpp -Lpaper_2402_15281_b200/_lib -lsweptnet_b200 \
//     -Wl,-rpath,$PWD/paper_2402_15281_b200/_lib -o scripts/latency_cpp
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <random>
#include <vector>

#include "sweptnet_b200.hpp"

using namespace sweptnet_b200;

int main() {
    struct Net {
        const char* name;
        Program prog;
        int bound;
    } nets[] = {{"fig2_5x512", Program::fig2(5, 512, 6), 0}, {"plain_4x256", Program::plain(4, 256, 6), 1}};
    std::mt19937 rng(1);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    for (const Net& n : nets) {
        Model m = Model::init(n.prog, 1, n.bound);
        for (int P : {3000, 20000}) {
            std::vector<Vec3> cloud(static_cast<size_t>(P));
            for (Vec3& p : cloud) p = {1.2 * U(rng), -0.4 + 0.8 * U(rng), 0.5 * U(rng)};
            Motion mo{{0.1, -0.2, 0.3, 0.0, 0.5, -0.4}, {1.0, 0.5, -0.3, 0.2, 0.1, 0.0}};
            for (Precision pr : {Precision::BF16, Precision::FP32}) {
                for (int i = 0; i < 30; ++i) predict_min_distance(m, cloud, mo, pr);
                // wall time per call first (kernel timing off: it would also disable the graph path),
                // then the fused kernel's CUDA-event time over another 300 calls
                std::vector<double> ts;
                for (int i = 0; i < 300; ++i) {
                    const auto t0 = std::chrono::steady_clock::now();
                    predict_min_distance(m, cloud, mo, pr);
                    ts.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
                }
                svn_kernel_timing_begin();
                for (int i = 0; i < 300; ++i) predict_min_distance(m, cloud, mo, pr);
                double kms = 0;
                int64_t kn = 0;
                svn_kernel_timing_end(&kms, &kn);
                std::sort(ts.begin(), ts.end());
                std::printf("%-12s P=%6d %-5s call median %7.1f us  p90 %7.1f us | fused kernel %7.1f us\n", n.name, P,
                            pr == Precision::BF16 ? "bf16" : "fp32", ts[ts.size() / 2], ts[ts.size() * 9 / 10],
                            kn ? kms * 1e3 / kn : 0.0);
            }
        }
    }
    return 0;
}
