// Where the time of one small host-buffer query goes (the reference's per-motion call: one
// motion x 3000 points of the Fig. 2 5x512 network in bf16): the same sequence svn_query_min
// runs — pinned staging fill, H2D, the C-ABI device query (K0 + fused kernel), D2H, stream
// sync — issued by hand with host timestamps after every API call and CUDA events between the
// stream operations.  Medians of 300 calls.
// g++ -std=c++17 -O2 -Iinclude -I/usr/local/cuda/include scripts/latency_breakdown.cpp \
//     -Lpaper_2402_15281_b200/_lib -lsweptnet_b200 -L/usr/local/cuda/lib64 -lcudart \
//     -Wl,-rpath,$PWD/paper_2402_15281_b200/_lib -o latency_breakdown
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "sweptnet_b200.hpp"

using namespace sweptnet_b200;
using clk = std::chrono::steady_clock;

static double us(clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::micro>(b - a).count(); }

int main(int argc, char** argv) {
    const int P = argc > 1 ? std::atoi(argv[1]) : 3000;
    Model m = Model::init(Program::fig2(5, 512, 6), 1, 0);
    std::mt19937 rng(1);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    std::vector<double> cloud(static_cast<size_t>(3 * P));
    for (double& x : cloud) x = U(rng);
    const double q0[6] = {0.1, -0.2, 0.3, 0.0, 0.5, -0.4}, q1[6] = {1.0, 0.5, -0.3, 0.2, 0.1, 0.0};
    const size_t in_bytes = sizeof(float) * (3 * P + 12);
    float* hin = nullptr;
    uint8_t* hout = nullptr;
    cudaMallocHost(&hin, in_bytes);
    cudaMallocHost(&hout, 64);
    float* din = nullptr;
    uint8_t* dout = nullptr;
    cudaMalloc(&din, in_bytes);
    cudaMalloc(&dout, 64);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaEvent_t ev[4];
    for (auto& e : ev) cudaEventCreate(&e);
    const char* names[] = {"fill", "H2D api", "query api (K0+fused)", "D2H api", "sync", "total"};
    std::vector<std::vector<double>> host(6);
    std::vector<std::vector<float>> gpu(3);
    for (int it = 0; it < 330; ++it) {
        const auto t0 = clk::now();
        for (int i = 0; i < 3 * P; ++i) hin[i] = static_cast<float>(cloud[i]);
        for (int i = 0; i < 6; ++i) hin[3 * P + i] = static_cast<float>(q0[i]), hin[3 * P + 6 + i] = static_cast<float>(q1[i]);
        const auto t1 = clk::now();
        cudaEventRecord(ev[0], st);
        cudaMemcpyAsync(din, hin, in_bytes, cudaMemcpyHostToDevice, st);
        cudaEventRecord(ev[1], st);
        const auto t2 = clk::now();
        check(svn_query_min_device(m.handle(), SVN_PREC_BF16, din, P, din + 3 * P, 1, 0.0,
                                   reinterpret_cast<float*>(dout), reinterpret_cast<int32_t*>(dout + 16), dout + 32,
                                   nullptr, st));
        cudaEventRecord(ev[2], st);
        const auto t3 = clk::now();
        cudaMemcpyAsync(hout, dout, 48, cudaMemcpyDeviceToHost, st);
        cudaEventRecord(ev[3], st);
        const auto t4 = clk::now();
        cudaStreamSynchronize(st);
        const auto t5 = clk::now();
        if (it < 30) continue;
        host[0].push_back(us(t0, t1));
        host[1].push_back(us(t1, t2));
        host[2].push_back(us(t2, t3));
        host[3].push_back(us(t3, t4));
        host[4].push_back(us(t4, t5));
        host[5].push_back(us(t0, t5));
        for (int k = 0; k < 3; ++k) {
            float ms = 0;
            cudaEventElapsedTime(&ms, ev[k], ev[k + 1]);
            gpu[k].push_back(ms * 1e3f);
        }
    }
    auto med = [](std::vector<double> v) { std::sort(v.begin(), v.end()); return v[v.size() / 2]; };
    auto medf = [](std::vector<float> v) { std::sort(v.begin(), v.end()); return v[v.size() / 2]; };
    std::printf("Fig. 2 5x512 bf16, 1 motion x %d points, medians of 300 calls\n", P);
    for (int k = 0; k < 6; ++k) std::printf("  host %-22s %7.1f us\n", names[k], med(host[k]));
    const char* gn[] = {"H2D", "K0 + fused", "D2H"};
    for (int k = 0; k < 3; ++k) std::printf("  gpu  %-22s %7.1f us\n", gn[k], medf(gpu[k]));
    return 0;
}
