// Host-side costs behind a small query (SVN_HOST_TRACE found the double->float fill and the fused
// kernel's launch to be the largest host phases): conversion of a cloud into pageable vs pinned
// memory, and launch cost of an empty kernel by parameter size, cluster dims and PDL attribute.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o host_costs scripts/host_costs.cu
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <vector>

struct Big { char b[3200]; };
struct Small { char b[256]; };
__global__ void __cluster_dims__(2, 1, 1) kbig_c(const __grid_constant__ Big p) { if (p.b[0] == 7 && threadIdx.x == 9999) asm volatile("trap;"); }
__global__ void __cluster_dims__(2, 1, 1) ksmall_c(const __grid_constant__ Small p) { if (p.b[0] == 7 && threadIdx.x == 9999) asm volatile("trap;"); }
__global__ void kbig(const __grid_constant__ Big p) { if (p.b[0] == 7 && threadIdx.x == 9999) asm volatile("trap;"); }
__global__ void ksmall(const __grid_constant__ Small p) { if (p.b[0] == 7 && threadIdx.x == 9999) asm volatile("trap;"); }

using clk = std::chrono::steady_clock;
static double us(clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::micro>(b - a).count(); }

template <class F>
static double med(F f, int n = 2000) {
    std::vector<double> t;
    for (int i = 0; i < n; ++i) {
        auto a = clk::now();
        f();
        t.push_back(us(a, clk::now()));
    }
    std::sort(t.begin(), t.end());
    return t[t.size() / 2];
}

int main() {
    const int P = 3000;
    std::vector<double> cloud(3 * P, 0.5);
    std::vector<float> pageable(3 * P + 64);
    float* pinned = nullptr;
    cudaMallocHost(&pinned, sizeof(float) * (3 * P + 64));
    auto conv = [&](float* dst) {
        for (int i = 0; i < 3 * P; ++i) dst[i] = static_cast<float>(cloud[i]);
    };
    std::printf("convert 3000 points into pageable: %.2f us, into pinned: %.2f us\n", med([&] { conv(pageable.data()); }),
                med([&] { conv(pinned); }));
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    Big big{};
    Small small{};
    auto ex = [&](auto kernel, auto param, int grid, bool pdl) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(352);
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = pdl ? 1 : 0;
        cudaLaunchKernelEx(&cfg, kernel, param);
    };
    for (int w = 0; w < 100; ++w) ex(kbig_c, big, 148, true);
    cudaStreamSynchronize(st);
    auto launch_sync = [&](auto f) {
        return med([&] { f(); }, 500);
    };
    std::printf("launch (host API only) us:  big+cluster+pdl %.2f | big+cluster %.2f | small+cluster %.2f | big %.2f | small %.2f | <<<>>> small %.2f\n",
                launch_sync([&] { ex(kbig_c, big, 148, true); cudaStreamSynchronize(st); }) - launch_sync([&] { cudaStreamSynchronize(st); }),
                launch_sync([&] { ex(kbig_c, big, 148, false); cudaStreamSynchronize(st); }) - launch_sync([&] { cudaStreamSynchronize(st); }),
                launch_sync([&] { ex(ksmall_c, small, 148, false); cudaStreamSynchronize(st); }) - launch_sync([&] { cudaStreamSynchronize(st); }),
                launch_sync([&] { ex(kbig, big, 148, false); cudaStreamSynchronize(st); }) - launch_sync([&] { cudaStreamSynchronize(st); }),
                launch_sync([&] { ex(ksmall, small, 148, false); cudaStreamSynchronize(st); }) - launch_sync([&] { cudaStreamSynchronize(st); }),
                launch_sync([&] { ksmall<<<148, 352, 0, st>>>(small); cudaStreamSynchronize(st); }) - launch_sync([&] { cudaStreamSynchronize(st); }));
    // API time alone (no sync inside the timed region)
    std::vector<double> a1, a2, a3;
    for (int i = 0; i < 500; ++i) {
        auto t0 = clk::now();
        ex(kbig_c, big, 148, true);
        auto t1 = clk::now();
        cudaStreamSynchronize(st);
        auto t2 = clk::now();
        ex(ksmall_c, small, 148, true);
        auto t3 = clk::now();
        cudaStreamSynchronize(st);
        auto t4 = clk::now();
        ksmall<<<1, 32, 0, st>>>(small);
        auto t5 = clk::now();
        cudaStreamSynchronize(st);
        a1.push_back(us(t0, t1));
        a2.push_back(us(t3, t4 - (t4 - t3)) + us(t2, t3));
        a3.push_back(us(t4, t5));
    }
    std::sort(a1.begin(), a1.end());
    std::sort(a2.begin(), a2.end());
    std::sort(a3.begin(), a3.end());
    std::printf("API call alone us: cluster+pdl 3200 B params %.2f | cluster+pdl 256 B %.2f | <<<1,32>>> 256 B %.2f\n",
                a1[a1.size() / 2], a2[a2.size() / 2], a3[a3.size() / 2]);
    return 0;
}
