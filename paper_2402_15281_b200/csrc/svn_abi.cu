// svn_abi.cu — implementation of the C-ABI declared in include/sweptnet_b200.h.
//
// Host-side model preparation (layer program parse, BN fold, per-layer device
// layouts, bf16 tcgen05 weight stream), argument validation with the reference's
// exception texts, stream-ordered scratch, kernel sequencing (K0 -> K1), the
// host-buffer convenience entry points that mirror the reference signatures, and
// the SVCKPT01 checkpoint reader.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <random>
#include <string>
#include <utility>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges for Nsight tools, no-ops otherwise

#include "../../include/sweptnet_b200.h"
#include "fused.cuh"
#include "gcc.cuh"
#include "ptx.cuh"

using namespace svn;

namespace {

thread_local std::string g_err;
thread_local int64_t g_launches = 0;
thread_local bool g_timing = false;
thread_local std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_events;
thread_local unsigned long long g_prof[kProfSlots] = {};
bool prof_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SVN_PROF");
        return e && e[0] == '1';
    }();
    return on;
}

svn_status fail(svn_status code, const std::string& msg) {
    g_err = msg;
    return code;
}

svn_status cuda_fail(cudaError_t e, const char* what) {
    const svn_status code = (e == cudaErrorMemoryAllocation) ? SVN_ERR_OUT_OF_MEMORY : SVN_ERR_CUDA;
    return fail(code, std::string("CUDA error in ") + what + ": " + cudaGetErrorName(e) + ": " + cudaGetErrorString(e));
}

#define SVN_CUDA(call, what)                       \
    do {                                           \
        cudaError_t e_ = (call);                   \
        if (e_ != cudaSuccess) return cuda_fail(e_, what); \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

int layer_k(const svn_layer* layers, int l, int N, int in) {
    if (l == 0) return in;
    return N + (layers[l].concat ? in : 0);
}

// bf16 kernels only: fold every Fig. 2 block's BN affine out of the epilogue (nn.cpp:125:
// h += max(a,0)*s + t).  With s >= 0 (or no activation), max(a,0)*s = max(s*a,0), so s scales
// the layer's weight rows and bias; the shifts t are carried as a running offset c (the
// kernel keeps h~ = h - c) and re-enter as W_h.c in the next layer's bias and wo.c in b_o.
// The epilogue of a folded layer is then ReLU + residual only.  Returns the folded
// parameter buffer (same layout) and which layers were folded; layers with a negative s
// under ReLU keep their affine (their offset still folds).  Arithmetic in double.
std::vector<float> fold_affine_bf16(const svn_model_desc* d, const float* params, int64_t n_params,
                                    std::vector<char>& folded) {
    const int N = d->width, in = 3 + 2 * d->dof, L = d->n_layers;
    std::vector<float> P(params, params + n_params);
    folded.assign(static_cast<size_t>(L), 0);
    std::vector<double> c(static_cast<size_t>(N), 0.0), cn(static_cast<size_t>(N), 0.0);
    int64_t off = 2 * in;
    for (int l = 0; l < L; ++l) {
        const svn_layer& ly = d->layers[l];
        const int K = layer_k(d->layers, l, N, in);
        float* W = P.data() + off;
        float* b = W + static_cast<int64_t>(N) * K;
        const bool res = ly.residual && l > 0;
        if (l > 0)
            for (int n = 0; n < N; ++n) {  // the incoming offset, through the h-part weights
                double acc = b[n];
                for (int k = 0; k < N; ++k) acc += static_cast<double>(W[static_cast<int64_t>(k) * N + n]) * c[k];
                b[n] = static_cast<float>(acc);
            }
        for (int n = 0; n < N; ++n) cn[n] = res ? c[n] : 0.0;
        if (ly.affine) {
            const float *gamma = b + N, *beta = b + 2 * N, *mean = b + 3 * N, *var = b + 4 * N;
            std::vector<float> sv(N), tv(N);
            bool ok = true;
            for (int n = 0; n < N; ++n) {
                sv[n] = gamma[n] / std::sqrt(var[n] + 1e-5f);  // as the model build (nn.cpp:108-110)
                tv[n] = std::fma(-mean[n], sv[n], beta[n]);
                if (ly.act && !(sv[n] >= 0.0f)) ok = false;
            }
            if (ok) {
                for (int n = 0; n < N; ++n) {
                    for (int k = 0; k < K; ++k) W[static_cast<int64_t>(k) * N + n] *= sv[n];
                    b[n] *= sv[n];
                    cn[n] += tv[n];
                }
                folded[static_cast<size_t>(l)] = 1;
            }
        }
        c.swap(cn);
        off += static_cast<int64_t>(N) * K + N + (ly.affine ? 4 * N : 0);
    }
    double bo = P[static_cast<size_t>(off + N)];
    for (int n = 0; n < N; ++n) bo += static_cast<double>(P[static_cast<size_t>(off + n)]) * c[n];
    P[static_cast<size_t>(off + N)] = static_cast<float>(bo);
    return P;
}

svn_status validate_desc(const svn_model_desc* d) {
    if (!d || !d->layers) return fail(SVN_ERR_INVALID_ARGUMENT, "model: null descriptor");
    if (d->n_layers < 1 || d->n_layers > kMaxLayers)
        return fail(SVN_ERR_INVALID_ARGUMENT, "model: n_layers must be in 1..32");
    if (d->width < 1) return fail(SVN_ERR_INVALID_ARGUMENT, "init_model: n_blocks, block_dim and dof must be >= 1");
    if (d->dof < 1 || 3 + 2 * d->dof > kMaxIn)
        return fail(SVN_ERR_INVALID_ARGUMENT, "model: dof must be in 1..14");
    return SVN_OK;
}

// cuTensorMapEncodeTiled from the driver, fetched through the runtime (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// A byte blob seen as a 2-D tensor [rows][row_bytes]; one TMA box = box_rows rows.
svn_status encode_blob_map(CUtensorMap* map, const void* base, uint64_t row_bytes, uint64_t rows, uint32_t box_rows) {
    auto fn = tmap_encoder();
    if (!fn) return fail(SVN_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {row_bytes, rows > 0 ? rows : 1};
    cuuint64_t strides[1] = {row_bytes};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(row_bytes), box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(SVN_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
    return SVN_OK;
}

// bf16 hi/lo split (host), matching split_bf16 on the device.
void split_bf16_host(float x, __nv_bfloat16& hi, __nv_bfloat16& lo) {
    hi = __float2bfloat16_rn(x);
    lo = __float2bfloat16_rn(x - __bfloat162float(hi));
}

}  // namespace

struct svn_model {
    int device = 0;
    int L = 0, N = 0, dof = 0, in = 0;
    int num_sms = 148;
    int n_mb = 0;
    std::vector<svn_layer> layers;
    std::vector<void*> allocs;
    FusedArgs base{};        // model part of the kernel arguments
    FusedArgs base_split{};  // width 256: fp32-accurate split-fp16 tensor-core kernel (kernels_split.cu)
    bool has_split = false;
    float* d_wq = nullptr;     // [n_mb][2dof][N]
    float* d_mbbase = nullptr; // [n_mb][N]
    float* d_wxslots = nullptr; // [n_mb][3][N] x-part columns of the concat layers
    bool has_bf16 = false;
    FusedArgs base_bf16{};       // bf16 kernels: base with the BN affine folded (see fold_affine_bf16)
    float* d_wq_bf = nullptr;     // K0 inputs of the bf16 kernels, from the folded parameters
    float* d_mbbase_bf = nullptr;
    float* d_wxslots_bf = nullptr;

    template <class T>
    svn_status upload(const T* host, size_t count, T** out) {
        void* p = nullptr;
        cudaError_t e = cudaMalloc(&p, sizeof(T) * (count ? count : 1));
        if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(model)");
        allocs.push_back(p);
        if (count) {
            e = cudaMemcpy(p, host, sizeof(T) * count, cudaMemcpyHostToDevice);
            if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(model)");
        }
        *out = static_cast<T*>(p);
        return SVN_OK;
    }
    ~svn_model() {
        DeviceGuard g(device);
        for (void* p : allocs) cudaFree(p);
    }
};

extern "C" {

SVN_API const char* svn_last_error(void) { return g_err.c_str(); }
SVN_API const char* svn_version(void) { return "sweptnet_b200 0.1 (sm_100a)"; }
SVN_API int64_t svn_launch_count(void) { return g_launches; }
SVN_API void svn_launch_count_reset(void) { g_launches = 0; }

SVN_API void svn_kernel_timing_begin(void) {
    for (auto& ev : g_events) {
        cudaEventDestroy(ev.first);
        cudaEventDestroy(ev.second);
    }
    g_events.clear();
    g_timing = true;
}

SVN_API svn_status svn_kernel_timing_end(double* total_ms, int64_t* launches) {
    g_timing = false;
    double sum = 0.0;
    for (auto& ev : g_events) {
        SVN_CUDA(cudaEventSynchronize(ev.second), "cudaEventSynchronize");
        float ms = 0.f;
        SVN_CUDA(cudaEventElapsedTime(&ms, ev.first, ev.second), "cudaEventElapsedTime");
        sum += ms;
        cudaEventDestroy(ev.first);
        cudaEventDestroy(ev.second);
    }
    if (total_ms) *total_ms = sum;
    if (launches) *launches = static_cast<int64_t>(g_events.size());
    g_events.clear();
    return SVN_OK;
}

SVN_API int64_t svn_param_count(const svn_model_desc* d) {
    if (validate_desc(d) != SVN_OK) return -1;
    const int N = d->width, in = 3 + 2 * d->dof;
    int64_t n = 2 * static_cast<int64_t>(in);
    for (int l = 0; l < d->n_layers; ++l) {
        n += static_cast<int64_t>(N) * layer_k(d->layers, l, N, in) + N;
        if (d->layers[l].affine) n += 4 * static_cast<int64_t>(N);
    }
    return n + N + 1;
}

SVN_API int64_t svn_trainable_param_count(const svn_model_desc* d) {
    if (validate_desc(d) != SVN_OK) return -1;
    const int N = d->width, in = 3 + 2 * d->dof;
    int64_t n = 0;
    for (int l = 0; l < d->n_layers; ++l) {
        n += static_cast<int64_t>(N) * layer_k(d->layers, l, N, in) + N;
        if (d->layers[l].affine) n += 2 * static_cast<int64_t>(N);
    }
    return n + N + 1;
}

// init_model (nn.cpp:57-93): one std::mt19937_64 stream; tensors in order layer 0 W,
// hidden W's, output W; each drawn row-major over [out x in] (nn.cpp:70-71) with
// Rng::uniform (rng.hpp:21-23) and stored column-major.
SVN_API svn_status svn_init_params(const svn_model_desc* d, uint64_t seed, int32_t bound_mode, float* p) {
    svn_status st = validate_desc(d);
    if (st != SVN_OK) return st;
    if (!p) return fail(SVN_ERR_INVALID_ARGUMENT, "init_params: null output");
    const int N = d->width, in = 3 + 2 * d->dof;
    std::mt19937_64 eng(seed);
    auto uniform = [&](double lo, double hi) {
        const double u = static_cast<double>(eng() >> 11) * 0x1.0p-53;
        return std::fma(hi - lo, u, lo);
    };
    float* q = p;
    for (int i = 0; i < in; ++i) *q++ = 0.0f;
    for (int i = 0; i < in; ++i) *q++ = 1.0f;
    for (int l = 0; l < d->n_layers; ++l) {
        const int K = layer_k(d->layers, l, N, in);
        const double bound = bound_mode ? std::sqrt(6.0 / K) : 1.0 / std::sqrt(static_cast<double>(K));
        for (int r = 0; r < N; ++r)
            for (int c = 0; c < K; ++c) q[static_cast<int64_t>(c) * N + r] = static_cast<float>(uniform(-bound, bound));
        q += static_cast<int64_t>(N) * K;
        for (int i = 0; i < N; ++i) *q++ = 0.0f;
        if (d->layers[l].affine) {
            for (int i = 0; i < N; ++i) *q++ = 1.0f;
            for (int i = 0; i < N; ++i) *q++ = 0.0f;
            for (int i = 0; i < N; ++i) *q++ = 0.0f;
            for (int i = 0; i < N; ++i) *q++ = 1.0f;
        }
    }
    const double bound = bound_mode ? std::sqrt(6.0 / N) : 1.0 / std::sqrt(static_cast<double>(N));
    for (int c = 0; c < N; ++c) *q++ = static_cast<float>(uniform(-bound, bound));
    *q = 0.0f;
    return SVN_OK;
}

SVN_API svn_status svn_model_create(const svn_model_desc* d, const float* params, int64_t n_params, int32_t device,
                                    svn_model** out) {
    svn_status st = validate_desc(d);
    if (st != SVN_OK) return st;
    if (!params || !out) return fail(SVN_ERR_INVALID_ARGUMENT, "model: null params/out");
    if (n_params != svn_param_count(d)) return fail(SVN_ERR_INVALID_ARGUMENT, "model: parameter count mismatch");
    int ndev = 0;
    SVN_CUDA(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) return fail(SVN_ERR_INVALID_ARGUMENT, "model: no such CUDA device");
    DeviceGuard guard(device);

    auto m = new svn_model();
    m->device = device;
    m->L = d->n_layers;
    m->N = d->width;
    m->dof = d->dof;
    m->in = 3 + 2 * d->dof;
    m->layers.assign(d->layers, d->layers + d->n_layers);
    cudaDeviceGetAttribute(&m->num_sms, cudaDevAttrMultiProcessorCount, device);
    const int N = m->N, in = m->in, L = m->L, nq = 2 * m->dof;
    FusedArgs& a = m->base;
    a.L = L;
    a.N = N;
    a.dof = m->dof;
    a.in = in;

    // parse the parameter buffer (layout: include/sweptnet_b200.h)
    const float* q = params;
    for (int k = 0; k < in; ++k) a.shift[k] = q[k];
    q += in;
    for (int k = 0; k < in; ++k) a.scale[k] = q[k];
    q += in;
    std::vector<float> wq_host, mbbase_host, wx_host;
    auto cleanup_fail = [&](svn_status s) {
        delete m;
        return s;
    };
    for (int l = 0; l < L; ++l) {
        const svn_layer& ly = m->layers[l];
        const int K = layer_k(d->layers, l, N, in);
        const float* W = q;  // column-major [N x K]: column k contiguous == row k of W^T
        q += static_cast<int64_t>(N) * K;
        const float* b = q;
        q += N;
        LayerDev& ld = a.layer[l];
        ld.flags = (ly.concat || l == 0 ? kConcat : 0) | (ly.act ? kAct : 0) | (ly.affine ? kAffine : 0) |
                   (ly.residual && l > 0 ? kResidual : 0);
        float* dW = nullptr;
        if ((st = m->upload(W, static_cast<size_t>(N) * K, &dW)) != SVN_OK) return cleanup_fail(st);
        a.wt[l] = dW;
        a.wt_rows[l] = K;
        float* db = nullptr;
        if ((st = m->upload(b, N, &db)) != SVN_OK) return cleanup_fail(st);
        ld.bias = db;
        ld.mb_slot = -1;
        ld.bias_zero = 1;
        for (int i = 0; i < N; ++i)
            if (b[i] != 0.0f) ld.bias_zero = 0;
        ld.wx = nullptr;
        if (ld.flags & kConcat) {
            const int xoff = (l == 0) ? 0 : N;
            ld.wx = dW + static_cast<int64_t>(xoff) * N;  // rows x0, x1, x2 of W^T
            ld.mb_slot = m->n_mb++;
            ld.bias_zero = 0;
            wq_host.insert(wq_host.end(), W + static_cast<int64_t>(xoff + 3) * N,
                           W + static_cast<int64_t>(xoff + 3 + nq) * N);
            wx_host.insert(wx_host.end(), W + static_cast<int64_t>(xoff) * N, W + static_cast<int64_t>(xoff + 3) * N);
            mbbase_host.insert(mbbase_host.end(), b, b + N);
        }
        ld.s = ld.t = nullptr;
        if (ly.affine) {
            const float *gamma = q, *beta = q + N, *mean = q + 2 * N, *var = q + 3 * N;
            q += 4 * N;
            // nn.cpp:108-110 in float: s = gamma / sqrt(var + eps); t = beta - mean * s
            std::vector<float> s(N), t(N);
            for (int i = 0; i < N; ++i) {
                s[i] = gamma[i] / std::sqrt(var[i] + 1e-5f);
                t[i] = std::fma(-mean[i], s[i], beta[i]);
            }
            float *ds = nullptr, *dt = nullptr;
            if ((st = m->upload(s.data(), N, &ds)) != SVN_OK) return cleanup_fail(st);
            if ((st = m->upload(t.data(), N, &dt)) != SVN_OK) return cleanup_fail(st);
            ld.s = ds;
            ld.t = dt;
        }
    }
    {
        float* dwo = nullptr;
        if ((st = m->upload(q, N, &dwo)) != SVN_OK) return cleanup_fail(st);
        a.wo = dwo;
        a.bo = q[N];
    }
    if ((st = m->upload(wq_host.data(), wq_host.size(), &m->d_wq)) != SVN_OK) return cleanup_fail(st);
    if ((st = m->upload(mbbase_host.data(), mbbase_host.size(), &m->d_mbbase)) != SVN_OK) return cleanup_fail(st);
    if ((st = m->upload(wx_host.data(), wx_host.size(), &m->d_wxslots)) != SVN_OK) return cleanup_fail(st);
    a.n_mb = m->n_mb;

    // bf16 tcgen05 weight stream for layers 1..L-1: h part only, per layer the
    // quarter-steps (n-half, k-half) = (0,0) (1,0) (0,1) (1,1), each as K/2/64 chunks
    // of (N/2 rows x 64 k) in the SW128 K-major image the MMA descriptors expect.
    if (N == 256 || N == 512) {
        const int NH = N / 2, KSL = NH / 64;
        const size_t chunk_elems = static_cast<size_t>(NH) * 64;
        std::vector<char> folded;
        const std::vector<float> pbf = fold_affine_bf16(d, params, n_params, folded);
        std::vector<__nv_bfloat16> ws(static_cast<size_t>(L > 1 ? L - 1 : 1) * N * N);
        const float* Wl = pbf.data() + 2 * in;
        size_t pos = 0;
        for (int l = 0; l < L; ++l) {
            const int K = layer_k(d->layers, l, N, in);
            if (l > 0 && N == 256) {
                // ping-pong kernel (width 256): per layer 4 K slabs, each [CTA r: 128 rows] x 64 k
                for (int ks = 0; ks < N / 64; ++ks)
                    for (int r = 0; r < 2; ++r) {
                        uint8_t* blob = reinterpret_cast<uint8_t*>(ws.data() + pos);
                        for (int nr = 0; nr < 128; ++nr)
                            for (int kc = 0; kc < 64; ++kc) {
                                const int n = r * 128 + nr, k = ks * 64 + kc;
                                *reinterpret_cast<__nv_bfloat16*>(blob + sw128_offset(nr, kc, 128)) =
                                    __float2bfloat16_rn(Wl[static_cast<int64_t>(k) * N + n]);
                            }
                        pos += 128 * 64;
                    }
            } else if (l > 0) {
                for (int step = 0; step < 4; ++step) {
                    const int nh = step & 1, kh = step >> 1;
                    for (int ks = 0; ks < KSL; ++ks) {
                        uint8_t* chunk = reinterpret_cast<uint8_t*>(ws.data() + pos);
                        for (int nr = 0; nr < NH; ++nr)
                            for (int kc = 0; kc < 64; ++kc) {
                                const int n = nh * NH + nr, k = (kh * KSL + ks) * 64 + kc;
                                const float w = Wl[static_cast<int64_t>(k) * N + n];
                                *reinterpret_cast<__nv_bfloat16*>(chunk + sw128_offset(nr, kc, NH)) =
                                    __float2bfloat16_rn(w);
                            }
                        pos += chunk_elems;
                    }
                }
            }
            Wl += static_cast<int64_t>(N) * K + N + (d->layers[l].affine ? 4 * N : 0);
        }
        __nv_bfloat16* dws = nullptr;
        if ((st = m->upload(ws.data(), ws.size(), &dws)) != SVN_OK) return cleanup_fail(st);
        a.wstream = dws;
        // CTA-pair kernel: TMA views of the weight stream and of the model-constant
        // K=16 extension rows (bias hi/lo of non-concat layers with a nonzero bias).
        const int BR = N == 256 ? N / 2 : N / 4;  // B rows per CTA per TMA box (128 for both kernels)
        if ((st = encode_blob_map(&a.tmap_w, dws, 128, ws.size() * 2 / 128, BR)) != SVN_OK) return cleanup_fail(st);
        std::vector<uint8_t> xm;
        const float* Wb = pbf.data() + 2 * in;
        std::vector<float> wq_bf, mbbase_bf, wx_bf;  // K0 inputs from the folded parameters
        for (int l = 0; l < L; ++l) {
            const int K = layer_k(d->layers, l, N, in);
            const float* Wfull = Wb;
            const float* b = Wb + static_cast<int64_t>(N) * K;
            LayerDev& ld = a.layer[l];
            ld.ext = 0;
            ld.ext_row = 0;
            bool bias_zero = true;
            for (int n = 0; n < N; ++n)
                if (b[n] != 0.0f) bias_zero = false;
            if (ld.mb_slot >= 0) {
                ld.ext = 2;
                const int xoff = (l == 0) ? 0 : N;
                wq_bf.insert(wq_bf.end(), Wfull + static_cast<int64_t>(xoff + 3) * N,
                             Wfull + static_cast<int64_t>(xoff + 3 + nq) * N);
                wx_bf.insert(wx_bf.end(), Wfull + static_cast<int64_t>(xoff) * N, Wfull + static_cast<int64_t>(xoff + 3) * N);
                mbbase_bf.insert(mbbase_bf.end(), b, b + N);
            } else if (!bias_zero) {
                ld.ext = 1;
                ld.ext_row = static_cast<int64_t>(xm.size() / 32);
                const size_t base = xm.size();
                xm.resize(base + static_cast<size_t>(N) * 32, 0);
                for (int n = 0; n < N; ++n) {
                    int blob_i, rr;
                    if (N == 256) {  // ping-pong layout: blobs [r] of N/2 rows
                        blob_i = n / BR;
                        rr = n % BR;
                    } else {         // pair layout: blobs [n-half][r] of N/4 rows
                        const int nh = n / (N / 2), wi = n % (N / 2);
                        blob_i = nh * 2 + wi / BR;
                        rr = wi % BR;
                    }
                    uint8_t* blob = xm.data() + base + static_cast<size_t>(blob_i * BR) * 32;
                    __nv_bfloat16 hi, lo;
                    split_bf16_host(b[n], hi, lo);
                    *reinterpret_cast<__nv_bfloat16*>(blob + ext_offset(rr, 0)) = hi;
                    *reinterpret_cast<__nv_bfloat16*>(blob + ext_offset(rr, 1)) = lo;
                }
            }
            Wb += static_cast<int64_t>(N) * K + N + (d->layers[l].affine ? 4 * N : 0);
        }
        if (xm.empty()) xm.resize(static_cast<size_t>(BR) * 32, 0);
        uint8_t* dxm = nullptr;
        if ((st = m->upload(xm.data(), xm.size(), &dxm)) != SVN_OK) return cleanup_fail(st);
        if ((st = encode_blob_map(&a.tmap_xm, dxm, 32, xm.size() / 32, BR)) != SVN_OK) return cleanup_fail(st);
        if ((st = m->upload(wq_bf.data(), wq_bf.size(), &m->d_wq_bf)) != SVN_OK) return cleanup_fail(st);
        if ((st = m->upload(mbbase_bf.data(), mbbase_bf.size(), &m->d_mbbase_bf)) != SVN_OK) return cleanup_fail(st);
        if ((st = m->upload(wx_bf.data(), wx_bf.size(), &m->d_wxslots_bf)) != SVN_OK) return cleanup_fail(st);
        m->base_bf16 = a;
        for (int l = 0; l < L; ++l)
            if (folded[static_cast<size_t>(l)]) m->base_bf16.layer[l].flags &= ~kAffine;
        m->base_bf16.bo = pbf[static_cast<size_t>(n_params - 1)];
        m->has_bf16 = true;
    }

    // fp32-accurate tensor-core path (width 256): every weight split into fp16 hi and
    // 2^11-scaled lo' planes, per (layer, quarter step, 64-wide K slab, CTA half r) a
    // [hi: 64 rows][lo': 64 rows] SW128 image; extension rows [main 64][corr 64] per
    // (n-half, r).  Needs |W|, |b| well inside the fp16 range.
    if (N == 256) {
        float wmax = 0.f;
        for (int64_t i = 2 * in; i < n_params; ++i) wmax = std::max(wmax, std::fabs(params[i]));
        if (wmax < 1.0e4f) {
            FusedArgs sa = a;
            auto split_h = [](float x, __half& hi, __half& lo) {
                hi = __float2half_rn(x);
                lo = __float2half_rn((x - __half2float(hi)) * 2048.0f);
            };
            std::vector<uint8_t> ws(static_cast<size_t>(L > 1 ? L - 1 : 1) * 4 * 2 * 2 * 2 * 64 * 128);
            uint8_t* out = ws.data();
            const float* Wl = params + 2 * in;
            for (int l = 0; l < L; ++l) {
                const int K = layer_k(d->layers, l, N, in);
                if (l > 0) {
                    for (int step = 0; step < 4; ++step) {
                        const int nh = step & 1, kh = step >> 1;
                        for (int ks = 0; ks < 2; ++ks)
                            for (int r = 0; r < 2; ++r) {
                                for (int nr = 0; nr < 64; ++nr)
                                    for (int kc = 0; kc < 64; ++kc) {
                                        const int n = nh * 128 + r * 64 + nr, k = (kh * 2 + ks) * 64 + kc;
                                        __half hi, lo;
                                        split_h(Wl[static_cast<int64_t>(k) * N + n], hi, lo);
                                        *reinterpret_cast<__half*>(out + sw128_offset(nr, kc, 64)) = hi;
                                        *reinterpret_cast<__half*>(out + 8192 + sw128_offset(nr, kc, 64)) = lo;
                                    }
                                out += 16384;
                            }
                    }
                }
                Wl += static_cast<int64_t>(N) * K + N + (d->layers[l].affine ? 4 * N : 0);
            }
            uint8_t* dws = nullptr;
            if ((st = m->upload(ws.data(), ws.size(), &dws)) != SVN_OK) return cleanup_fail(st);
            if ((st = encode_blob_map(&sa.tmap_w, dws, 128, ws.size() / 128, 128)) != SVN_OK) return cleanup_fail(st);
            std::vector<uint8_t> xm;
            const float* Wb = params + 2 * in;
            for (int l = 0; l < L; ++l) {
                const int K = layer_k(d->layers, l, N, in);
                const float* b = Wb + static_cast<int64_t>(N) * K;
                LayerDev& ld = sa.layer[l];
                ld.ext_row = 0;
                if (ld.ext == 1) {
                    ld.ext_row = static_cast<int64_t>(xm.size() / 32);
                    const size_t base = xm.size();
                    xm.resize(base + static_cast<size_t>(N) * 2 * 32, 0);
                    for (int n = 0; n < N; ++n) {
                        const int nh = n / 128, wi = n % 128, r = wi / 64, rr = wi % 64;
                        uint8_t* blob = xm.data() + base + static_cast<size_t>((nh * 2 + r) * 128) * 32;
                        __half hi, lo;
                        split_h(b[n], hi, lo);
                        *reinterpret_cast<__half*>(blob + ext_offset(rr, 0)) = hi;         // main: b_h
                        *reinterpret_cast<__half*>(blob + 2048 + ext_offset(rr, 0)) = lo;  // corr: b_l'
                    }
                }
                Wb += static_cast<int64_t>(N) * K + N + (d->layers[l].affine ? 4 * N : 0);
            }
            if (xm.empty()) xm.resize(128 * 32, 0);
            uint8_t* dxm = nullptr;
            if ((st = m->upload(xm.data(), xm.size(), &dxm)) != SVN_OK) return cleanup_fail(st);
            if ((st = encode_blob_map(&sa.tmap_xm, dxm, 32, xm.size() / 32, 128)) != SVN_OK) return cleanup_fail(st);
            m->base_split = sa;
            m->has_split = true;
        }
    }
    *out = m;
    return SVN_OK;
}

SVN_API svn_status svn_model_destroy(svn_model* m) {
    delete m;
    return SVN_OK;
}

}  // extern "C"

namespace {

svn_status check_prec(const svn_model* m, svn_precision prec) {
    if (prec == SVN_PREC_BF16) {
        if (!m->has_bf16) return fail(SVN_ERR_UNSUPPORTED, "bf16 path needs width 256 or 512");
    } else if (prec == SVN_PREC_FP32 || prec == SVN_PREC_FP32_EXACT) {
        if (m->N != 128 && m->N != 256 && m->N != 512)
            return fail(SVN_ERR_UNSUPPORTED, "fp32 path needs width 128, 256 or 512");
    } else if (prec == SVN_PREC_FP32_SPLIT) {
        if (!m->has_split)
            return fail(SVN_ERR_UNSUPPORTED, "fp32_split path needs width 256, >= 2 layers and |W| < 1e4");
    } else {
        return fail(SVN_ERR_INVALID_ARGUMENT, "unknown precision");
    }
    return SVN_OK;
}

// Which fused kernel serves a (model, precision): bf16 tensor cores; fp32-grade split-fp16
// tensor cores (fp32_split, width 256); or SIMT FFMA in the oracle's order (fp32, fp32_exact).
enum class Kind { BF16, SPLIT, SIMT };
Kind kernel_kind(const svn_model*, svn_precision prec) {
    if (prec == SVN_PREC_BF16) return Kind::BF16;
    if (prec == SVN_PREC_FP32_SPLIT) return Kind::SPLIT;
    return Kind::SIMT;
}

int tile_rows(Kind k, int N) { return k == Kind::SIMT ? (N >= 512 ? 64 : 128) : 256; }
// SIMT: a query with fewer big tiles than SMs is cut into 32-row tiles (4 warps per CTA,
// more SMs busy; each output's k-ordered FMA chain is unchanged)
int tile_rows_for(Kind k, int N, int64_t big_tiles, int num_sms) {
    const int t = tile_rows(k, N);
    return (k == Kind::SIMT && big_tiles < num_sms) ? kFp32SmallTile : t;
}

// NVTX range for the duration of a scope (names the entry points and kernels in Nsight).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// Scratch buffers freed on the stream when the call's kernels are done.
struct Scratch {
    cudaStream_t st;
    std::vector<void*> ptrs;
    explicit Scratch(cudaStream_t s) : st(s) {}
    cudaError_t alloc(void** p, size_t bytes) {
        cudaError_t e = cudaMallocAsync(p, bytes ? bytes : 16, st);
        if (e == cudaSuccess) ptrs.push_back(*p);
        return e;
    }
    ~Scratch() {
        for (void* p : ptrs) cudaFreeAsync(p, st);
    }
};

// Per-thread, per-device staging of the host-buffer entry points: one pinned host block and
// one device block, grown on demand and reused, so a call costs one H2D, one D2H and no
// allocation (calls are synchronous, so reuse after the stream sync is safe).
struct Staging {
    int device = -1;
    uint8_t* host = nullptr;
    uint8_t* dev = nullptr;
    size_t bytes = 0;
    cudaError_t reserve(int dev_id, size_t need) {
        if (need <= bytes && device == dev_id) return cudaSuccess;
        release();
        size_t n = 1 << 16;
        while (n < need) n <<= 1;
        cudaError_t e = cudaMallocHost(reinterpret_cast<void**>(&host), n);
        if (e != cudaSuccess) return e;
        e = cudaMalloc(reinterpret_cast<void**>(&dev), n);
        if (e != cudaSuccess) {
            cudaFreeHost(host);
            host = nullptr;
            return e;
        }
        bytes = n;
        device = dev_id;
        return cudaSuccess;
    }
    void release() {
        if (host) cudaFreeHost(host);
        if (dev) {
            int prev = 0;
            cudaGetDevice(&prev);
            cudaSetDevice(device);
            cudaFree(dev);
            cudaSetDevice(prev);
        }
        host = dev = nullptr;
        bytes = 0;
    }
    ~Staging() { release(); }  // thread exit (worker threads come and go)
};

Staging& thread_staging(int device) {
    thread_local Staging st[8];
    thread_local Staging other;
    return (device >= 0 && device < 8) ? st[device] : other;
}

inline size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

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
                      int64_t n_keys, Scratch& sc, cudaStream_t st, bool split = false) {
    uint8_t* ext = nullptr;
    if (split) {  // [motion][slot][n-half][CTA half][main 64 rows | corr 64 rows] x 32 B
        const size_t rows = static_cast<size_t>(M) * (m->n_mb ? m->n_mb : 1) * 2 * m->N;
        SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&ext), rows * 32), "cudaMallocAsync(split ext)");
        svn_status s = encode_blob_map(&a.tmap_xq, ext, 32, rows, 128);
        if (s != SVN_OK) return s;
        SVN_CUDA(launch_split_ext(a, m->d_wq, m->d_mbbase, m->d_wxslots, ext, keys, counters, n_keys, st),
                 "split_ext kernel");
        ++g_launches;
        return SVN_OK;
    }
    const size_t rows = static_cast<size_t>(M) * (m->n_mb ? m->n_mb : 1) * m->N;
    SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&ext), rows * 32), "cudaMallocAsync(motion ext)");
    svn_status s = encode_blob_map(&a.tmap_xq, ext, 32, rows, static_cast<uint32_t>(m->N == 256 ? m->N / 2 : m->N / 4));
    if (s != SVN_OK) return s;
    SVN_CUDA(launch_motion_ext(a, m->d_wq_bf, m->d_mbbase_bf, m->d_wxslots_bf, ext, keys, counters, n_keys, st),
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
    FusedArgs a = kind0 == Kind::SPLIT ? m->base_split : kind0 == Kind::BF16 ? m->base_bf16 : m->base;
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
    const int TM = tile_rows_for(kind, m->N, M * ((P + TM0 - 1) / TM0), m->num_sms);
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
    SVN_CUDA(launch_k1(a, kind, m->num_sms, st), "fused MLP kernel");
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

}  // namespace

extern "C" {

SVN_API svn_status svn_query_min_device(const svn_model* m, svn_precision prec, const float* points, int64_t P,
                                        const float* q01, int64_t M, double margin, float* min_out,
                                        int32_t* argmin_out, uint8_t* free_out, float* per_point, void* stream) {
    if (!min_out || !argmin_out || !free_out) return fail(SVN_ERR_INVALID_ARGUMENT, "query: null output");
    return query_dense(m, prec, points, P, 0, q01, M, margin, min_out, argmin_out, free_out, per_point, nullptr,
                       static_cast<cudaStream_t>(stream));
}

SVN_API svn_status svn_keys_init_device(uint64_t* keys, int64_t M, void* stream) {
    SVN_CUDA(launch_keys_init(reinterpret_cast<unsigned long long*>(keys), M, static_cast<cudaStream_t>(stream)),
             "keys_init kernel");
    ++g_launches;
    return SVN_OK;
}

SVN_API svn_status svn_query_min_keys_device(const svn_model* m, svn_precision prec, const float* points, int64_t P,
                                             int64_t index_offset, const float* q01, int64_t M, uint64_t* keys,
                                             void* stream) {
    if (!keys) return fail(SVN_ERR_INVALID_ARGUMENT, "query: null keys");
    return query_dense(m, prec, points, P, index_offset, q01, M, 0.0, nullptr, nullptr, nullptr, nullptr, keys,
                       static_cast<cudaStream_t>(stream));
}

SVN_API svn_status svn_keys_finalize_device(const uint64_t* keys, int64_t M, double margin, float* min_out,
                                            int32_t* argmin_out, uint8_t* free_out, void* stream) {
    SVN_CUDA(launch_keys_finalize(reinterpret_cast<const unsigned long long*>(keys), M, margin, min_out, argmin_out,
                                  free_out, static_cast<cudaStream_t>(stream)),
             "keys_finalize kernel");
    ++g_launches;
    return SVN_OK;
}

SVN_API svn_status svn_query_min(const svn_model* m, svn_precision prec, const float* points, int64_t P,
                                 const float* q01, int64_t M, double margin, float* min_out, int32_t* argmin_out,
                                 uint8_t* free_out, float* per_point) {
    if (!m) return fail(SVN_ERR_INVALID_ARGUMENT, "query: null model");
    if (P < 1) return fail(SVN_ERR_INVALID_ARGUMENT, "predict_min_distance: empty point cloud");
    if (M < 1) return fail(SVN_ERR_INVALID_ARGUMENT, "query: no motions");
    if (!points || !q01 || !min_out || !argmin_out || !free_out)
        return fail(SVN_ERR_INVALID_ARGUMENT, "query: null buffer");
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
    std::memcpy(sg.host, points, sizeof(float) * 3 * P);
    std::memcpy(sg.host + o_q, q01, sizeof(float) * nq * M);
    svn_status s;
    {
        Scratch sc(st);
        float* dpp = nullptr;
        if (per_point)
            SVN_CUDA(sc.alloc(reinterpret_cast<void**>(&dpp), sizeof(float) * P * M), "cudaMallocAsync");
        SVN_CUDA(cudaMemcpyAsync(sg.dev, sg.host, o_min, cudaMemcpyHostToDevice, st), "H2D points + motions");
        s = query_dense(m, prec, reinterpret_cast<const float*>(sg.dev), P, 0,
                        reinterpret_cast<const float*>(sg.dev + o_q), M, margin,
                        reinterpret_cast<float*>(sg.dev + o_min), reinterpret_cast<int32_t*>(sg.dev + o_arg),
                        sg.dev + o_free, dpp, nullptr, st);
        if (s != SVN_OK) return s;
        SVN_CUDA(cudaMemcpyAsync(sg.host + o_min, sg.dev + o_min, total - o_min, cudaMemcpyDeviceToHost, st),
                 "D2H min/argmin/free");
        if (per_point)
            SVN_CUDA(cudaMemcpyAsync(per_point, dpp, sizeof(float) * P * M, cudaMemcpyDeviceToHost, st), "D2H delta");
    }
    SVN_CUDA(cudaStreamSynchronize(st), "query kernels");
    std::memcpy(min_out, sg.host + o_min, sizeof(float) * M);
    std::memcpy(argmin_out, sg.host + o_arg, sizeof(int32_t) * M);
    std::memcpy(free_out, sg.host + o_free, M);
    return SVN_OK;
}

// forward_eval (nn.cpp:95-130).  Consecutive rows with identical (q0, q1) form one
// motion segment; each segment is cut into tiles of one motion.
static svn_status forward_rows(const svn_model* m, svn_precision prec, const float* raw_host, const float* raw_dev,
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
    const Kind kind = kernel_kind(m, prec);
    const int TM0 = tile_rows(kind, m->N);
    const int nq = 2 * m->dof, TM = tile_rows_for(kind, m->N, (B + TM0 - 1) / TM0, m->num_sms);
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
    FusedArgs a = kind == Kind::SPLIT ? m->base_split : kind == Kind::BF16 ? m->base_bf16 : m->base;
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

SVN_API svn_status svn_forward_eval(const svn_model* m, svn_precision prec, const float* raw, int64_t B, int64_t cols,
                                    float* out) {
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
}

SVN_API svn_status svn_forward_eval_device(const svn_model* m, svn_precision prec, const float* raw, int64_t B,
                                           int64_t cols, float* out, void* stream) {
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
}

SVN_API svn_status svn_predict_min_distance(const svn_model* m, svn_precision prec, const double* cloud, int64_t P,
                                            const double* q0, const double* q1, int32_t dof, double* min_out,
                                            int32_t* argmin_out) {
    if (!m) return fail(SVN_ERR_INVALID_ARGUMENT, "predict_min_distance: null model");
    if (P < 1) return fail(SVN_ERR_INVALID_ARGUMENT, "predict_min_distance: empty point cloud");
    if (3 + 2 * dof != m->in) return fail(SVN_ERR_INVALID_ARGUMENT, "predict_min_distance: motion dof does not match model");
    if (!cloud || !q0 || !q1 || !min_out || !argmin_out)
        return fail(SVN_ERR_INVALID_ARGUMENT, "predict_min_distance: null buffer");
    // nn.cpp:469-473: every coordinate and joint value is cast to float
    std::vector<float> pts(static_cast<size_t>(3 * P)), q(static_cast<size_t>(2 * dof));
    for (int64_t i = 0; i < 3 * P; ++i) pts[i] = static_cast<float>(cloud[i]);
    for (int i = 0; i < dof; ++i) q[i] = static_cast<float>(q0[i]);
    for (int i = 0; i < dof; ++i) q[dof + i] = static_cast<float>(q1[i]);
    float mn = 0.f;
    int32_t idx = 0;
    uint8_t fr = 0;
    svn_status s = svn_query_min(m, prec, pts.data(), P, q.data(), 1, 0.0, &mn, &idx, &fr, nullptr);
    if (s != SVN_OK) return s;
    *min_out = static_cast<double>(mn);
    *argmin_out = idx;
    return SVN_OK;
}

SVN_API svn_status svn_eval_grid(const svn_model* m, svn_precision prec, const double* origin, double voxel_size,
                                 const int32_t* dims, const double* q0, const double* q1, int32_t dof, float* values) {
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
}

static svn_status gcc_args(const svn_robot_desc* r, int32_t steps, GccArgs& a) {
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
static svn_status gcc_run(const svn_robot_desc* robot, const double* points, int64_t P, const double* q01, int64_t M,
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
static svn_status gcc_host(const svn_robot_desc* robot, const double* points, int64_t P, const double* q01, int64_t M,
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

SVN_API svn_status svn_gcc_min_distance_device(const svn_robot_desc* robot, const double* points, int64_t P,
                                               const double* q01, int64_t M, int32_t steps, double margin,
                                               double* dist_out, uint8_t* free_out, void* stream) {
    return gcc_run(robot, points, P, q01, M, steps, margin, false, dist_out, free_out,
                   static_cast<cudaStream_t>(stream));
}

SVN_API svn_status svn_gcc_min_distance(const svn_robot_desc* robot, const double* points, int64_t P,
                                        const double* q01, int64_t M, int32_t steps, double margin, int32_t device,
                                        double* dist_out, uint8_t* free_out) {
    return gcc_host(robot, points, P, q01, M, steps, margin, false, device, dist_out, free_out);
}

// Alg. 1 (collision.cpp:55-107) with both callables on the GPU; see the header.
SVN_API svn_status svn_gcc_nn_search(const svn_model* m, svn_precision prec, const svn_robot_desc* robot,
                                     const double* cloud, int64_t P, const double* q01, int64_t M, int32_t steps,
                                     double margin, int32_t batch, svn_search_result* out) {
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
}

// SVCKPT01 (nn.cpp:482-576): magic, u32 {version, n_blocks, block_dim, input_dim},
// then the Fig. 2 parameter body; strict trailing-byte check.
SVN_API svn_status svn_model_load_checkpoint(const char* path, int32_t device, svn_model** out) {
    if (!path || !out) return fail(SVN_ERR_INVALID_ARGUMENT, "load_checkpoint: null argument");
    const std::string p(path);
    FILE* f = std::fopen(path, "rb");
    if (!f) return fail(SVN_ERR_IO, "cannot open checkpoint: " + p);
    char magic[8];
    if (std::fread(magic, 1, 8, f) != 8 || std::memcmp(magic, "SVCKPT01", 8) != 0) {
        std::fclose(f);
        return fail(SVN_ERR_FORMAT, p + ": not a sweptnet checkpoint");
    }
    uint32_t hdr[4];
    if (std::fread(hdr, sizeof(uint32_t), 4, f) != 4) {
        std::fclose(f);
        return fail(SVN_ERR_TRUNCATION, p + ": file ends inside header");
    }
    if (hdr[0] != 1u) {
        std::fclose(f);
        return fail(SVN_ERR_VERSION, p + ": checkpoint version " + std::to_string(hdr[0]) +
                                         " not supported (expected 1)");
    }
    const int n_blocks = static_cast<int>(hdr[1]), block_dim = static_cast<int>(hdr[2]),
              input_dim = static_cast<int>(hdr[3]);
    if (n_blocks < 1 || block_dim < 1 || input_dim < 5 || (input_dim - 3) % 2 != 0 || n_blocks + 1 > kMaxLayers ||
        input_dim > kMaxIn) {
        std::fclose(f);
        return fail(SVN_ERR_FORMAT, p + ": implausible architecture header");
    }
    std::vector<svn_layer> layers(static_cast<size_t>(n_blocks + 1), svn_layer{1, 1, 1, 1});
    layers[0] = svn_layer{1, 0, 0, 0};
    svn_model_desc d{n_blocks + 1, block_dim, (input_dim - 3) / 2, layers.data()};
    const int64_t n = svn_param_count(&d);
    std::vector<float> params(static_cast<size_t>(n));
    if (std::fread(params.data(), sizeof(float), static_cast<size_t>(n), f) != static_cast<size_t>(n)) {
        std::fclose(f);
        return fail(SVN_ERR_TRUNCATION, p + ": file ends inside tensor data");
    }
    char extra;
    const bool trailing = std::fread(&extra, 1, 1, f) == 1;
    std::fclose(f);
    if (trailing) return fail(SVN_ERR_FORMAT, p + ": trailing bytes after parameters");
    return svn_model_create(&d, params.data(), n, device, out);
}

}  // extern "C"
