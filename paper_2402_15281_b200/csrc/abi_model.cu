// abi_model.cu — C-ABI: errors and counters, parameter counts and seeded init, model
// creation (layer program parse, BN fold, per-kernel device layouts: fp32 rows, the bf16
// tcgen05 weight stream with the Fig. 2 affine fold, the split-fp16 stream), the SVCKPT01
// checkpoint reader.
#include "abi_internal.cuh"

using namespace svn;
using namespace svn::abi;

namespace svn {
namespace abi {


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

// Every C-ABI entry point catches what its C++ body may throw (host allocations, worker
// threads) and reports it as a status: no exception crosses the C boundary.
svn_status host_exception() {
    try {
        throw;
    } catch (const std::bad_alloc&) {
        return fail(SVN_ERR_OUT_OF_MEMORY, "host allocation failed");
    } catch (const std::exception& e) {
        return fail(SVN_ERR_HOST, std::string("host error: ") + e.what());
    } catch (...) {
        return fail(SVN_ERR_HOST, "host error");
    }
}

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

}  // namespace abi
}  // namespace svn

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
    try {
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
    } catch (...) {
        return host_exception();
    }
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
    try {
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
    } catch (...) {
        return host_exception();
    }
}

SVN_API svn_status svn_model_create(const svn_model_desc* d, const float* params, int64_t n_params, int32_t device,
                                    svn_model** out) {
    try {
        svn_status st = validate_desc(d);
        if (st != SVN_OK) return st;
        if (!params || !out) return fail(SVN_ERR_INVALID_ARGUMENT, "model: null params/out");
        if (n_params != svn_param_count(d)) return fail(SVN_ERR_INVALID_ARGUMENT, "model: parameter count mismatch");
        int ndev = 0;
        SVN_CUDA(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
        if (device < 0 || device >= ndev) return fail(SVN_ERR_INVALID_ARGUMENT, "model: no such CUDA device");
        DeviceGuard guard(device);

        auto m = new svn_model();
        static std::atomic<uint64_t> next_serial{1};
        m->serial = next_serial.fetch_add(1);
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
            std::vector<char> folded;
            const std::vector<float> pbf = fold_affine_bf16(d, params, n_params, folded);
            std::vector<float> wq_bf, mbbase_bf, wx_bf;  // K0 inputs from the folded parameters (fp32)
            // One pass per 16-bit operand format: bf16 (precision bf16) and, when every folded
            // parameter fits its range, fp16 (precision fp16: same kernels and instruction rate,
            // 11 significant bits instead of 8).  Elements are written as raw 16-bit patterns.
            auto build16 = [&](FusedArgs& a, bool half) -> svn_status {
                auto cvt16 = [half](float x) -> uint16_t {
                    return half ? __half_as_ushort(__float2half_rn(x)) : __bfloat16_as_ushort(__float2bfloat16_rn(x));
                };
                auto split16 = [half](float x, uint16_t& hi, uint16_t& lo) {
                    if (half) {
                        const __half h = __float2half_rn(x);
                        hi = __half_as_ushort(h);
                        lo = __half_as_ushort(__float2half_rn(x - __half2float(h)));
                    } else {
                        __nv_bfloat16 h, l;
                        split_bf16_host(x, h, l);
                        hi = __bfloat16_as_ushort(h);
                        lo = __bfloat16_as_ushort(l);
                    }
                };
                svn_status st = SVN_OK;
                const int NH = N / 2, KSL = NH / 64;
                const size_t chunk_elems = static_cast<size_t>(NH) * 64;
                std::vector<uint16_t> ws(static_cast<size_t>(L > 1 ? L - 1 : 1) * N * N);
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
                                        *reinterpret_cast<uint16_t*>(blob + sw128_offset(nr, kc, 128)) =
                                            cvt16(Wl[static_cast<int64_t>(k) * N + n]);
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
                                        *reinterpret_cast<uint16_t*>(chunk + sw128_offset(nr, kc, NH)) = cvt16(w);
                                    }
                                pos += chunk_elems;
                            }
                        }
                    }
                    Wl += static_cast<int64_t>(N) * K + N + (d->layers[l].affine ? 4 * N : 0);
                }
                uint16_t* dws = nullptr;
                if ((st = m->upload(ws.data(), ws.size(), &dws)) != SVN_OK) return st;
                a.wstream = dws;
                // CTA-pair kernel: TMA views of the weight stream and of the model-constant
                // K=16 extension rows (bias hi/lo of non-concat layers with a nonzero bias).
                const int BR = N == 256 ? N / 2 : N / 4;  // B rows per CTA per TMA box (128 for both kernels)
                if ((st = encode_blob_map(&a.tmap_w, dws, 128, ws.size() * 2 / 128, BR)) != SVN_OK) return st;
                std::vector<uint8_t> xm;
                const float* Wb = pbf.data() + 2 * in;
                const bool fill_k0 = wq_bf.empty() && mbbase_bf.empty();  // first pass only
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
                        if (fill_k0) {
                            wq_bf.insert(wq_bf.end(), Wfull + static_cast<int64_t>(xoff + 3) * N,
                                         Wfull + static_cast<int64_t>(xoff + 3 + nq) * N);
                            wx_bf.insert(wx_bf.end(), Wfull + static_cast<int64_t>(xoff) * N,
                                         Wfull + static_cast<int64_t>(xoff + 3) * N);
                            mbbase_bf.insert(mbbase_bf.end(), b, b + N);
                        }
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
                            uint16_t hi, lo;
                            split16(b[n], hi, lo);
                            *reinterpret_cast<uint16_t*>(blob + ext_offset(rr, 0)) = hi;
                            *reinterpret_cast<uint16_t*>(blob + ext_offset(rr, 1)) = lo;
                        }
                    }
                    Wb += static_cast<int64_t>(N) * K + N + (d->layers[l].affine ? 4 * N : 0);
                }
                if (xm.empty()) xm.resize(static_cast<size_t>(BR) * 32, 0);
                uint8_t* dxm = nullptr;
                if ((st = m->upload(xm.data(), xm.size(), &dxm)) != SVN_OK) return st;
                if ((st = encode_blob_map(&a.tmap_xm, dxm, 32, xm.size() / 32, BR)) != SVN_OK) return st;
                if (N == 512 && !wq_bf.empty()) {
                    // rows of mixed motions (forward_eval batches whose rows all differ in q): per
                    // (concat slot, n-half, CTA half r) four K=16 slabs of BR rows — [b hi, b lo, W_x
                    // splits] as in motion_ext_kernel but with the model bias, then W_q in (hi, lo, hi)
                    // triples matching the per-row A slabs (z_q hi, z_q hi, z_q lo) of the kernel
                    const int NH = N / 2, n_slots = static_cast<int>(mbbase_bf.size() / N);
                    std::vector<uint8_t> mix(static_cast<size_t>(n_slots) * 2 * 2 * 4 * BR * 32, 0);
                    for (int sl = 0; sl < n_slots; ++sl)
                        for (int n = 0; n < N; ++n) {
                            const int nh = n / NH, wi = n % NH, r = wi / BR, rr = wi % BR;
                            uint8_t* blob = mix.data() + static_cast<size_t>(((sl * 2 + nh) * 2 + r) * 4) * BR * 32;
                            auto put = [&](int sub, int k, uint16_t v) {
                                *reinterpret_cast<uint16_t*>(blob + sub * BR * 32 + ext_offset(rr, k)) = v;
                            };
                            uint16_t hi, lo;
                            split16(mbbase_bf[static_cast<size_t>(sl) * N + n], hi, lo);
                            put(0, 0, hi);
                            put(0, 1, lo);
                            for (int c = 0; c < 3; ++c) {
                                split16(wx_bf[(static_cast<size_t>(sl) * 3 + c) * N + n], hi, lo);
                                put(0, 2 + 3 * c, hi);
                                put(0, 3 + 3 * c, lo);
                                put(0, 4 + 3 * c, hi);
                            }
                            for (int k = 0; k < nq; ++k) {
                                split16(wq_bf[(static_cast<size_t>(sl) * nq + k) * N + n], hi, lo);
                                const int q0 = 3 * k;
                                put(1 + q0 / 16, q0 % 16, hi);
                                put(1 + (q0 + 1) / 16, (q0 + 1) % 16, lo);
                                put(1 + (q0 + 2) / 16, (q0 + 2) % 16, hi);
                            }
                        }
                    uint8_t* dmix = nullptr;
                    if ((st = m->upload(mix.data(), mix.size(), &dmix)) != SVN_OK) return st;
                    if ((st = encode_blob_map(&a.tmap_xmix, dmix, 128, mix.size() / 128, 128)) != SVN_OK) return st;
                    m->has_mixed = 3 * nq <= 48;
                }
                return SVN_OK;
            };  // build16
            if ((st = build16(a, false)) != SVN_OK) return cleanup_fail(st);
            if ((st = m->upload(wq_bf.data(), wq_bf.size(), &m->d_wq_bf)) != SVN_OK) return cleanup_fail(st);
            if ((st = m->upload(mbbase_bf.data(), mbbase_bf.size(), &m->d_mbbase_bf)) != SVN_OK) return cleanup_fail(st);
            if ((st = m->upload(wx_bf.data(), wx_bf.size(), &m->d_wxslots_bf)) != SVN_OK) return cleanup_fail(st);
            m->base_bf16 = a;
            for (int l = 0; l < L; ++l)
                if (folded[static_cast<size_t>(l)]) m->base_bf16.layer[l].flags &= ~kAffine;
            m->base_bf16.bo = pbf[static_cast<size_t>(n_params - 1)];
            m->has_bf16 = true;
            // fp16 operands: every folded parameter must be finite in fp16 (activations that leave
            // the range at run time are reported per row, kernels_bf16_pair.cu)
            float wmax16 = 0.f;
            for (size_t i = static_cast<size_t>(2 * in); i < pbf.size(); ++i) wmax16 = std::max(wmax16, std::fabs(pbf[i]));
            if (wmax16 < 6.0e4f) {
                FusedArgs h = m->base_bf16;
                if ((st = build16(h, true)) != SVN_OK) return cleanup_fail(st);
                h.f16 = 1;
                m->base_f16 = h;
                m->has_f16 = true;
            }
        }

        // fp32-accurate tensor-core path (width 256 and 512): every weight split into fp16 hi
        // and 2^11-scaled lo' planes, per (layer, quarter step, 64-wide K slab, CTA half r) a
        // [hi: BRH rows][lo': BRH rows] SW128 image (BRH = width / 4 B rows per CTA and
        // n-half); extension rows [main BRH][corr BRH] per (n-half, r).  Needs |W|, |b| well
        // inside the fp16 range.
        if (N == 256 || N == 512) {
            float wmax = 0.f;
            for (int64_t i = 2 * in; i < n_params; ++i) wmax = std::max(wmax, std::fabs(params[i]));
            if (wmax < 1.0e4f) {
                FusedArgs sa = a;
                auto split_h = [](float x, __half& hi, __half& lo) {
                    hi = __float2half_rn(x);
                    lo = __float2half_rn((x - __half2float(hi)) * 2048.0f);
                };
                const int NHO = N / 2, BRH = N / 4, KSL = N / 128;
                const size_t plane = static_cast<size_t>(BRH) * 128;
                std::vector<uint8_t> ws(static_cast<size_t>(L > 1 ? L - 1 : 1) * 4 * KSL * 2 * 2 * plane);
                uint8_t* out = ws.data();
                const float* Wl = params + 2 * in;
                for (int l = 0; l < L; ++l) {
                    const int K = layer_k(d->layers, l, N, in);
                    if (l > 0) {
                        for (int step = 0; step < 4; ++step) {
                            const int nh = step & 1, kh = step >> 1;
                            for (int ks = 0; ks < KSL; ++ks)
                                for (int r = 0; r < 2; ++r) {
                                    for (int nr = 0; nr < BRH; ++nr)
                                        for (int kc = 0; kc < 64; ++kc) {
                                            const int n = nh * NHO + r * BRH + nr, k = (kh * KSL + ks) * 64 + kc;
                                            __half hi, lo;
                                            split_h(Wl[static_cast<int64_t>(k) * N + n], hi, lo);
                                            *reinterpret_cast<__half*>(out + sw128_offset(nr, kc, BRH)) = hi;
                                            *reinterpret_cast<__half*>(out + plane + sw128_offset(nr, kc, BRH)) = lo;
                                        }
                                    out += 2 * plane;
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
                            const int nh = n / NHO, wi = n % NHO, r = wi / BRH, rr = wi % BRH;
                            uint8_t* blob = xm.data() + base + static_cast<size_t>((nh * 2 + r) * 2 * BRH) * 32;
                            __half hi, lo;
                            split_h(b[n], hi, lo);
                            *reinterpret_cast<__half*>(blob + ext_offset(rr, 0)) = hi;             // main: b_h
                            *reinterpret_cast<__half*>(blob + BRH * 32 + ext_offset(rr, 0)) = lo;  // corr: b_l'
                        }
                    }
                    Wb += static_cast<int64_t>(N) * K + N + (d->layers[l].affine ? 4 * N : 0);
                }
                if (xm.empty()) xm.resize(static_cast<size_t>(2 * BRH) * 32, 0);
                uint8_t* dxm = nullptr;
                if ((st = m->upload(xm.data(), xm.size(), &dxm)) != SVN_OK) return cleanup_fail(st);
                if ((st = encode_blob_map(&sa.tmap_xm, dxm, 32, xm.size() / 32, static_cast<uint32_t>(2 * BRH))) !=
                    SVN_OK)
                    return cleanup_fail(st);
                // expected truncation loss per MMA instruction, in ulps of the final main
                // accumulator (calibrated); SVN_SPLIT_RZ overrides it (A/B hook)
                static const float rz = [] {
                    const char* e = std::getenv("SVN_SPLIT_RZ");
                    return e ? static_cast<float>(std::atof(e)) : -1.0f;
                }();
                sa.rz_comp = rz >= 0.f ? rz : (N == 256 ? kSplitRzComp256 : kSplitRzComp512);
                m->base_split = sa;
                m->has_split = true;
            }
        }
        *out = m;
        return SVN_OK;
    } catch (...) {
        return host_exception();
    }
}

SVN_API svn_status svn_model_destroy(svn_model* m) {
    try {
        delete m;
        return SVN_OK;
    } catch (...) {
        return host_exception();
    }
}

SVN_API svn_status svn_model_get_program(const svn_model* m, int32_t* width, int32_t* dof, int32_t* n_layers,
                                         svn_layer* layers, int32_t capacity) {
    if (!m || !width || !dof || !n_layers) return fail(SVN_ERR_INVALID_ARGUMENT, "get_program: null argument");
    *width = m->N;
    *dof = m->dof;
    *n_layers = m->L;
    if (layers) {
        if (capacity < m->L) return fail(SVN_ERR_INVALID_ARGUMENT, "get_program: layer buffer too small");
        for (int i = 0; i < m->L; ++i) layers[i] = m->layers[i];
    }
    return SVN_OK;
}

}  // extern "C"

extern "C" {
// SVCKPT01 (nn.cpp:482-576): magic, u32 {version, n_blocks, block_dim, input_dim},
// then the Fig. 2 parameter body; strict trailing-byte check.
SVN_API svn_status svn_model_load_checkpoint(const char* path, int32_t device, svn_model** out) {
    try {
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
    } catch (...) {
        return host_exception();
    }
}

}  // extern "C"
