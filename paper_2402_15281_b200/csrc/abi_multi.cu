// abi_multi.cu — several GPUs of one box from one host process: one
// persistent worker thread per device, each with its own model copy, stream and staging.
//
//   motions sharding (default): worker d evaluates motions [d*M/G, (d+1)*M/G) against the
//     whole cloud through the single-GPU path and writes its slice of the outputs; no
//     communication, results bit-identical to one GPU (every shard runs the whole batch's
//     tile shape, svn_set_whole_batch).
//   points sharding (single-motion batches, M < G): worker d evaluates the point chunk
//     [d*P/G, (d+1)*P/G) into packed u64 keys with global point indices, the shards meet in
//     one NCCL MIN all-reduce of 8 B per motion, and device 0 decodes (min, argmin, class);
//     bit-identical to one GPU by construction (min is order-free, ties keep the lowest index).
//
// The reference's callers are C++ in one process: run_box_world calls predict_min_distance
// from parallel_for workers (bench.cpp:156,193), so this is the entry a drop-in C++ host uses
// to spread a scene's motions over the box.  NCCL is opened with dlopen on first use
// (libnccl.so.2: the system 2.27 here, or the copy a host process has already loaded).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <functional>
#include <memory>
#include <thread>

#include "abi_internal.cuh"

namespace svn {
namespace abi {
namespace {

struct NcclApi {
    ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    std::string why;
    bool ok() const { return comm_init_all && all_reduce && comm_destroy && error_string; }
};

const NcclApi& nccl_api() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.why = std::string("NCCL not loadable: ") + dlerror();
            return a;
        }
        a.comm_init_all = reinterpret_cast<decltype(a.comm_init_all)>(dlsym(h, "ncclCommInitAll"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
        if (!a.ok()) a.why = "NCCL library lacks ncclCommInitAll / ncclAllReduce";
        return a;
    }();
    return api;
}

// A worker thread pinned to one device: runs one job at a time, posted by the caller.
class Worker {
  public:
    Worker() : th_([this] { loop(); }) {}
    ~Worker() {
        {
            std::lock_guard<std::mutex> l(mu_);
            quit_ = true;
        }
        cv_.notify_all();
        th_.join();
    }
    void post(std::function<void()> job) {
        {
            std::lock_guard<std::mutex> l(mu_);
            job_ = std::move(job);
            busy_ = true;
        }
        cv_.notify_all();
    }
    void wait() {
        std::unique_lock<std::mutex> l(mu_);
        cv_.wait(l, [this] { return !busy_; });
    }

  private:
    void loop() {
        for (;;) {
            std::function<void()> job;
            {
                std::unique_lock<std::mutex> l(mu_);
                cv_.wait(l, [this] { return quit_ || (busy_ && job_); });
                if (quit_) return;
                job = std::move(job_);
                job_ = nullptr;
            }
            job();
            {
                std::lock_guard<std::mutex> l(mu_);
                busy_ = false;
            }
            cv_.notify_all();
        }
    }
    std::mutex mu_;
    std::condition_variable cv_;
    std::function<void()> job_;
    bool busy_ = false, quit_ = false;
    std::thread th_;
};

// Workers meet here before the collective, so no rank enters the all-reduce when another
// one has already failed (it would wait for it forever).
class Rendezvous {
  public:
    explicit Rendezvous(int n) : n_(n) {}
    bool arrive_all_ok(bool ok) {
        std::unique_lock<std::mutex> l(mu_);
        ok_ = ok_ && ok;
        const int gen = gen_;
        if (++count_ == n_) {
            count_ = 0;
            ++gen_;
            result_ = ok_;
            ok_ = true;
            cv_.notify_all();
            return result_;
        }
        cv_.wait(l, [&] { return gen_ != gen; });
        return result_;
    }

  private:
    std::mutex mu_;
    std::condition_variable cv_;
    int n_, count_ = 0, gen_ = 0;
    bool ok_ = true, result_ = true;
};

struct Outcome {
    svn_status status = SVN_OK;
    std::string msg;
    int64_t launches = 0;
};

}  // namespace
}  // namespace abi
}  // namespace svn

struct svn_multi {
    std::vector<int32_t> devices;
    std::vector<svn_model*> models;
    std::vector<ncclComm_t> comms;  // empty unless every device is distinct and NCCL loads
    std::string no_comm_why;
    std::vector<std::unique_ptr<svn::abi::Worker>> workers;
    std::mutex call_mu;  // one call at a time: collectives of two calls must not interleave
    std::vector<float*> scene;  // the resident cloud, one whole copy per listed device (svn_multi_set_scene)
    int64_t scene_points = 0;
    void drop_scene() {
        for (size_t d = 0; d < scene.size(); ++d)
            if (scene[d]) {
                svn::abi::DeviceGuard guard(models[d]->device);
                cudaFree(scene[d]);
            }
        scene.clear();
        scene_points = 0;
    }
    ~svn_multi() {
        workers.clear();
        drop_scene();
        if (!comms.empty())
            for (ncclComm_t c : comms) svn::abi::nccl_api().comm_destroy(c);
        for (svn_model* m : models) svn_model_destroy(m);
    }
};

namespace svn {
namespace abi {
namespace {

// Worker threads are persistent: the whole-batch shape (svn_set_whole_batch) is set for one job.
struct WholeBatch {
    WholeBatch(int64_t M, int64_t P) { svn_set_whole_batch(M, P); }
    ~WholeBatch() { svn_set_whole_batch(0, 0); }
};

void record(Outcome& o, svn_status s) {
    if (s != SVN_OK && o.status == SVN_OK) {
        o.status = s;
        o.msg = svn_last_error();
    }
}

// Run job(d) on every worker and collect the outcomes (status, message, launches) in the
// caller's thread-local error / launch state.
svn_status run_all(svn_multi* mg, const std::function<void(int, Outcome&)>& job) {
    const int G = static_cast<int>(mg->devices.size());
    std::vector<Outcome> out(static_cast<size_t>(G));
    for (int d = 0; d < G; ++d)
        mg->workers[d]->post([&, d] {
            const int64_t l0 = g_launches;
            try {
                job(d, out[d]);
            } catch (...) {
                record(out[d], host_exception());
            }
            out[d].launches = g_launches - l0;
        });
    for (int d = 0; d < G; ++d) mg->workers[d]->wait();
    for (const Outcome& o : out) g_launches += o.launches;
    for (const Outcome& o : out)
        if (o.status != SVN_OK) return fail(o.status, o.msg);
    return SVN_OK;
}

}  // namespace
}  // namespace abi
}  // namespace svn

using namespace svn::abi;

extern "C" {

SVN_API svn_status svn_multi_create(const svn_model_desc* desc, const float* params, int64_t n_params,
                                    const int32_t* devices, int32_t n_devices, svn_multi** out) {
    try {
        if (!out) return fail(SVN_ERR_INVALID_ARGUMENT, "multi: null output");
        *out = nullptr;
        if (!devices || n_devices < 1) return fail(SVN_ERR_INVALID_ARGUMENT, "multi: no devices");
        int count = 0;
        SVN_CUDA(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
        for (int d = 0; d < n_devices; ++d)
            if (devices[d] < 0 || devices[d] >= count) return fail(SVN_ERR_INVALID_ARGUMENT, "multi: no such device");
        std::unique_ptr<svn_multi> mg(new svn_multi);
        mg->devices.assign(devices, devices + n_devices);
        for (int d = 0; d < n_devices; ++d) {
            svn_model* m = nullptr;
            const svn_status s = svn_model_create(desc, params, n_params, devices[d], &m);
            if (s != SVN_OK) return s;
            mg->models.push_back(m);
        }
        bool distinct = true;
        for (int i = 0; i < n_devices; ++i)
            for (int j = 0; j < i; ++j)
                if (devices[i] == devices[j]) distinct = false;
        if (!distinct) {
            mg->no_comm_why = "point sharding needs distinct devices (one NCCL rank per GPU)";
        } else if (!nccl_api().ok()) {
            mg->no_comm_why = nccl_api().why;
        } else {
            mg->comms.resize(static_cast<size_t>(n_devices));
            const ncclResult_t r = nccl_api().comm_init_all(mg->comms.data(), n_devices, mg->devices.data());
            if (r != ncclSuccess) {
                mg->comms.clear();
                return fail(SVN_ERR_NCCL, std::string("ncclCommInitAll: ") + nccl_api().error_string(r));
            }
        }
        for (int d = 0; d < n_devices; ++d) mg->workers.emplace_back(new Worker);
        *out = mg.release();
        return SVN_OK;
    } catch (...) {
        return host_exception();
    }
}

SVN_API svn_status svn_multi_destroy(svn_multi* mg) {
    try {
        delete mg;
        return SVN_OK;
    } catch (...) {
        return host_exception();
    }
}

SVN_API int32_t svn_multi_device_count(const svn_multi* mg) {
    return mg ? static_cast<int32_t>(mg->devices.size()) : 0;
}

SVN_API svn_status svn_multi_set_scene(svn_multi* mg, const float* points, int64_t P) {
    try {
        if (!mg) return fail(SVN_ERR_INVALID_ARGUMENT, "multi: null handle");
        if (P < 0 || (P > 0 && !points) || (P == 0 && points))
            return fail(SVN_ERR_INVALID_ARGUMENT, "multi: scene needs points and a point count (NULL, 0 drops it)");
        std::lock_guard<std::mutex> lock(mg->call_mu);
        mg->drop_scene();
        if (P == 0) return SVN_OK;
        mg->scene.assign(mg->devices.size(), nullptr);
        mg->scene_points = P;
        const size_t bytes = sizeof(float) * 3 * static_cast<size_t>(P);
        // the copies to the devices run side by side, one per worker (one host link each)
        const svn_status s = run_all(mg, [&](int d, Outcome& o) {
            DeviceGuard guard(mg->models[d]->device);
            cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&mg->scene[d]), bytes);
            if (e == cudaSuccess) e = cudaMemcpy(mg->scene[d], points, bytes, cudaMemcpyHostToDevice);
            if (e != cudaSuccess) record(o, cuda_fail(e, "scene upload"));
        });
        if (s != SVN_OK) {
            const std::string why = svn_last_error();
            mg->drop_scene();
            return fail(s, why);
        }
        return SVN_OK;
    } catch (...) {
        return host_exception();
    }
}

SVN_API svn_status svn_query_min_multi(svn_multi* mg, svn_precision prec, const float* points, int64_t P,
                                       const float* q01, int64_t M, double margin, svn_shard_mode mode,
                                       float* min_out, int32_t* argmin_out, uint8_t* free_out) {
    try {
        if (!mg) return fail(SVN_ERR_INVALID_ARGUMENT, "query: null model");
        if (P < 1) return fail(SVN_ERR_INVALID_ARGUMENT, "predict_min_distance: empty point cloud");
        if (M < 1) return fail(SVN_ERR_INVALID_ARGUMENT, "query: no motions");
        if (!q01 || !min_out || !argmin_out || !free_out)
            return fail(SVN_ERR_INVALID_ARGUMENT, "query: null buffer");
        NvtxRange nvtx("svn query_min_multi");
        std::lock_guard<std::mutex> lock(mg->call_mu);
        const bool resident = points == nullptr;
        if (resident && mg->scene.empty()) return fail(SVN_ERR_INVALID_ARGUMENT, "query: null buffer");
        if (resident && P != mg->scene_points)
            return fail(SVN_ERR_INVALID_ARGUMENT, "multi: P differs from the resident scene's point count");
        const int G = static_cast<int>(mg->devices.size());
        if (mode == SVN_SHARD_AUTO) mode = M < G ? SVN_SHARD_POINTS : SVN_SHARD_MOTIONS;
        const int64_t nq = 2 * static_cast<int64_t>(mg->models[0]->dof);

        if (mode == SVN_SHARD_MOTIONS && resident) {
            // the cloud is already on every device: per call only this device's motions go in
            // and its slice of (min, argmin, free) comes out
            return run_all(mg, [&](int d, Outcome& o) {
                const int64_t b = d * M / G, e = (d + 1) * M / G, n = e - b;
                if (n < 1) return;
                WholeBatch whole(M, P);
                const svn_model* m = mg->models[d];
                DeviceGuard guard(m->device);
                ensure_pool(m->device);
                cudaStream_t st = thread_stream(m->device);
                auto cu = [&](cudaError_t err, const char* what) {
                    if (err != cudaSuccess) record(o, cuda_fail(err, what));
                    return err == cudaSuccess;
                };
                // one block: [q | min | argmin | free]
                const size_t q_bytes = sizeof(float) * static_cast<size_t>(nq * n);
                const size_t off_min = (q_bytes + 15) & ~size_t(15), off_arg = off_min + sizeof(float) * n,
                             off_free = off_arg + sizeof(int32_t) * n;
                char* blk = nullptr;
                if (!cu(cudaMallocAsync(reinterpret_cast<void**>(&blk), off_free + n, st), "cudaMallocAsync")) return;
                float* dq = reinterpret_cast<float*>(blk);
                float* dmin = reinterpret_cast<float*>(blk + off_min);
                int32_t* darg = reinterpret_cast<int32_t*>(blk + off_arg);
                uint8_t* dfree = reinterpret_cast<uint8_t*>(blk + off_free);
                if (cu(cudaMemcpyAsync(dq, q01 + b * nq, q_bytes, cudaMemcpyHostToDevice, st), "H2D motions")) {
                    record(o, svn_query_min_device(m, prec, mg->scene[d], P, dq, n, margin, dmin, darg, dfree, nullptr, st));
                    if (o.status == SVN_OK)
                        cu(cudaMemcpyAsync(min_out + b, dmin, sizeof(float) * n, cudaMemcpyDeviceToHost, st), "D2H min") &&
                            cu(cudaMemcpyAsync(argmin_out + b, darg, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st),
                               "D2H argmin") &&
                            cu(cudaMemcpyAsync(free_out + b, dfree, n, cudaMemcpyDeviceToHost, st), "D2H free");
                }
                cudaFreeAsync(blk, st);
                cu(cudaStreamSynchronize(st), "resident-scene query");
            });
        }
        if (mode == SVN_SHARD_MOTIONS) {
            return run_all(mg, [&](int d, Outcome& o) {
                const int64_t b = d * M / G, e = (d + 1) * M / G;
                WholeBatch whole(M, P);
                if (e > b)
                    record(o, svn_query_min(mg->models[d], prec, points, P, q01 + b * nq, e - b, margin, min_out + b,
                                            argmin_out + b, free_out + b, nullptr));
            });
        }
        if (mode != SVN_SHARD_POINTS) return fail(SVN_ERR_INVALID_ARGUMENT, "multi: unknown shard mode");
        if (mg->comms.empty()) return fail(SVN_ERR_UNSUPPORTED, "multi: " + mg->no_comm_why);
        Rendezvous meet(G);
        return run_all(mg, [&](int d, Outcome& o) {
            const svn_model* m = mg->models[d];
            const int64_t pb = d * P / G, pe = (d + 1) * P / G;
            WholeBatch whole(M, P);
            DeviceGuard guard(m->device);
            ensure_pool(m->device);
            cudaStream_t st = thread_stream(m->device);
            float *dp = nullptr, *dq = nullptr, *dmin = nullptr;
            uint64_t* keys = nullptr;
            int32_t* darg = nullptr;
            uint8_t* dfree = nullptr;
            auto cu = [&](cudaError_t e, const char* what) {
                if (e != cudaSuccess) record(o, cuda_fail(e, what));
                return e == cudaSuccess;
            };
            bool ok = cu(cudaMallocAsync(reinterpret_cast<void**>(&dq), sizeof(float) * nq * M, st), "cudaMallocAsync") &&
                      cu(cudaMallocAsync(reinterpret_cast<void**>(&keys), sizeof(uint64_t) * M, st), "cudaMallocAsync") &&
                      cu(cudaMemcpyAsync(dq, q01, sizeof(float) * nq * M, cudaMemcpyHostToDevice, st), "H2D motions");
            float* chunk = nullptr;  // this device's point chunk, freed below unless it is the resident scene's
            constexpr int64_t kPiece = int64_t(1) << 20;
            bool piped = false;
            if (ok && resident) {
                dp = mg->scene[d] + 3 * pb;
            } else if (ok) {
                ok = cu(cudaMallocAsync(reinterpret_cast<void**>(&chunk), sizeof(float) * 3 * (pe > pb ? pe - pb : 1), st),
                        "cudaMallocAsync");
                // a large chunk travels in pieces on a second stream while this stream folds the
                // pieces already here into the keys (as svn_query_min does for large clouds)
                piped = ok && pe - pb >= 2 * kPiece;
                if (ok && !piped)
                    ok = cu(cudaMemcpyAsync(chunk, points + 3 * pb, sizeof(float) * 3 * (pe - pb), cudaMemcpyHostToDevice, st),
                            "H2D point chunk");
                dp = chunk;
            }
            if (ok) {
                record(o, svn_keys_init_device(keys, M, st));
                if (o.status == SVN_OK && piped) {
                    cudaStream_t cs = nullptr;
                    cudaEvent_t ev = nullptr;
                    ok = cu(cudaStreamSynchronize(st), "cudaMallocAsync(point chunk)") &&  // the chunk exists before cs writes it
                         cu(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "cudaStreamCreate") &&
                         cu(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
                    for (int64_t p0 = 0; ok && o.status == SVN_OK && p0 < pe - pb; p0 += kPiece) {
                        const int64_t n = std::min<int64_t>(kPiece, pe - pb - p0);
                        ok = cu(cudaMemcpyAsync(chunk + 3 * p0, points + 3 * (pb + p0), sizeof(float) * 3 * n,
                                                cudaMemcpyHostToDevice, cs),
                                "H2D point piece") &&
                             cu(cudaEventRecord(ev, cs), "cudaEventRecord") && cu(cudaStreamWaitEvent(st, ev, 0), "cudaStreamWaitEvent");
                        if (ok) record(o, svn_query_min_keys_device(m, prec, chunk + 3 * p0, n, pb + p0, dq, M, keys, st));
                    }
                    if (cs) cudaStreamSynchronize(cs);
                    if (ev) cudaEventDestroy(ev);
                    if (cs) cudaStreamDestroy(cs);
                } else if (o.status == SVN_OK && pe > pb) {
                    record(o, svn_query_min_keys_device(m, prec, dp, pe - pb, pb, dq, M, keys, st));
                }
                ok = ok && o.status == SVN_OK && cu(cudaStreamSynchronize(st), "point-shard kernels");
            }
            if (meet.arrive_all_ok(ok)) {
                // the one exchange of the path: 8 B per motion, u64 MIN over NVLink
                const ncclResult_t r = nccl_api().all_reduce(keys, keys, static_cast<size_t>(M), ncclUint64, ncclMin,
                                                             mg->comms[d], st);
                if (r != ncclSuccess) {
                    o.status = SVN_ERR_NCCL;
                    o.msg = std::string("ncclAllReduce: ") + nccl_api().error_string(r);
                } else if (d == 0) {
                    ok = cu(cudaMallocAsync(reinterpret_cast<void**>(&dmin), sizeof(float) * M, st), "cudaMallocAsync") &&
                         cu(cudaMallocAsync(reinterpret_cast<void**>(&darg), sizeof(int32_t) * M, st), "cudaMallocAsync") &&
                         cu(cudaMallocAsync(reinterpret_cast<void**>(&dfree), M, st), "cudaMallocAsync");
                    if (ok) record(o, svn_keys_finalize_device(keys, M, margin, dmin, darg, dfree, st));
                    if (ok && o.status == SVN_OK)
                        ok = cu(cudaMemcpyAsync(min_out, dmin, sizeof(float) * M, cudaMemcpyDeviceToHost, st), "D2H min") &&
                             cu(cudaMemcpyAsync(argmin_out, darg, sizeof(int32_t) * M, cudaMemcpyDeviceToHost, st),
                                "D2H argmin") &&
                             cu(cudaMemcpyAsync(free_out, dfree, M, cudaMemcpyDeviceToHost, st), "D2H free");
                }
                cu(cudaStreamSynchronize(st), "all-reduce");
            } else if (o.status == SVN_OK) {
                o.status = SVN_ERR_CUDA;
                o.msg = "multi: another device failed before the all-reduce";
            }
            for (void* p : {static_cast<void*>(chunk), static_cast<void*>(dq), static_cast<void*>(keys),
                            static_cast<void*>(dmin), static_cast<void*>(darg), static_cast<void*>(dfree)})
                if (p) cudaFreeAsync(p, st);
            cudaStreamSynchronize(st);
        });
    } catch (...) {
        return host_exception();
    }
}

SVN_API svn_status svn_query_min_cascade_multi(svn_multi* mg, svn_precision coarse, double band_coarse,
                                               double band_split, const float* points, int64_t P,
                                               const float* q01, int64_t M, double margin, float* min_out,
                                               int32_t* argmin_out, uint8_t* free_out, int64_t* stage_motions) {
    try {
        if (!mg) return fail(SVN_ERR_INVALID_ARGUMENT, "query: null model");
        if (P < 1) return fail(SVN_ERR_INVALID_ARGUMENT, "predict_min_distance: empty point cloud");
        if (M < 1) return fail(SVN_ERR_INVALID_ARGUMENT, "query: no motions");
        if (!points || !q01 || !min_out || !argmin_out || !free_out)
            return fail(SVN_ERR_INVALID_ARGUMENT, "query: null buffer");
        NvtxRange nvtx("svn query_min_cascade_multi");
        std::lock_guard<std::mutex> lock(mg->call_mu);
        const int G = static_cast<int>(mg->devices.size());
        const int64_t nq = 2 * static_cast<int64_t>(mg->models[0]->dof);
        std::vector<int64_t> stages(static_cast<size_t>(3 * G), 0);
        const svn_status s = run_all(mg, [&](int d, Outcome& o) {
            const int64_t b = d * M / G, e = (d + 1) * M / G;
            if (e <= b) return;
            WholeBatch whole(M, P);
            record(o, svn_query_min_cascade(mg->models[d], coarse, band_coarse, band_split, points, P, q01 + b * nq,
                                            e - b, margin, min_out + b, argmin_out + b, free_out + b, &stages[3 * d]));
        });
        if (s != SVN_OK) return s;
        if (stage_motions)
            for (int k = 0; k < 3; ++k) {
                stage_motions[k] = 0;
                for (int d = 0; d < G; ++d) stage_motions[k] += stages[3 * d + k];
            }
        return SVN_OK;
    } catch (...) {
        return host_exception();
    }
}

}  // extern "C"
