/*
 * sweptnet_b200.h — C-ABI of the B200-native swept-volume proxy (arXiv 2402.15281).
 *
 * The drop-in boundary for the reference's inference hot path.  Every entry
 * point takes plain pointers and sizes; no C++, Eigen or torch types cross it.
 * Each function cites the reference interface it replaces (paths under
 * /root/reference/proj):
 *
 *   svn_model_create          MlpT<float> construction  include/sweptnet/nn.hpp:16-44
 *   svn_init_params           init_model<float>         include/sweptnet/nn.hpp:80-81, src/nn.cpp:57-93
 *   svn_model_load_checkpoint load_checkpoint           include/sweptnet/nn.hpp:168, src/nn.cpp:524-576
 *   svn_forward_eval          forward_eval<float>       include/sweptnet/nn.hpp:92-93, src/nn.cpp:95-130
 *   svn_predict_min_distance  predict_min_distance      include/sweptnet/nn.hpp:162-163, src/nn.cpp:460-480
 *   svn_query_min             ProxyEvaluator batch for gcc_nn_search_impl (collision.hpp:45,54-55;
 *                             collision.cpp:63-69) and eval_classification (bench.cpp:98-124):
 *                             predict_min_distance over M motions + `proxy > margin` in one call
 *   svn_query_min_keys_device point-sharded partial of the above (new)
 *   svn_eval_grid             NN branch of cmd_reconstruct  src/cli.cpp:240-261
 *   svn_gcc_min_distance      gcc_min_distance / gcc_clearance  src/collision.cpp:18-34
 *   svn_gcc_nn_search         gcc_nn_search / gcc_nn_search_impl  src/collision.cpp:55-107,120-130 (Alg. 1)
 *   svn_keys_finalize_device  decode + margin classification of reduced keys (new)
 *   svn_last_error            std::invalid_argument / IoError what() strings (nn.cpp:98-99,462,465;
 *                             errors.hpp:8-27)
 *
 * Error convention: every function returns an svn_status; 0 = OK.  On failure the
 * thread-local svn_last_error() holds the message.  Messages for the argument
 * errors are the reference's own exception texts, so a C++ shim can rethrow
 * std::invalid_argument(svn_last_error()) unchanged.
 *
 * Threading: all entry points are re-entrant.  Models are immutable after
 * creation (nn.hpp:84-87) and may be shared by any number of threads; each call
 * runs on the caller's stream (device entry points) or on a per-thread stream
 * (host entry points).  run_box_world calls predict_min_distance from
 * parallel_for workers (bench.cpp:156,193), and that pattern is supported.
 */
#ifndef SWEPTNET_B200_H
#define SWEPTNET_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SVN_API __attribute__((visibility("default")))

typedef enum {
    SVN_OK = 0,
    SVN_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    SVN_ERR_CUDA = 2,
    SVN_ERR_OUT_OF_MEMORY = 3,
    SVN_ERR_UNSUPPORTED = 4, /* shape/program the device kernels do not implement */
    SVN_ERR_IO = 5,          /* IoError          errors.hpp:8  */
    SVN_ERR_FORMAT = 6,      /* FormatError      errors.hpp:13 */
    SVN_ERR_TRUNCATION = 7,  /* TruncationError  errors.hpp:18 */
    SVN_ERR_VERSION = 8,     /* VersionError     errors.hpp:23 */
    SVN_ERR_NCCL = 9,        /* NCCL communicator / collective failure (multi-GPU) */
    SVN_ERR_HOST = 10        /* other host-side failure (e.g. a worker thread could not start) */
} svn_status;

/* Arithmetic of the fused MLP kernel.
 *  BF16        tcgen05 tensor cores, bf16 weights/activations, fp32 accumulate
 *              in TMEM; per-point delta within the bound stated per config.
 *  FP32        the FP32 path: SIMT fp32 FMA in the reference's exact accumulation order
 *  FP32_EXACT  (bias, h part, x, q0, q1 — nn.cpp:118-124), bit-identical to the reference
 *              float path up to the documented dot-product order, so the 1e-5 bar holds
 *              with zero error.  The two names are the same path.
 *  FP32_SPLIT  fp32-grade on tcgen05 (width 256 and 512): every operand split into fp16
 *              hi + 2^11-scaled lo, three f16 MMAs per product into two fp32 TMEM
 *              accumulators (the tensor core's per-instruction truncation compensated in the
 *              epilogue), per-motion q-fold.  Not in the reference's rounding order:
 *              per-point delta within the bound of tests/golden/fp32_split_bounds.json —
 *              the 1e-5 FP32 bar at width 256 and for the reference's Fig. 2 networks, a
 *              stated bound of 2.2e-5 to 2.5e-5 for the width-512 plain/DeepSDF networks
 *              (UNSUPPORTED at other widths or when a weight exceeds 1e4).  A row whose
 *              hidden activation reaches the fp16 range
 *              (|h| >= 65520) or whose input is not finite is reported as delta = -inf: its
 *              motion's min is -inf and its class "not free" (handed to the exact checker),
 *              never dropped.
 *  FP16        the BF16 kernels on fp16 operands (width 256 and 512): the same tcgen05
 *              instruction rate with 11 significant bits instead of 8, so the per-network
 *              bound is about 8 times tighter (tests/golden/fp16_bounds.json; DeepSDF 8x512:
 *              0.012 against 0.089, i.e. inside the 0.02 m margin).  UNSUPPORTED when a
 *              (BN-folded) weight is outside the fp16 range; a row whose activations leave
 *              it at run time is reported as delta = -inf (class "not free"), as in
 *              FP32_SPLIT. */
typedef enum {
    SVN_PREC_BF16 = 0,
    SVN_PREC_FP32 = 1,
    SVN_PREC_FP32_EXACT = 2,
    SVN_PREC_FP32_SPLIT = 3,
    SVN_PREC_FP16 = 4
} svn_precision;

/* One hidden layer of a layer program.  Layer 0 reads the
 * normalised input z only; layer l>0 reads [h_{l-1}; z] when concat != 0.
 *   a = W.in + b ; r = act ? max(a,0) : a ; p = affine ? r*s + t : r ;
 *   h = residual ? h_{l-1} + p : p
 * The reference's Fig. 2 network (nn.hpp:11-15) is layer 0 {1,0,0,0} followed
 * by n_blocks layers {1,1,1,1}. */
typedef struct {
    int32_t concat;
    int32_t act;
    int32_t affine;
    int32_t residual;
} svn_layer;

typedef struct {
    int32_t n_layers;        /* hidden layers incl. the input layer, 1..32   */
    int32_t width;           /* N (block_dim); 128, 256 or 512 on device     */
    int32_t dof;             /* input_dim = 3 + 2*dof                        */
    const svn_layer* layers; /* [n_layers]                                    */
} svn_model_desc;

typedef struct svn_model svn_model;

/* Number of floats in the parameter buffer for `desc`:
 *   norm_shift[in], norm_scale[in],
 *   per layer l: W_l column-major [N x K_l] (K_0 = in; K_l = N + concat*in),
 *                b_l[N], if affine: gamma[N], beta[N], running_mean[N], running_var[N],
 *   output_weight[N], output_bias.
 * For the Fig. 2 program this equals the SVCKPT01 body (nn.cpp:507-520). */
SVN_API int64_t svn_param_count(const svn_model_desc* desc);

/* Trainable parameter count as MlpT::param_count (nn.cpp:19-24). */
SVN_API int64_t svn_trainable_param_count(const svn_model_desc* desc);

/* Seeded weights as init_model (nn.cpp:57-93) on std::mt19937_64(seed):
 * bound_mode 0 = uniform(+-1/sqrt(fan_in)) (init_model), 1 = uniform(+-sqrt(6/fan_in))
 * (He-uniform, the BASELINE.json configs).  Writes svn_param_count floats. */
SVN_API svn_status svn_init_params(const svn_model_desc* desc, uint64_t seed, int32_t bound_mode,
                                   float* params_out);

/* Upload a model to `device` and build every device layout (folded BN, bf16
 * pre-swizzled tcgen05 weight stream, fp32 transposed weights). */
SVN_API svn_status svn_model_create(const svn_model_desc* desc, const float* params, int64_t n_params,
                                    int32_t device, svn_model** out);

/* Read a reference SVCKPT01 checkpoint (nn.cpp:499-576) as a Fig. 2 program. */
SVN_API svn_status svn_model_load_checkpoint(const char* path, int32_t device, svn_model** out);

SVN_API svn_status svn_model_destroy(svn_model* model);

/* The layer program a model runs (width, dof, layers) — e.g. of a model read from a
 * checkpoint, whose header fixes it (nn.cpp:535-548: n_blocks, block_dim, input_dim).
 * `layers` may be null (sizes only); else it must hold `capacity` >= n_layers entries. */
SVN_API svn_status svn_model_get_program(const svn_model* model, int32_t* width, int32_t* dof,
                                         int32_t* n_layers, svn_layer* layers, int32_t capacity);

/* Batched proxy, device-resident inputs (pointers are device memory):
 *   points  float [P x 3]            (x, y, z)
 *   q01     float [M x 2*dof]        (q0 | q1 per motion)
 * outputs per motion m:
 *   min_out    float [M]   min over points of delta(x_p, q0_m, q1_m)
 *   argmin_out int32 [M]   lowest index attaining it (nn.cpp:476-478)
 *   free_out   uint8 [M]   double(min) > margin (collision.cpp:68)
 *   per_point  float [M x P] or NULL: every delta (only written when non-NULL)
 * `stream` is a cudaStream_t (NULL = legacy default stream).  Asynchronous. */
SVN_API svn_status svn_query_min_device(const svn_model* model, svn_precision prec, const float* points,
                                        int64_t P, const float* q01, int64_t M, double margin,
                                        float* min_out, int32_t* argmin_out, uint8_t* free_out,
                                        float* per_point, void* stream);

/* Same with HOST buffers; copies in and out, synchronous. */
SVN_API svn_status svn_query_min(const svn_model* model, svn_precision prec, const float* points, int64_t P,
                                 const float* q01, int64_t M, double margin, float* min_out,
                                 int32_t* argmin_out, uint8_t* free_out, float* per_point);

/* svn_query_min with a margin classification that is exact for EVERY motion (new; the
 * classification step of collision.cpp:68 / bench.cpp:108): the batch runs on `coarse` (a
 * tensor-core precision: FP16 or BF16); the motions whose min lies within band_coarse of the
 * margin — the precision's stated bound, tests/golden/{fp16,bf16}_bounds.json — or is not finite
 * (FP16's range report) run again on FP32_SPLIT (when the model has it), and those still within
 * band_split of the margin on the FP32 path, whose min, argmin and class are the reference's bit
 * for bit.  Outside the bands the coarse class already equals the reference's, so free_out equals
 * the FP32 path's for all M motions, at the coarse path's cost plus the few re-evaluated
 * motions.  min_out / argmin_out hold the finest stage evaluated per motion.  stage_motions
 * (int64 [3], or NULL) receives the motions evaluated per stage {coarse, FP32_SPLIT, FP32}.
 * HOST buffers, synchronous. */
SVN_API svn_status svn_query_min_cascade(const svn_model* model, svn_precision coarse, double band_coarse,
                                         double band_split, const float* points, int64_t P, const float* q01,
                                         int64_t M, double margin, float* min_out, int32_t* argmin_out,
                                         uint8_t* free_out, int64_t* stage_motions);

/* Point-sharded partial (device pointers): folds min over this shard's points
 * into keys[M] with atomicMin.  key = (orderable(delta) << 32) | (index_offset + p);
 * the caller initialises keys to UINT64_MAX (svn_keys_init_device) and reduces
 * shards with a u64 MIN all-reduce before svn_keys_finalize_device. */
SVN_API svn_status svn_keys_init_device(uint64_t* keys, int64_t M, void* stream);
SVN_API svn_status svn_query_min_keys_device(const svn_model* model, svn_precision prec, const float* points,
                                             int64_t P, int64_t index_offset, const float* q01, int64_t M,
                                             uint64_t* keys, void* stream);
SVN_API svn_status svn_keys_finalize_device(const uint64_t* keys, int64_t M, double margin, float* min_out,
                                            int32_t* argmin_out, uint8_t* free_out, void* stream);

/* forward_eval<float> (nn.cpp:95-130): raw row-major [B x cols], row = [x, q0, q1];
 * rows may mix motions (consecutive rows with equal q share a motion). HOST buffers. */
SVN_API svn_status svn_forward_eval(const svn_model* model, svn_precision prec, const float* raw, int64_t B,
                                    int64_t cols, float* out);
SVN_API svn_status svn_forward_eval_device(const svn_model* model, svn_precision prec, const float* raw,
                                           int64_t B, int64_t cols, float* out, void* stream);

/* predict_min_distance (nn.cpp:460-480) with the reference's argument types:
 * cloud double [P x 3], q0/q1 double [dof].  HOST buffers. */
SVN_API svn_status svn_predict_min_distance(const svn_model* model, svn_precision prec, const double* cloud,
                                            int64_t P, const double* q0, const double* q1, int32_t dof,
                                            double* min_out, int32_t* argmin_out);

/* Dense-grid evaluation for NN reconstruction (cmd_reconstruct, cli.cpp:240-261): voxel
 * centres origin + voxel_size * (ix, iy, iz) (SdfGrid::voxel_center, sweptvol.hpp:73-75)
 * are generated on the device in double, cast to float, and every centre is evaluated
 * for the single motion (q0, q1).  values: HOST float [dims[0] * dims[1] * dims[2]] in
 * (ix, iy, iz) row-major order, the order of SdfGrid::values. */
SVN_API svn_status svn_eval_grid(const svn_model* model, svn_precision prec, const double* origin, double voxel_size,
                                 const int32_t* dims, const double* q0, const double* q1, int32_t dof,
                                 float* values);

/* ------------------------------------------------ geometric checker (GCC) --
 * The exact swept-volume clearance the proxy is checked against:
 * for each motion, min over points and over the `steps` configurations of
 * discretize(m, steps) (sweptvol.cpp:22-46) of the signed distance to the posed link
 * capsules (forward_kinematics robot.cpp:48-67, sdf_capsule geometry.cpp:29-36), with
 * the bounding-sphere skip of SweptCapsules::sdf (sweptvol.cpp:73-84); double precision.
 *   dist_out[m] = gcc_min_distance (collision.cpp:18-24)
 *   free_out[m] = dist_out[m] > margin = gcc_clearance(...).free (collision.cpp:26-34) */
typedef struct {
    double axis[3];   /* unit rotation axis in the parent frame (Joint::axis, robot.hpp:15) */
    double offset[3]; /* translation after the rotation (Joint::offset, robot.hpp:16) */
} svn_joint;

typedef struct {
    int32_t link; /* link index; capsules sorted by link (link-major, robot.cpp:62-67) */
    int32_t pad;
    double a[3], b[3]; /* segment end points in the link frame */
    double radius;
} svn_capsule;

typedef struct {
    int32_t dof;              /* 1..16 */
    const svn_joint* joints;  /* [dof] */
    int32_t n_capsules;       /* 1..64 */
    const svn_capsule* capsules;
    const double* base_pose;  /* 3x4 row-major isometry, NULL = identity (robot.hpp:26) */
} svn_robot_desc;

/* HOST buffers: points double [P x 3], q01 double [M x 2 dof]; outputs [M]. */
SVN_API svn_status svn_gcc_min_distance(const svn_robot_desc* robot, const double* points, int64_t P,
                                        const double* q01, int64_t M, int32_t steps, double margin, int32_t device,
                                        double* dist_out, uint8_t* free_out);
/* DEVICE buffers on `stream`. */
SVN_API svn_status svn_gcc_min_distance_device(const svn_robot_desc* robot, const double* points, int64_t P,
                                               const double* q01, int64_t M, int32_t steps, double margin,
                                               double* dist_out, uint8_t* free_out, void* stream);

/* ---------------------------------------- Alg. 1: proxy-guided search (§8f) --
 * gcc_nn_search (collision.cpp:120-130 -> gcc_nn_search_impl, collision.cpp:55-107) with
 * both callables on the GPU: every proxy in one batched launch (predict_min_distance's
 * float casts, nn.cpp:466-474), then the geometric checker on the motions in exactly the
 * order the sequential algorithm visits them — first those with proxy > margin in index
 * order, then the rest by proxy descending (stable) — in batches of `batch` motions (<= 0:
 * 64) until the first free one.  found / motion_index / certified_distance are the
 * sequential algorithm's; nn_checks / exact_checks are the counts IT would report (the GPU
 * evaluates every proxy and may check up to batch-1 motions past the answer); the seconds
 * are the wall time of the GPU phases.  HOST buffers: cloud double [P x 3], q01 double
 * [M x 2 dof]. */
typedef struct {
    int32_t found;
    int32_t motion_index;       /* -1 when no motion is free */
    double certified_distance;  /* checker distance of the certified motion */
    int64_t exact_checks;
    int64_t nn_checks;
    double proxy_seconds, exact_seconds, total_seconds;
} svn_search_result;

SVN_API svn_status svn_gcc_nn_search(const svn_model* model, svn_precision prec, const svn_robot_desc* robot,
                                     const double* cloud, int64_t P, const double* q01, int64_t M, int32_t steps,
                                     double margin, int32_t batch, svn_search_result* out);

/* Several GPUs of one box from one host process (the reference's callers
 * run predict_min_distance from parallel_for workers in one process, bench.cpp:156,193).
 * svn_multi_create builds one model per listed device and one persistent worker thread per
 * device; with distinct devices it also opens an NCCL communicator over them.
 * svn_query_min_multi has svn_query_min's contract (HOST buffers, synchronous), split:
 *   SVN_SHARD_MOTIONS  device d takes motions [d*M/G, (d+1)*M/G); no communication;
 *   SVN_SHARD_POINTS   device d takes points [d*P/G, (d+1)*P/G); one NCCL u64 MIN
 *                      all-reduce of the packed (delta, index) keys, 8 B per motion;
 *                      needs distinct devices (UNSUPPORTED otherwise);
 *   SVN_SHARD_AUTO     points when M < G, else motions.
 * Results are bit-identical to one device in every mode and precision (the shards run the
 * whole batch's tile shape, svn_set_whole_batch).  Calls on one svn_multi are serialised.
 * svn_multi_set_scene keeps one scene's cloud resident: the whole cloud is copied once to
 * every device (run_box_world evaluates all of a scene's motions against one cloud,
 * bench.cpp:185-198), and svn_query_min_multi calls with points == NULL run against it — P
 * must then be the scene's point count — moving only the motions in and (min, argmin, free)
 * out per call.  points == NULL, P == 0 drops the scene.  Without a scene, points == NULL is
 * an argument error as before. */
typedef struct svn_multi svn_multi;
typedef enum { SVN_SHARD_AUTO = 0, SVN_SHARD_MOTIONS = 1, SVN_SHARD_POINTS = 2 } svn_shard_mode;
SVN_API svn_status svn_multi_create(const svn_model_desc* desc, const float* params, int64_t n_params,
                                    const int32_t* devices, int32_t n_devices, svn_multi** out);
SVN_API svn_status svn_multi_destroy(svn_multi* multi);
SVN_API int32_t svn_multi_device_count(const svn_multi* multi);
SVN_API svn_status svn_multi_set_scene(svn_multi* multi, const float* points, int64_t P);
SVN_API svn_status svn_query_min_multi(svn_multi* multi, svn_precision prec, const float* points, int64_t P,
                                       const float* q01, int64_t M, double margin, svn_shard_mode mode,
                                       float* min_out, int32_t* argmin_out, uint8_t* free_out);
/* svn_query_min_cascade over the box: device d runs the cascade on motions [d*M/G, (d+1)*M/G)
 * against the whole cloud (no communication); free_out equals the FP32 path's for every motion
 * and every output equals one device's.  stage_motions (int64 [3] or NULL) receives the
 * motions evaluated per stage, summed over the devices.  HOST buffers, synchronous. */
SVN_API svn_status svn_query_min_cascade_multi(svn_multi* multi, svn_precision coarse, double band_coarse,
                                               double band_split, const float* points, int64_t P,
                                               const float* q01, int64_t M, double margin, float* min_out,
                                               int32_t* argmin_out, uint8_t* free_out, int64_t* stage_motions);

/* Shards of one batch.  The tensor-core precisions pick their tile shape from the size of the
 * launch (a launch with fewer 256-row tiles than CTA pairs runs 128-row tiles, for latency),
 * and the two shapes sum the output dot in different orders: results ~1e-6 apart, far inside
 * the precision's bound, but not the same bits.  A caller that evaluates one batch in several
 * calls — motion ranges or point chunks on other devices or ranks — declares the whole
 * batch's shape first; every shard then runs the tile shape the whole batch would, and the
 * results are bit-identical to one call whatever the split, in every precision (the FP32
 * paths are regardless).  Thread-local, applies to svn_query_min, svn_query_min_device and
 * svn_query_min_keys_device until cleared with (0, 0).  svn_query_min_multi does this
 * itself. */
SVN_API void svn_set_whole_batch(int64_t M_total, int64_t P_total);

/* Kernel launches issued by this thread since the last reset (evidence for bench.py). */
SVN_API int64_t svn_launch_count(void);
SVN_API void svn_launch_count_reset(void);

/* Kernel timing for the roofline: between begin and end, every fused-MLP kernel
 * launched by this thread is bracketed by CUDA events on its own stream.  end
 * synchronises those events and returns the summed device time and the count. */
SVN_API void svn_kernel_timing_begin(void);
SVN_API svn_status svn_kernel_timing_end(double* total_ms, int64_t* launches);

SVN_API const char* svn_last_error(void);
SVN_API const char* svn_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SWEPTNET_B200_H */
