/*
 * sweptnet_oracle.c — CPU restatement of the reference inference path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * path and the CPU baseline for bench.py.  Only tests/, __graft_entry__.smoke()
 * and bench.py (cpu_baseline leg and --impl reference) may load it.  The
 * product library (paper_2402_15281_b200/) never links, loads or calls it.
 *
 * Parity status: PINNED to the reference's own code.  oracle/ref/Makefile
 * compiles the unmodified reference sources (src/nn.cpp, robot.cpp, geometry.cpp,
 * sha256-checked) against an Eigen-API subset written for this repo
 * (oracle/ref/eigen_subset; Eigen3 is absent here) into oracle/_ref/; its
 * init_model, forward_eval<float/double>, predict_min_distance, make_normalizer and
 * load_checkpoint produced tests/golden/ref_*.npz (tests/golden/make_ref_golden.py),
 * and this file reproduces them bit for bit (tests/test_ref_oracle.py).  Also
 * pinned by the std::mt19937_64 dump (oracle/pin_rng.cpp), the SPEC.md
 * known-answer properties and an independent torch fp64 oracle.  See DESIGN.md §3.
 *
 * What it restates (reference file:line under /root/reference/proj):
 *   Rng / mt19937_64 / uniform      include/sweptnet/rng.hpp:14-26
 *   substream_seed                  include/sweptnet/rng.hpp:68-73
 *   init_model                      src/nn.cpp:57-93
 *   BN fold (eval affine)           src/nn.cpp:104-111
 *   forward_eval                    src/nn.cpp:95-130
 *   predict_min_distance            src/nn.cpp:460-480
 *   margin predicate                src/collision.cpp:68, src/bench.cpp:108
 *   parallel_for partition          src/parallel.cpp:26-53
 *
 * Generalisation ("layer program"): the reference MlpT is the
 * paper's Fig. 2 network only.  A program is a list of hidden layers, each with
 * flags {concat, act, affine, residual}.  Layer 0 always reads z only (the input
 * layer, nn.cpp:118-119).  Layer l>0 reads [h_{l-1}; z] if concat else h_{l-1}.
 *   a    = b_l + sum_k in_k * W_l[:,k]        (bias first, k ascending: h part, then z)
 *   r    = act ? max(a, 0) : a
 *   post = affine ? fma(r, s_l, t_l) : r       (BN folded to s,t in float, nn.cpp:104-111)
 *   h_l  = residual ? h_{l-1} + post : post
 *   out  = sum_k w_o[k] * h_k + b_o
 * Fig. 2 = layer 0 {1,0,0,0} + n_b blocks {1,1,1,1}; this reproduces nn.cpp:116-128.
 *
 * Floating-point contract.  The reference builds with -O3 -march=native and
 * GCC's default -ffp-contract=fast (CMakeLists.txt:31-38); Eigen's column axpy
 * `a += h[k] * W.col(k)` (nn.cpp:119,123,124) then evaluates as one fused
 * multiply-add per element with k ascending.  This file writes every such
 * multiply-add as an explicit fma()/fmaf() and is compiled with
 * -ffp-contract=off, so its results do not depend on compiler flags.  Spots
 * where the reference's contraction is compiler-dependent are fixed here as the
 * contracted form GCC emits for -std=gnu++20 (CMAKE_CXX_STANDARD 20 with
 * extensions on): Rng::uniform = fma(hi-lo, u, lo) (rng.hpp:23), BN shift
 * t = fma(-mu, s, beta) (nn.cpp:110), block update h + fmaf(r, s, t)
 * (nn.cpp:125).  The output dot (nn.cpp:127): rounded products summed in k order,
 * which is what g++ -O3 makes of Eigen's scalar reduction (pinned below); Eigen's
 * vectorised packet tree orders it differently (ISA-dependent, a few e-7 absolute).
 *
 * Parameter buffer layout (float, shared with the C-ABI svn_model_create):
 *   norm_shift[in], norm_scale[in],
 *   per layer l: W_l column-major [N x K_l] (column k = input feature k),
 *                b_l[N], and if affine: gamma[N], beta[N], mean[N], var[N],
 *   w_o[N], b_o.
 * For the Fig. 2 program this is exactly the SVCKPT01 body after its header
 * (nn.cpp:507-520).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------ RNG -- */
/* std::mt19937_64 (the reference's engine, rng.hpp:16) restated from the
 * published MT19937-64 algorithm (Matsumoto & Nishimura 2000). */
typedef struct {
    uint64_t mt[312];
    int mti;
} mt64_t;

static void mt64_seed(mt64_t* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->mti = 312;
}

static uint64_t mt64_next(mt64_t* s) {
    static const uint64_t mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    if (s->mti >= 312) {
        int i;
        for (i = 0; i < 312 - 156; ++i) {
            uint64_t x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
            s->mt[i] = s->mt[i + 156] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        }
        for (; i < 311; ++i) {
            uint64_t x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
            s->mt[i] = s->mt[i + (156 - 312)] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        }
        uint64_t x = (s->mt[311] & UM) | (s->mt[0] & LM);
        s->mt[311] = s->mt[155] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        s->mti = 0;
    }
    uint64_t x = s->mt[s->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

/* rng.hpp:21 — uniform in [0,1) with 53 random bits. */
static double rng_uniform01(mt64_t* s) { return (double)(mt64_next(s) >> 11) * 0x1.0p-53; }
/* rng.hpp:23 — lo + (hi - lo) * u.  GCC contracts this to fma(hi - lo, u, lo)
 * under the reference's -std=gnu++20 -O3 -march=native build (see header). */
static double rng_uniform(mt64_t* s, double lo, double hi) {
    const double u = rng_uniform01(s);
    return fma(hi - lo, u, lo);
}

OR_API uint64_t oracle_mt64_nth(uint64_t seed, int64_t n) {
    mt64_t s;
    mt64_seed(&s, seed);
    uint64_t v = 0;
    for (int64_t i = 0; i < n; ++i) v = mt64_next(&s);
    return v;
}

OR_API void oracle_mt64_stream(uint64_t seed, int64_t n, uint64_t* out) {
    mt64_t s;
    mt64_seed(&s, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = mt64_next(&s);
}

OR_API void oracle_uniform_stream(uint64_t seed, int64_t n, double lo, double hi, double* out) {
    mt64_t s;
    mt64_seed(&s, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = rng_uniform(&s, lo, hi);
}

/* rng.hpp:68-73 — SplitMix64 finaliser. */
OR_API uint64_t oracle_substream_seed(uint64_t base, uint64_t index) {
    uint64_t z = base + 0x9e3779b97f4a7c15ULL * (index + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* --------------------------------------------------------- layer program -- */
#define F_CONCAT 0
#define F_ACT 1
#define F_AFFINE 2
#define F_RESID 3

static int layer_k(const int* flags, int l, int N, int in) {
    if (l == 0) return in;
    return N + (flags[4 * l + F_CONCAT] ? in : 0);
}

/* Number of floats in the parameter buffer. */
OR_API int64_t oracle_param_floats(const int* flags, int L, int N, int dof) {
    const int in = 3 + 2 * dof;
    int64_t n = 2 * (int64_t)in;
    for (int l = 0; l < L; ++l) {
        n += (int64_t)N * layer_k(flags, l, N, in) + N;
        if (flags[4 * l + F_AFFINE]) n += 4 * (int64_t)N;
    }
    return n + N + 1;
}

/* Trainable parameters only (nn.cpp:19-24): W, b, gamma, beta, output. */
OR_API int64_t oracle_trainable_params(const int* flags, int L, int N, int dof) {
    const int in = 3 + 2 * dof;
    int64_t n = 0;
    for (int l = 0; l < L; ++l) {
        n += (int64_t)N * layer_k(flags, l, N, in) + N;
        if (flags[4 * l + F_AFFINE]) n += 2 * (int64_t)N;
    }
    return n + N + 1;
}

/*
 * Seeded init (nn.cpp:57-93).  One Rng stream, tensors in order: layer 0 W,
 * hidden W's, output W; each drawn row-major over [out x in] (nn.cpp:70-71) and
 * stored column-major.  bound_mode 0 = 1/sqrt(fan_in) (init_model), 1 =
 * sqrt(6/fan_in) (He-uniform, BASELINE.json configs).  Biases 0, gamma 1,
 * beta 0, running mean 0, var 1, identity normaliser.
 */
OR_API void oracle_init_params(const int* flags, int L, int N, int dof, uint64_t seed, int bound_mode,
                               float* p) {
    const int in = 3 + 2 * dof;
    mt64_t s;
    mt64_seed(&s, seed);
    float* q = p;
    for (int i = 0; i < in; ++i) q[i] = 0.0f;
    q += in;
    for (int i = 0; i < in; ++i) q[i] = 1.0f;
    q += in;
    for (int l = 0; l < L; ++l) {
        const int K = layer_k(flags, l, N, in);
        const double bound = bound_mode ? sqrt(6.0 / (double)K) : 1.0 / sqrt((double)K);
        for (int r = 0; r < N; ++r)
            for (int c = 0; c < K; ++c) q[(int64_t)c * N + r] = (float)rng_uniform(&s, -bound, bound);
        q += (int64_t)N * K;
        for (int i = 0; i < N; ++i) q[i] = 0.0f; /* bias */
        q += N;
        if (flags[4 * l + F_AFFINE]) {
            for (int i = 0; i < N; ++i) q[i] = 1.0f; /* gamma */
            q += N;
            for (int i = 0; i < N; ++i) q[i] = 0.0f; /* beta */
            q += N;
            for (int i = 0; i < N; ++i) q[i] = 0.0f; /* running mean */
            q += N;
            for (int i = 0; i < N; ++i) q[i] = 1.0f; /* running var */
            q += N;
        }
    }
    {
        const double bound = bound_mode ? sqrt(6.0 / (double)N) : 1.0 / sqrt((double)N);
        for (int c = 0; c < N; ++c) q[c] = (float)rng_uniform(&s, -bound, bound);
        q += N;
        q[0] = 0.0f;
    }
}

/* --------------------------------------------------------------- forward -- */
/* Instantiated for float (production type, nn.cpp:587) and double (test
 * oracle type, nn.cpp:588). */
#define DEFINE_MODEL(S, FMA, SQRT, SUF)                                                              \
    typedef struct {                                                                                 \
        int L, N, in;                                                                                \
        const int* flags;                                                                            \
        const S* shift;                                                                              \
        const S* scale;                                                                              \
        const S* W[64];                                                                              \
        const S* b[64];                                                                              \
        S* s[64];                                                                                    \
        S* t[64];                                                                                    \
        const S* wo;                                                                                 \
        S bo;                                                                                        \
        S* fold; /* owned BN fold storage */                                                         \
    } model_##SUF;                                                                                   \
                                                                                                     \
    static int model_bind_##SUF(model_##SUF* m, const int* flags, int L, int N, int dof, const S* p) { \
        if (L < 1 || L > 64 || N < 1 || dof < 1) return 1;                                           \
        m->L = L;                                                                                    \
        m->N = N;                                                                                    \
        m->in = 3 + 2 * dof;                                                                         \
        m->flags = flags;                                                                            \
        int n_aff = 0;                                                                               \
        for (int l = 0; l < L; ++l) n_aff += flags[4 * l + F_AFFINE] ? 1 : 0;                       \
        m->fold = n_aff ? (S*)malloc(sizeof(S) * 2 * (size_t)N * n_aff) : NULL;                      \
        S* f = m->fold;                                                                              \
        const S* q = p;                                                                              \
        m->shift = q;                                                                                \
        q += m->in;                                                                                  \
        m->scale = q;                                                                                \
        q += m->in;                                                                                  \
        for (int l = 0; l < L; ++l) {                                                                \
            const int K = layer_k(flags, l, N, m->in);                                               \
            m->W[l] = q;                                                                             \
            q += (int64_t)N * K;                                                                     \
            m->b[l] = q;                                                                             \
            q += N;                                                                                  \
            m->s[l] = m->t[l] = NULL;                                                                \
            if (flags[4 * l + F_AFFINE]) {                                                           \
                const S* gamma = q;                                                                  \
                const S* beta = q + N;                                                               \
                const S* mean = q + 2 * N;                                                           \
                const S* var = q + 3 * N;                                                            \
                q += 4 * N;                                                                          \
                m->s[l] = f;                                                                         \
                m->t[l] = f + N;                                                                     \
                f += 2 * N;                                                                          \
                /* nn.cpp:108-110 in S arithmetic: s = g / sqrt(v + eps); t = b - mu * s (contracted) */ \
                for (int i = 0; i < N; ++i) {                                                        \
                    const S sc = gamma[i] / SQRT(var[i] + (S)1e-5);                                  \
                    m->s[l][i] = sc;                                                                 \
                    m->t[l][i] = FMA(-mean[i], sc, beta[i]);                                         \
                }                                                                                    \
            }                                                                                        \
        }                                                                                            \
        m->wo = q;                                                                                   \
        q += N;                                                                                      \
        m->bo = q[0];                                                                                \
        return 0;                                                                                    \
    }                                                                                                \
                                                                                                     \
    /* One row (nn.cpp:117-127).  z: scratch [in], h,a: scratch [N]. */                             \
    static S forward_row_##SUF(const model_##SUF* m, const S* raw, S* z, S* h, S* a) {                \
        const int N = m->N, in = m->in;                                                              \
        for (int k = 0; k < in; ++k) {                                                               \
            z[k] = (raw[k] - m->shift[k]) * m->scale[k];                                             \
        }                                                                                            \
        for (int l = 0; l < m->L; ++l) {                                                             \
            const int* fl = m->flags + 4 * l;                                                        \
            const S* W = m->W[l];                                                                    \
            memcpy(a, m->b[l], sizeof(S) * (size_t)N);                                               \
            int col = 0;                                                                             \
            if (l > 0) {                                                                             \
                for (int k = 0; k < N; ++k, ++col) {                                                 \
                    const S hk = h[k];                                                               \
                    const S* w = W + (int64_t)col * N;                                               \
                    for (int n = 0; n < N; ++n) a[n] = FMA(hk, w[n], a[n]);                          \
                }                                                                                    \
            }                                                                                        \
            if (l == 0 || fl[F_CONCAT]) {                                                            \
                for (int k = 0; k < in; ++k, ++col) {                                                \
                    const S zk = z[k];                                                               \
                    const S* w = W + (int64_t)col * N;                                               \
                    for (int n = 0; n < N; ++n) a[n] = FMA(zk, w[n], a[n]);                          \
                }                                                                                    \
            }                                                                                        \
            const int act = fl[F_ACT], aff = fl[F_AFFINE], res = (l > 0) && fl[F_RESID];             \
            const S* sv = m->s[l];                                                                   \
            const S* tv = m->t[l];                                                                   \
            for (int n = 0; n < N; ++n) {                                                            \
                S r = a[n];                                                                          \
                if (act) r = r > (S)0 ? r : (S)0;                                                    \
                if (aff) r = FMA(r, sv[n], tv[n]);                                                   \
                h[n] = res ? h[n] + r : r;                                                           \
            }                                                                                        \
        }                                                                                            \
        /* nn.cpp:127 as the reference's own build evaluates it (oracle/ref): Eigen's scalar    \
         * redux res = p0; res = res + p_k, whose loop g++ -O3 vectorises as rounded products   \
         * added in k order (no contraction across the vector multiply).  Contract is off here. */ \
        S acc = m->wo[0] * h[0];                                                                     \
        for (int k = 1; k < N; ++k) acc = acc + m->wo[k] * h[k];                                     \
        return acc + m->bo;                                                                          \
    }

DEFINE_MODEL(float, fmaf, sqrtf, f32)
DEFINE_MODEL(double, fma, sqrt, f64)

/* forward_eval (nn.cpp:95-130): raw row-major [B x in] -> out[B].
 * Returns 0, or 1 for invalid argument (width mismatch / empty batch). */
OR_API int oracle_forward_eval_f32(const int* flags, int L, int N, int dof, const float* params,
                                   const float* raw, int64_t B, int64_t cols, float* out) {
    if (cols != 3 + 2 * dof || B < 1) return 1;
    model_f32 m;
    if (model_bind_f32(&m, flags, L, N, dof, params)) return 1;
    float* scratch = (float*)malloc(sizeof(float) * (size_t)(cols + 2 * N));
    for (int64_t r = 0; r < B; ++r)
        out[r] = forward_row_f32(&m, raw + r * cols, scratch, scratch + cols, scratch + cols + N);
    free(scratch);
    free(m.fold);
    return 0;
}

OR_API int oracle_forward_eval_f64(const int* flags, int L, int N, int dof, const double* params,
                                   const double* raw, int64_t B, int64_t cols, double* out) {
    if (cols != 3 + 2 * dof || B < 1) return 1;
    model_f64 m;
    if (model_bind_f64(&m, flags, L, N, dof, params)) return 1;
    double* scratch = (double*)malloc(sizeof(double) * (size_t)(cols + 2 * N));
    for (int64_t r = 0; r < B; ++r)
        out[r] = forward_row_f64(&m, raw + r * cols, scratch, scratch + cols, scratch + cols + N);
    free(scratch);
    free(m.fold);
    return 0;
}

/* predict_min_distance (nn.cpp:460-480): double cloud and q are cast to float
 * per row (nn.cpp:469-473); argmin by strict '<' so ties keep the lowest index
 * and a NaN at row 0 sticks (nn.cpp:476-478).  Returns 0, 1 = empty cloud,
 * 2 = dof mismatch. */
OR_API int oracle_predict_min_distance(const int* flags, int L, int N, int dof, const float* params,
                                       const double* cloud, int64_t P, const double* q0, const double* q1,
                                       int q_dof, double* min_out, int32_t* argmin_out) {
    if (P < 1) return 1;
    if (q_dof != dof) return 2;
    model_f32 m;
    if (model_bind_f32(&m, flags, L, N, dof, params)) return 1;
    const int in = 3 + 2 * dof;
    float* raw = (float*)malloc(sizeof(float) * (size_t)in);
    float* scratch = (float*)malloc(sizeof(float) * (size_t)(in + 2 * N));
    for (int i = 0; i < dof; ++i) raw[3 + i] = (float)q0[i];
    for (int i = 0; i < dof; ++i) raw[3 + dof + i] = (float)q1[i];
    float best_v = 0.0f;
    int32_t best = 0;
    for (int64_t r = 0; r < P; ++r) {
        raw[0] = (float)cloud[3 * r + 0];
        raw[1] = (float)cloud[3 * r + 1];
        raw[2] = (float)cloud[3 * r + 2];
        const float v = forward_row_f32(&m, raw, scratch, scratch + in, scratch + in + N);
        if (r == 0 || v < best_v) {
            if (r == 0) best_v = v, best = 0;
            else best_v = v, best = (int32_t)r;
        }
    }
    *min_out = (double)best_v;
    *argmin_out = best;
    free(raw);
    free(scratch);
    free(m.fold);
    return 0;
}

/* ---------------------------------------------- batched query (baseline) -- */
/* Every (point x motion) pair, per-motion min/argmin and `double(min) > margin`
 * (collision.cpp:68).  points: float [P x 3]; q01: float [M x 2dof] = [q0 | q1].
 * per_point (nullable): float [M x P].  Work items are (motion, point chunk); a
 * motion is cut into chunks only when there are fewer motions than threads.  Items
 * are split over `threads` workers with the contiguous partition of
 * parallel.cpp:33-41; chunk results are merged in ascending chunk order with the
 * same strict '<' as nn.cpp:476-478, so the answer does not depend on `threads`. */
typedef struct {
    const model_f32* m;
    const float* pts;
    int64_t P;
    const float* q01;
    int64_t nchunk, chunk_len;
    int64_t i0, i1; /* item range */
    float* best_v;  /* [items] */
    int32_t* best;  /* [items] */
    float* per_point;
} qjob_t;

static void* query_worker(void* arg) {
    const qjob_t* j = (const qjob_t*)arg;
    const model_f32* m = j->m;
    const int in = m->in, dof = (in - 3) / 2, N = m->N;
    float* raw = (float*)malloc(sizeof(float) * (size_t)in);
    float* scratch = (float*)malloc(sizeof(float) * (size_t)(in + 2 * N));
    for (int64_t it = j->i0; it < j->i1; ++it) {
        const int64_t mi = it / j->nchunk, c = it % j->nchunk;
        const int64_t r0 = c * j->chunk_len;
        const int64_t r1 = r0 + j->chunk_len < j->P ? r0 + j->chunk_len : j->P;
        memcpy(raw + 3, j->q01 + mi * 2 * dof, sizeof(float) * 2 * (size_t)dof);
        float best_v = 0.0f;
        int32_t best = -1;
        for (int64_t r = r0; r < r1; ++r) {
            raw[0] = j->pts[3 * r];
            raw[1] = j->pts[3 * r + 1];
            raw[2] = j->pts[3 * r + 2];
            const float v = forward_row_f32(m, raw, scratch, scratch + in, scratch + in + N);
            if (j->per_point) j->per_point[mi * j->P + r] = v;
            if (best < 0 || v < best_v) {
                best_v = v;
                best = (int32_t)r;
            }
        }
        j->best_v[it] = best_v;
        j->best[it] = best;
    }
    free(raw);
    free(scratch);
    return NULL;
}

OR_API int oracle_query_min(const int* flags, int L, int N, int dof, const float* params, const float* pts,
                            int64_t P, const float* q01, int64_t M, double margin, float* min_out,
                            int32_t* argmin_out, uint8_t* free_out, float* per_point, int threads) {
    if (P < 1 || M < 1) return 1;
    model_f32 m;
    if (model_bind_f32(&m, flags, L, N, dof, params)) return 1;
    const int64_t T = threads < 1 ? 1 : threads;
    int64_t nchunk = M >= T ? 1 : (T + M - 1) / M;
    if (nchunk > P) nchunk = P;
    const int64_t chunk_len = (P + nchunk - 1) / nchunk;
    nchunk = (P + chunk_len - 1) / chunk_len;
    const int64_t items = M * nchunk;
    float* bv = (float*)malloc(sizeof(float) * (size_t)items);
    int32_t* bi = (int32_t*)malloc(sizeof(int32_t) * (size_t)items);
    int64_t workers = T < items ? T : items;
    const int64_t per = (items + workers - 1) / workers;
    qjob_t* jobs = (qjob_t*)calloc((size_t)workers, sizeof(qjob_t));
    pthread_t* tid = (pthread_t*)calloc((size_t)workers, sizeof(pthread_t));
    int64_t launched = 0;
    for (int64_t w = 0; w < workers; ++w) {
        const int64_t b = w * per, e = b + per < items ? b + per : items;
        if (b >= e) break;
        jobs[w] = (qjob_t){&m, pts, P, q01, nchunk, chunk_len, b, e, bv, bi, per_point};
        if (workers == 1)
            query_worker(&jobs[w]);
        else
            pthread_create(&tid[w], NULL, query_worker, &jobs[w]);
        ++launched;
    }
    if (workers > 1)
        for (int64_t w = 0; w < launched; ++w) pthread_join(tid[w], NULL);
    for (int64_t mi = 0; mi < M; ++mi) {
        float best_v = bv[mi * nchunk];
        int32_t best = bi[mi * nchunk];
        for (int64_t c = 1; c < nchunk; ++c)
            if (bv[mi * nchunk + c] < best_v) {
                best_v = bv[mi * nchunk + c];
                best = bi[mi * nchunk + c];
            }
        min_out[mi] = best_v;
        argmin_out[mi] = best;
        free_out[mi] = (double)best_v > margin ? 1 : 0;
    }
    free(bv);
    free(bi);
    free(jobs);
    free(tid);
    free(m.fold);
    return 0;
}

/* ================================================================ GCC -- */
/* Geometric collision checker restated (the ground truth the proxy is checked
 * against):
 *   discretize                  src/sweptvol.cpp:22-46
 *   forward_kinematics          src/robot.cpp:48-60 (Eigen AngleAxis / Isometry3d)
 *   pose_link_capsules          src/robot.cpp:62-67
 *   pose_swept_capsules bounds  src/sweptvol.cpp:48-71
 *   SweptCapsules::sdf          src/sweptvol.cpp:73-84 (bounding-sphere pruning)
 *   sdf_capsule                 src/geometry.cpp:29-36
 *   gcc_min_distance            src/collision.cpp:18-24
 *   gcc_clearance               src/collision.cpp:26-34
 * Double precision throughout, as the reference.  Multiply-adds inside one
 * expression are written as fma() (the reference's GCC -ffp-contract=fast build);
 * the CUDA checker uses the same formulas. */
typedef struct {
    double axis[3], offset[3];
} or_joint;
typedef struct {
    int32_t link;
    double a[3], b[3], r;
} or_capsule;

/* Eigen AngleAxis<double>::toRotationMatrix (Rodrigues), row-major R[9]. */
static void or_angle_axis(double ang, const double* ax, double* R) {
    const double s = sin(ang), c = cos(ang), c1 = 1.0 - c;
    const double sa0 = s * ax[0], sa1 = s * ax[1], sa2 = s * ax[2];
    const double ca0 = c1 * ax[0], ca1 = c1 * ax[1], ca2 = c1 * ax[2];
    double tmp;
    tmp = ca0 * ax[1];
    R[1] = tmp - sa2;
    R[3] = tmp + sa2;
    tmp = ca0 * ax[2];
    R[2] = tmp + sa1;
    R[6] = tmp - sa1;
    tmp = ca1 * ax[2];
    R[5] = tmp - sa0;
    R[7] = tmp + sa0;
    R[0] = fma(ca0, ax[0], c);
    R[4] = fma(ca1, ax[1], c);
    R[8] = fma(ca2, ax[2], c);
}

static double or_dot3(const double* u, const double* v) { return fma(u[2], v[2], fma(u[1], v[1], u[0] * v[0])); }

/* y = R x + p */
static void or_apply(const double* R, const double* p, const double* x, double* y) {
    for (int i = 0; i < 3; ++i) y[i] = fma(R[3 * i + 2], x[2], fma(R[3 * i + 1], x[1], fma(R[3 * i], x[0], p[i])));
}

/* sdf_capsule (geometry.cpp:29-36) */
static double or_sdf_capsule(const double* x, const double* a, const double* b, double r) {
    double pa[3], ba[3];
    for (int k = 0; k < 3; ++k) {
        pa[k] = x[k] - a[k];
        ba[k] = b[k] - a[k];
    }
    const double bb = or_dot3(ba, ba);
    if (bb == 0.0) return sqrt(or_dot3(pa, pa)) - r;
    double t = or_dot3(pa, ba) / bb;
    t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    double d[3];
    for (int k = 0; k < 3; ++k) d[k] = fma(-t, ba[k], pa[k]);
    return sqrt(or_dot3(d, d)) - r;
}

/* Posed sweep of one motion: caps [steps][ncap] (a, b, r) and bounds [steps] (c, R). */
static void or_pose_sweep(const or_joint* J, int dof, const or_capsule* caps, int ncap, const double* base,
                          const double* q0, const double* q1, int steps, double* pc, double* bounds) {
    double q[64];
    const double denom = steps - 1;
    for (int i = 0; i < steps; ++i) {
        for (int c = 0; c < dof; ++c) {
            if (q0[c] == q1[c] || i == 0)
                q[c] = q0[c];
            else if (i == steps - 1)
                q[c] = q1[c];
            else
                q[c] = fma((double)i, q1[c], (double)(steps - 1 - i) * q0[c]) / denom; /* sweptvol.cpp:40 */
        }
        /* forward kinematics: T = base; T = T * rot(axis_j, q_j) * trans(offset_j) */
        double Rt[9], pt[3];
        for (int k = 0; k < 9; ++k) Rt[k] = base[(k / 3) * 4 + (k % 3)];
        for (int k = 0; k < 3; ++k) pt[k] = base[k * 4 + 3];
        int ci = 0;
        double* out = pc + (size_t)i * ncap * 7;
        for (int j = 0; j < dof; ++j) {
            double R[9], M[9];
            or_angle_axis(q[j], J[j].axis, R);
            for (int r = 0; r < 3; ++r)
                for (int cc = 0; cc < 3; ++cc)
                    M[3 * r + cc] = fma(Rt[3 * r + 2], R[6 + cc], fma(Rt[3 * r + 1], R[3 + cc], Rt[3 * r] * R[cc]));
            memcpy(Rt, M, sizeof(M));
            double np[3];
            or_apply(Rt, pt, J[j].offset, np);
            memcpy(pt, np, sizeof(np));
            for (; ci < ncap && caps[ci].link == j; ++ci) {
                or_apply(Rt, pt, caps[ci].a, out + 7 * ci);
                or_apply(Rt, pt, caps[ci].b, out + 7 * ci + 3);
                out[7 * ci + 6] = caps[ci].r;
            }
        }
        /* bounding sphere (sweptvol.cpp:57-67) */
        double cen[3] = {0, 0, 0};
        for (int k = 0; k < ncap; ++k)
            for (int d = 0; d < 3; ++d) cen[d] += out[7 * k + d] + out[7 * k + 3 + d];
        for (int d = 0; d < 3; ++d) cen[d] /= 2.0 * ncap;
        double rad = 0;
        for (int k = 0; k < ncap; ++k) {
            double da[3], db[3];
            for (int d = 0; d < 3; ++d) {
                da[d] = out[7 * k + d] - cen[d];
                db[d] = out[7 * k + 3 + d] - cen[d];
            }
            const double na = sqrt(or_dot3(da, da)), nb = sqrt(or_dot3(db, db));
            const double e = (na > nb ? na : nb) + out[7 * k + 6];
            rad = rad > e ? rad : e;
        }
        bounds[4 * i + 0] = cen[0];
        bounds[4 * i + 1] = cen[1];
        bounds[4 * i + 2] = cen[2];
        bounds[4 * i + 3] = rad;
    }
}

/* SweptCapsules::sdf with the 1e-9-slack bounding-sphere skip (sweptvol.cpp:73-84). */
static double or_sweep_sdf(const double* pc, const double* bounds, int steps, int ncap, const double* x, int prune) {
    double best = INFINITY;
    for (int i = 0; i < steps; ++i) {
        double d[3] = {x[0] - bounds[4 * i], x[1] - bounds[4 * i + 1], x[2] - bounds[4 * i + 2]};
        const double lb = sqrt(or_dot3(d, d)) - bounds[4 * i + 3];
        if (prune && lb - 1e-9 > best) continue;
        const double* c = pc + (size_t)i * ncap * 7;
        for (int k = 0; k < ncap; ++k) {
            const double v = or_sdf_capsule(x, c + 7 * k, c + 7 * k + 3, c[7 * k + 6]);
            best = v < best ? v : best;
        }
    }
    return best;
}

/* gcc_min_distance (early_exit = 0) or gcc_clearance (early_exit = 1) for M motions.
 * joints: [dof] {axis, offset}; caps: [ncap] {link, a, b, r}, link-major; base: 3x4
 * row-major isometry; points double [P x 3]; q01 double [M x 2 dof].  Outputs per motion
 * the distance (exact min, or the clearance scan's value) and free = value > margin. */
OR_API int oracle_gcc(const double* joints, int dof, const double* caps_flat, int ncap, const double* base,
                      const double* points, int64_t P, const double* q01, int64_t M, int steps, double margin,
                      int early_exit, int prune, double* dist_out, uint8_t* free_out) {
    if (P < 1 || steps < 2 || dof < 1 || dof > 64 || ncap < 1) return 1;
    or_joint* J = (or_joint*)malloc(sizeof(or_joint) * (size_t)dof);
    or_capsule* C = (or_capsule*)malloc(sizeof(or_capsule) * (size_t)ncap);
    for (int j = 0; j < dof; ++j)
        for (int k = 0; k < 3; ++k) {
            J[j].axis[k] = joints[6 * j + k];
            J[j].offset[k] = joints[6 * j + 3 + k];
        }
    for (int c = 0; c < ncap; ++c) {
        C[c].link = (int32_t)caps_flat[8 * c];
        for (int k = 0; k < 3; ++k) {
            C[c].a[k] = caps_flat[8 * c + 1 + k];
            C[c].b[k] = caps_flat[8 * c + 4 + k];
        }
        C[c].r = caps_flat[8 * c + 7];
    }
    double* pc = (double*)malloc(sizeof(double) * (size_t)steps * ncap * 7);
    double* bounds = (double*)malloc(sizeof(double) * (size_t)steps * 4);
    for (int64_t m = 0; m < M; ++m) {
        or_pose_sweep(J, dof, C, ncap, base, q01 + m * 2 * dof, q01 + m * 2 * dof + dof, steps, pc, bounds);
        double best = INFINITY;
        int free = 1;
        for (int64_t p = 0; p < P; ++p) {
            const double v = or_sweep_sdf(pc, bounds, steps, ncap, points + 3 * p, prune);
            best = v < best ? v : best;
            if (early_exit && best <= margin) {
                free = 0;
                break;
            }
        }
        dist_out[m] = best;
        free_out[m] = early_exit ? (uint8_t)free : (uint8_t)(best > margin);
    }
    free(J);
    free(C);
    free(pc);
    free(bounds);
    return 0;
}
