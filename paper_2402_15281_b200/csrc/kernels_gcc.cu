// kernels_gcc.cu — the geometric collision checker (GCC) on the GPU.
//
// Exact minimum, over a point cloud and the `steps` configurations of a linear
// joint-space motion, of the signed distance to the posed link capsules:
//   gcc_min_distance  /root/reference/proj/src/collision.cpp:18-24
//   SweptCapsules::sdf (bounding-sphere skip)  sweptvol.cpp:73-84
//   pose_swept_capsules / discretize           sweptvol.cpp:22-71
//   forward_kinematics (Eigen AngleAxis)        robot.cpp:48-67
//   sdf_capsule                                 geometry.cpp:29-36
// `free` = min > margin is the classification gcc_clearance returns (collision.cpp:26-34).
// Double precision as the reference; multiply-adds written as fma() exactly as in the
// CPU restatement (oracle/sweptnet_oracle.c), so the two agree to the last few ulps.
//
// One CTA per (motion, chunk of points): threads pose one configuration each into
// shared memory (FK + bounding sphere), then every thread scans its points.  The
// per-motion minimum is combined with an atomicMin on an order-preserving u64 map of
// the double.
#include <cuda_runtime.h>

#include <cstdint>

#include <mutex>

#include "gcc.cuh"

namespace svn {

__device__ __forceinline__ double dot3(const double* u, const double* v) {
    return fma(u[2], v[2], fma(u[1], v[1], u[0] * v[0]));
}

__device__ __forceinline__ void apply(const double* R, const double* p, const double* x, double* y) {
#pragma unroll
    for (int i = 0; i < 3; ++i) y[i] = fma(R[3 * i + 2], x[2], fma(R[3 * i + 1], x[1], fma(R[3 * i], x[0], p[i])));
}

__device__ __forceinline__ void angle_axis(double ang, const double* ax, double* R) {
    double s, c;
    sincos(ang, &s, &c);
    const double c1 = 1.0 - c;
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

// sdf_capsule (geometry.cpp:29-36) for a capsule pre-posed as (a, ba = b - a, r, inv_bb = 1/|ba|^2
// or 0 for a degenerate segment, which then gives t = 0): one multiply instead of the
// divide; t moves by at most an ulp, the distance by ~1e-16 relative.
// Returns the squared distance to the segment; the capsule distance is sqrt(.) - c[6].
__device__ __forceinline__ double seg_dist2_pre(const double* x, const double* c) {
    double pa[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) pa[k] = x[k] - c[k];
    double t = dot3(pa, c + 3) * c[7];
    t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    double d[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) d[k] = fma(-t, c[3 + k], pa[k]);
    return dot3(d, d);
}

__device__ __forceinline__ unsigned long long orderable64(double v) {
    unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(v));
    if ((u & 0x7fffffffffffffffull) > 0x7ff0000000000000ull) return ~0ull;  // NaN: never the min
    if (u == 0x8000000000000000ull) u = 0ull;
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

__device__ __forceinline__ double from_orderable64(unsigned long long o) {
    const unsigned long long u = (o & 0x8000000000000000ull) ? (o & 0x7fffffffffffffffull) : ~o;
    return __longlong_as_double(static_cast<long long>(u));
}

__global__ void __launch_bounds__(256) gcc_kernel(const __grid_constant__ GccArgs a) {
    extern __shared__ double sm[];
    const int ncap = a.ncap, steps = a.steps;
    double* pc = sm;                                          // [steps][ncap][8]: a, b, r | later a, ba, r, 1/|ba|^2
    double* bounds = sm + static_cast<size_t>(steps) * ncap * 8;  // [steps][4]
    // chunk-major order: the first waves cover the first chunk of every motion, so in
    // early-exit mode a colliding motion is usually flagged before its later chunks start
    const int64_t m = blockIdx.x % a.M;
    const int64_t chunk = blockIdx.x / a.M;
    if (a.early_exit) {
        __shared__ unsigned int skip;
        if (threadIdx.x == 0) skip = *reinterpret_cast<volatile unsigned int*>(a.hit + m);
        __syncthreads();
        if (skip) return;
    }
    const double* q0 = a.q01 + m * 2 * a.dof;
    const double* q1 = q0 + a.dof;

    // pose: thread i -> configuration i (discretize + FK + bounding sphere)
    for (int i = threadIdx.x; i < steps; i += blockDim.x) {
        double q[kGccMaxDof];
        const double denom = steps - 1;
        for (int c = 0; c < a.dof; ++c) {
            if (q0[c] == q1[c] || i == 0)
                q[c] = q0[c];
            else if (i == steps - 1)
                q[c] = q1[c];
            else
                q[c] = fma(static_cast<double>(i), q1[c], static_cast<double>(steps - 1 - i) * q0[c]) / denom;
        }
        double Rt[9], pt[3];
        for (int k = 0; k < 9; ++k) Rt[k] = a.base[(k / 3) * 4 + (k % 3)];
        for (int k = 0; k < 3; ++k) pt[k] = a.base[k * 4 + 3];
        double* out = pc + static_cast<size_t>(i) * ncap * 8;
        int ci = 0;
        for (int j = 0; j < a.dof; ++j) {
            double R[9], M[9];
            angle_axis(q[j], a.joints[j].axis, R);
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
                for (int cc = 0; cc < 3; ++cc)
                    M[3 * r + cc] = fma(Rt[3 * r + 2], R[6 + cc], fma(Rt[3 * r + 1], R[3 + cc], Rt[3 * r] * R[cc]));
#pragma unroll
            for (int k = 0; k < 9; ++k) Rt[k] = M[k];
            double np[3];
            apply(Rt, pt, a.joints[j].offset, np);
            pt[0] = np[0];
            pt[1] = np[1];
            pt[2] = np[2];
            for (; ci < ncap && a.caps[ci].link == j; ++ci) {
                apply(Rt, pt, a.caps[ci].a, out + 8 * ci);
                apply(Rt, pt, a.caps[ci].b, out + 8 * ci + 3);
                out[8 * ci + 6] = a.caps[ci].radius;
            }
        }
        double cen[3] = {0, 0, 0};
        for (int k = 0; k < ncap; ++k)
            for (int d = 0; d < 3; ++d) cen[d] += out[8 * k + d] + out[8 * k + 3 + d];
        for (int d = 0; d < 3; ++d) cen[d] /= 2.0 * ncap;
        double rad = 0;
        for (int k = 0; k < ncap; ++k) {
            double da[3], db[3];
            for (int d = 0; d < 3; ++d) {
                da[d] = out[8 * k + d] - cen[d];
                db[d] = out[8 * k + 3 + d] - cen[d];
            }
            const double na = sqrt(dot3(da, da)), nb = sqrt(dot3(db, db));
            const double e = (na > nb ? na : nb) + out[8 * k + 6];
            rad = rad > e ? rad : e;
        }
        bounds[4 * i + 0] = cen[0];
        bounds[4 * i + 1] = cen[1];
        bounds[4 * i + 2] = cen[2];
        bounds[4 * i + 3] = rad + 1e-9;  // the skip slack of SweptCapsules::sdf, folded in
        // scan form of each capsule: b -> ba = b - a, and 1/|ba|^2 (0 for a degenerate segment)
        for (int k = 0; k < ncap; ++k) {
            double* c = out + 8 * k;
            double ba[3];
            for (int d = 0; d < 3; ++d) ba[d] = c[3 + d] - c[d];
            const double bb = dot3(ba, ba);
            for (int d = 0; d < 3; ++d) c[3 + d] = ba[d];
            c[7] = bb == 0.0 ? 0.0 : 1.0 / bb;
        }
    }
    __syncthreads();

    // scan: SweptCapsules::sdf per point, min over this chunk
    double best = INFINITY;
    const int64_t p0 = chunk * a.points_per_chunk;
    int64_t p1 = p0 + a.points_per_chunk;
    if (p1 > a.P) p1 = a.P;
    for (int64_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
        const double x[3] = {a.points[3 * p], a.points[3 * p + 1], a.points[3 * p + 2]};
        double bp = INFINITY;
        for (int i = 0; i < steps; ++i) {
            // skip when |x - centre| - R - 1e-9 > bp (sweptvol.cpp:73-84), tested on squares:
            // no square root per configuration
            const double thr = bp + bounds[4 * i + 3];
            if (thr < 0.0) continue;
            const double d[3] = {x[0] - bounds[4 * i], x[1] - bounds[4 * i + 1], x[2] - bounds[4 * i + 2]};
            if (dot3(d, d) > thr * thr) continue;
            const double* c = pc + static_cast<size_t>(i) * ncap * 8;
            for (int k = 0; k < ncap; ++k) {
                const double v = sqrt(seg_dist2_pre(x, c + 8 * k)) - c[8 * k + 6];
                bp = v < bp ? v : bp;
            }
        }
        best = bp < best ? bp : best;
        if (a.early_exit && bp <= a.margin) {  // not free: stop this motion everywhere
            *reinterpret_cast<volatile unsigned int*>(a.hit + m) = 1u;
            break;
        }
    }
    // block min -> one atomic per CTA
    unsigned long long key = orderable64(best);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(0xffffffffu, key, o);
        key = w < key ? w : key;
    }
    __shared__ unsigned long long wmin[8];
    if ((threadIdx.x & 31) == 0) wmin[threadIdx.x >> 5] = key;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long k = wmin[0];
        for (int w = 1; w < (blockDim.x + 31) / 32; ++w) k = wmin[w] < k ? wmin[w] : k;
        atomicMin(a.keys + m, k);
    }
}

__global__ void gcc_init_kernel(unsigned long long* keys, int64_t M) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < M) keys[i] = ~0ull;
}

__global__ void gcc_finalize_kernel(const unsigned long long* keys, int64_t M, double margin, double* dist,
                                    uint8_t* free_out) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= M) return;
    const unsigned long long k = keys[i];
    const double v = k == ~0ull ? __longlong_as_double(0x7ff8000000000000ll) : from_orderable64(k);
    dist[i] = v;
    free_out[i] = v > margin ? 1 : 0;  // gcc_clearance: free <=> min > margin (collision.cpp:27-33)
}

size_t gcc_smem_bytes(int steps, int ncap) {
    return sizeof(double) * (static_cast<size_t>(steps) * ncap * 8 + static_cast<size_t>(steps) * 4);
}

cudaError_t launch_gcc(const GccArgs& a, double margin, double* dist, uint8_t* free_out, cudaStream_t st) {
    if (a.M <= 0) return cudaSuccess;
    const unsigned g = static_cast<unsigned>((a.M + 255) / 256);
    gcc_init_kernel<<<g, 256, 0, st>>>(a.keys, a.M);
    const size_t smem = gcc_smem_bytes(a.steps, a.ncap);
    {
        // the opt-in size depends on (steps, capsules): set and launch under one lock so
        // concurrent host callers with different sizes cannot interleave
        static std::mutex mu;
        std::lock_guard<std::mutex> lock(mu);
        cudaError_t e = cudaFuncSetAttribute(gcc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        gcc_kernel<<<static_cast<unsigned>(a.M * a.chunks), 256, smem, st>>>(a);
    }
    gcc_finalize_kernel<<<g, 256, 0, st>>>(a.keys, a.M, margin, dist, free_out);
    return cudaGetLastError();
}

}  // namespace svn
