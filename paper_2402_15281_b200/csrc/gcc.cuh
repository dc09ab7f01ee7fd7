// gcc.cuh — launch parameters of the GPU geometric collision checker (kernels_gcc.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace svn {

constexpr int kGccMaxDof = 16;
constexpr int kGccMaxCaps = 64;

struct GccJoint {
    double axis[3];
    double offset[3];
};

struct GccCapsule {
    int32_t link;
    int32_t pad;
    double a[3], b[3];
    double radius;
};

struct GccArgs {
    int dof, ncap, steps;
    double base[12];  // 3x4 row-major isometry
    GccJoint joints[kGccMaxDof];
    GccCapsule caps[kGccMaxCaps];
    const double* points;  // [P x 3]
    int64_t P;
    const double* q01;     // [M x 2 dof]
    int64_t M;
    int64_t chunks;            // point chunks per motion
    int64_t points_per_chunk;
    unsigned long long* keys;  // [M] orderable-u64 minima
    // gcc_clearance mode (collision.cpp:26-34): stop a motion as soon as some point is within
    // the margin (its distance is then a partial minimum <= margin; free motions scan fully)
    int early_exit;
    double margin;
    unsigned int* hit;  // [M] set once a point within the margin is found
};

size_t gcc_smem_bytes(int steps, int ncap);
cudaError_t launch_gcc(const GccArgs& a, double margin, double* dist, uint8_t* free_out, cudaStream_t st);

}  // namespace svn
