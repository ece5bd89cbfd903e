// bed_launch.h -- internal launcher interface between the C ABI
// (bed_capi.cu) and the per-size kernel instantiation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "bed_common.cuh"

namespace bed {

struct FwdArgs {
  const float* A;
  int64_t batch;
  int n;
  float* evals;
  float* evecs;  // null => values only
  int32_t* status;
  int32_t* steps;
  int32_t* flags;
  KernelCfg cfg;
  cudaStream_t stream;
};

struct BwdArgs {
  const float* V;
  const float* lam;
  const float* gV;
  const float* gL;
  float* gA;
  int64_t batch;
  int n;
  int degree;
  cudaStream_t stream;
};

struct PowArgs {
  const float* V;
  const float* lam;
  float* out;
  int32_t* status;
  int32_t* flags;
  int64_t batch;
  int n;
  float p;
  float floor_abs;  // < 0: 1e-12 * lambda_max per matrix
  int needs_positive;
  cudaStream_t stream;
};

struct ScatArgs {
  const float* X;  // (batch, n, m)
  float* out;      // (batch, n, n)
  int64_t batch;
  int n;
  int m;
  float eps;
  cudaStream_t stream;
};

cudaError_t launch_small(const FwdArgs& a);      // 1 <= n <= 8   (bed_small.cu)
cudaError_t launch_split16(const FwdArgs& a);    // 9 <= n <= 16  (bed_split16.cu)
cudaError_t launch_split32(const FwdArgs& a);    // 17 <= n <= 32 (bed_split32.cu)
cudaError_t launch_split64(const FwdArgs& a);    // 33 <= n <= 64 (bed_split64.cu)
cudaError_t launch_backward(const BwdArgs& a);   // 1 <= n <= 64  (bed_backward.cu)
cudaError_t launch_power(const PowArgs& a);      // 1 <= n <= 64  (bed_power.cu)
cudaError_t launch_scatter(const ScatArgs& a);   // 1 <= n <= 64  (bed_scatter.cu)

}  // namespace bed
