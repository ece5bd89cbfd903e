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
  DiagOut dg;       // optional per-matrix diagnostics
  void* ws;         // n >= 9: device workspace (bed_forward_workspace_bytes)
  size_t ws_bytes;  // a smaller workspace solves the batch in chunks
  const PowSpec* pw = nullptr;  // write the spectral power to evecs instead of V
  const ScatSpec* sc = nullptr;  // n <= 8: form A from X (A is ignored)
};

// Workspace bytes the n >= 9 path needs for `batch` matrices in one chunk
// (bed_split_launch.cuh); 0 for n <= 8.  With a smaller workspace the
// batch is solved in chunks; the minimum is split_workspace_bytes(32, ...).
size_t split_workspace_bytes(int64_t batch, int n, bool vecs, int max_steps);

struct BwdArgs {
  const float* V;
  const float* lam;
  const float* gV;
  const float* gL;
  float* gA;
  int64_t batch;
  int n;
  int degree;
  int32_t* status;  // nullable
  int32_t* flags;   // nullable
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
  int merge = 0;    // 1: write status only for a non-positive spectrum (after a forward)
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

// Opt kernel `kern` in to `bytes` of dynamic shared memory on the CURRENT
// device (a per-device function attribute; a no-op at <= 48 KB).  Cached per
// (kernel, device) under a lock, so concurrent callers and several devices in
// one process are both safe (bed_capi.cu).
cudaError_t ensure_smem(const void* kern, size_t bytes);
template <typename K>
inline cudaError_t ensure_smem(K* kern, size_t bytes) {
  return ensure_smem(reinterpret_cast<const void*>(kern), bytes);
}

cudaError_t launch_small(const FwdArgs& a);      // 1 <= n <= 8   (bed_small.cu)
cudaError_t launch_split16(const FwdArgs& a);    // 9 <= n <= 16  (bed_split16.cu)
cudaError_t launch_split24(const FwdArgs& a);    // 17 <= n <= 24 (bed_split24.cu)
cudaError_t launch_split32(const FwdArgs& a);    // 25 <= n <= 32 (bed_split32.cu)
cudaError_t launch_split64(const FwdArgs& a);    // 33 <= n <= 64 (bed_split64.cu)
cudaError_t launch_backward(const BwdArgs& a);   // 1 <= n <= 64  (bed_backward.cu)
cudaError_t launch_power(const PowArgs& a);      // 1 <= n <= 64  (bed_power.cu)
cudaError_t launch_scatter(const ScatArgs& a);   // 1 <= n <= 64  (bed_scatter.cu)

}  // namespace bed
