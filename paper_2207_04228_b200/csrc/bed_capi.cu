// bed_capi.cu -- the extern "C" boundary (include/bed200.h): argument
// checking, size dispatch, and the host-buffer streaming entry point.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>

#include "../../include/bed200.h"
#include "bed_launch.h"

namespace {

thread_local char g_last_cuda[256] = "no error";

int cuda_fail(cudaError_t e, const char* where) {
  snprintf(g_last_cuda, sizeof(g_last_cuda), "%s: %s (%s)", where, cudaGetErrorName(e),
           cudaGetErrorString(e));
  return BED_ERR_CUDA;
}

constexpr float kDeflationFloor = 0x1p-22f;

bool aligned4(const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 3) == 0; }

int check_forward(const float* A, int64_t batch, int32_t n, const float* evals,
                  const float* evecs, const bed_config* cfg) {
  if (!cfg || batch < 0 || n < 1 || n > 64) return BED_ERR_INVALID_ARGUMENT;
  if (cfg->sort < 0 || cfg->sort > 2 || cfg->reserved != 0) return BED_ERR_INVALID_ARGUMENT;
  if (!(cfg->deflation_tol >= 0.0f) || !(cfg->symmetry_tol >= 0.0f)) return BED_ERR_INVALID_ARGUMENT;
  if (batch > 0 && (!A || !evals)) return BED_ERR_INVALID_ARGUMENT;
  if (batch > 0 && cfg->compute_vectors && !evecs) return BED_ERR_INVALID_ARGUMENT;
  if (!aligned4(A) || !aligned4(evals) || !aligned4(evecs)) return BED_ERR_MISALIGNED;
  return BED_SUCCESS;
}

bed::KernelCfg kernel_cfg(const bed_config* cfg, int n) {
  bed::KernelCfg k;
  // FP32 floor: below ~2 eps32 of the equilibrated band a trailing coupling
  // cannot be driven further down (the shifts themselves carry eps32-level
  // error and the second shift of each pair pumps the coupling back up), so a
  // tighter tolerance would only burn the step budget.  Deflating at 2^-22
  // perturbs eigenvalues by < 2^-21 * spectral radius.
  k.eps = cfg->deflation_tol > kDeflationFloor ? cfg->deflation_tol : kDeflationFloor;
  k.sym_tol = cfg->symmetry_tol;
  k.max_steps = cfg->max_double_steps > 0 ? cfg->max_double_steps : 2 * n;  // core.py:270-271
  k.sort = cfg->sort;
  return k;
}

// The n >= 9 path takes its workspace from the device's stream-ordered
// memory pool; keep freed blocks cached in the pool across calls.
void keep_pool_warm() {
  static bool done[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done[dev] = true;
}

cudaError_t dispatch_forward(const bed::FwdArgs& a) {
  if (a.n > 8) keep_pool_warm();
  if (a.n <= 8) return bed::launch_small(a);
  if (a.n <= 16) return bed::launch_split16(a);
  if (a.n <= 32) return bed::launch_split32(a);
  return bed::launch_split64(a);
}

}  // namespace

extern "C" {

int bed_abi_version(void) { return BED200_ABI_VERSION; }

const char* bed_error_string(int code) {
  switch (code) {
    case BED_SUCCESS: return "success";
    case BED_ERR_INVALID_ARGUMENT: return "invalid argument (null pointer, n outside [1, 64], negative batch or bad config)";
    case BED_ERR_MISALIGNED: return "pointer not aligned to its element size";
    case BED_ERR_CUDA: return "CUDA launch or runtime error (see bed_last_cuda_error)";
    case BED_ERR_NO_DEVICE: return "no CUDA device available";
    default: return "unknown error code";
  }
}

const char* bed_last_cuda_error(void) { return g_last_cuda; }

int bed_forward_f32(const float* A, int64_t batch, int32_t n, float* evals, float* evecs,
                    int32_t* status, int32_t* steps, int32_t* flags, const bed_config* cfg,
                    void* stream) {
  int rc = check_forward(A, batch, n, evals, evecs, cfg);
  if (rc) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (flags) {
    cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(int32_t), s);
    if (e != cudaSuccess) return cuda_fail(e, "bed_forward_f32 memset(flags)");
  }
  if (batch == 0) return BED_SUCCESS;
  bed::FwdArgs a{A, batch, n, evals, cfg->compute_vectors ? evecs : nullptr, status, steps,
                 flags, kernel_cfg(cfg, n), s};
  cudaError_t e = dispatch_forward(a);
  if (e != cudaSuccess) return cuda_fail(e, "bed_forward_f32 launch");
  return BED_SUCCESS;
}

int bed_backward_f32(const float* V, const float* evals, const float* gV, const float* gL,
                     float* gA, int64_t batch, int32_t n, int32_t taylor_degree, void* stream) {
  if (batch < 0 || n < 1 || n > 64 || taylor_degree < 0) return BED_ERR_INVALID_ARGUMENT;
  if (batch > 0 && (!V || !evals || !gA)) return BED_ERR_INVALID_ARGUMENT;
  if (!aligned4(V) || !aligned4(evals) || !aligned4(gV) || !aligned4(gL) || !aligned4(gA))
    return BED_ERR_MISALIGNED;
  if (batch == 0) return BED_SUCCESS;
  bed::BwdArgs a{V, evals, gV, gL, gA, batch, n, taylor_degree, static_cast<cudaStream_t>(stream)};
  cudaError_t e = bed::launch_backward(a);
  if (e != cudaSuccess) return cuda_fail(e, "bed_backward_f32 launch");
  return BED_SUCCESS;
}

// Host-buffer entry: the batch streams through the device in chunks on
// three rotating streams, so the H2D copy of chunk i+1 and the D2H copy of
// chunk i-1 overlap the solve of chunk i (copies are only asynchronous when
// the host buffers are page-locked; pageable buffers still give correct,
// serialised results).
int bed_forward_host_f32(const float* A, int64_t batch, int32_t n, float* evals, float* evecs,
                         int32_t* status, int32_t* steps, const bed_config* cfg, int32_t device) {
  int rc = check_forward(A, batch, n, evals, evecs, cfg);
  if (rc) return rc;
  if (batch == 0) return BED_SUCCESS;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return BED_ERR_NO_DEVICE;
  if (device < 0 || device >= ndev) return BED_ERR_INVALID_ARGUMENT;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");

  const bool vecs = cfg->compute_vectors != 0;
  const int64_t nn = (int64_t)n * n;
  const int64_t per = 4 * (nn + n + (vecs ? nn : 0)) + 8;  // bytes in flight per matrix
  const int64_t target = 64ll << 20;                         // ~64 MB per chunk
  const int64_t chunk = std::max<int64_t>(1024, std::min<int64_t>(batch, target / per));
  constexpr int kStreams = 3;
  cudaStream_t streams[kStreams] = {};
  float *dA[kStreams] = {}, *dL[kStreams] = {}, *dV[kStreams] = {};
  int32_t *dS[kStreams] = {}, *dK[kStreams] = {};
  int out = BED_SUCCESS;
  for (int i = 0; i < kStreams && out == BED_SUCCESS; ++i) {
    if ((e = cudaStreamCreateWithFlags(&streams[i], cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaMallocAsync(&dA[i], sizeof(float) * chunk * nn, streams[i])) != cudaSuccess ||
        (e = cudaMallocAsync(&dL[i], sizeof(float) * chunk * n, streams[i])) != cudaSuccess ||
        (vecs && (e = cudaMallocAsync(&dV[i], sizeof(float) * chunk * nn, streams[i])) != cudaSuccess) ||
        (e = cudaMallocAsync(&dS[i], sizeof(int32_t) * chunk, streams[i])) != cudaSuccess ||
        (e = cudaMallocAsync(&dK[i], sizeof(int32_t) * chunk, streams[i])) != cudaSuccess)
      out = cuda_fail(e, "bed_forward_host_f32 allocation");
  }
  for (int64_t off = 0, it = 0; off < batch && out == BED_SUCCESS; off += chunk, ++it) {
    const int i = (int)(it % kStreams);
    const int64_t b = std::min<int64_t>(chunk, batch - off);
    cudaStream_t s = streams[i];
    if ((e = cudaMemcpyAsync(dA[i], A + off * nn, sizeof(float) * b * nn, cudaMemcpyHostToDevice, s)) != cudaSuccess) {
      out = cuda_fail(e, "H2D");
      break;
    }
    bed::FwdArgs a{dA[i], b, n, dL[i], vecs ? dV[i] : nullptr, dS[i], dK[i], nullptr,
                   kernel_cfg(cfg, n), s};
    if ((e = dispatch_forward(a)) != cudaSuccess) {
      out = cuda_fail(e, "bed_forward_host_f32 launch");
      break;
    }
    if ((e = cudaMemcpyAsync(evals + off * n, dL[i], sizeof(float) * b * n, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
        (vecs && (e = cudaMemcpyAsync(evecs + off * nn, dV[i], sizeof(float) * b * nn, cudaMemcpyDeviceToHost, s)) != cudaSuccess) ||
        (status && (e = cudaMemcpyAsync(status + off, dS[i], sizeof(int32_t) * b, cudaMemcpyDeviceToHost, s)) != cudaSuccess) ||
        (steps && (e = cudaMemcpyAsync(steps + off, dK[i], sizeof(int32_t) * b, cudaMemcpyDeviceToHost, s)) != cudaSuccess)) {
      out = cuda_fail(e, "D2H");
      break;
    }
  }
  for (int i = 0; i < kStreams; ++i) {
    if (!streams[i]) continue;
    if (dA[i]) cudaFreeAsync(dA[i], streams[i]);
    if (dL[i]) cudaFreeAsync(dL[i], streams[i]);
    if (dV[i]) cudaFreeAsync(dV[i], streams[i]);
    if (dS[i]) cudaFreeAsync(dS[i], streams[i]);
    if (dK[i]) cudaFreeAsync(dK[i], streams[i]);
    e = cudaStreamSynchronize(streams[i]);
    if (e != cudaSuccess && out == BED_SUCCESS) out = cuda_fail(e, "bed_forward_host_f32 sync");
    cudaStreamDestroy(streams[i]);
  }
  cudaSetDevice(prev);
  return out;
}

}  // extern "C"
