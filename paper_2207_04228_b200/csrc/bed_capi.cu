// bed_capi.cu -- the extern "C" boundary (include/bed200.h): argument
// checking, size dispatch, and the host-buffer streaming entry point.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <omp.h>
#include <sys/mman.h>

#include <algorithm>
#include <mutex>
#include <thread>

#include "../../include/bed200.h"
#include "bed_launch.h"
#include "bed_split_plan.h"

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

// Device memory the library allocates itself (the n >= 9 workspace of
// bed_forward_f32, the slot buffers of bed_forward_host_f32) comes from a
// private stream-ordered pool per device that keeps freed blocks cached --
// the device's default pool and its settings are left alone.  Callers that
// want their own allocator to own the memory use bed_forward_ws_f32.
cudaError_t pool_alloc(void** p, size_t bytes, cudaStream_t s) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  cudaMemPool_t pool;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!pools[dev]) {
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      if ((e = cudaMemPoolCreate(&pools[dev], &props)) != cudaSuccess) return e;
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
    }
    pool = pools[dev];
  }
  return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

// Workspace bed_forward_f32 allocates per call: the whole batch in one chunk
// up to 4 GiB, chunked beyond; halved while the pool refuses.
constexpr size_t kWorkspaceCap = size_t(4) << 30;

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// Bytes of input+output per host-path chunk (env BED_HOST_CHUNK_MB, default 32).
int64_t host_chunk_bytes() {
  static int64_t v = [] {
    const char* e = getenv("BED_HOST_CHUNK_MB");
    long mb = e ? strtol(e, nullptr, 10) : 0;
    return (int64_t)(mb > 0 ? mb : 32) << 20;
  }();
  return v;
}

cudaError_t dispatch_forward(const bed::FwdArgs& a) {
  if (a.n <= 8) return bed::launch_small(a);
  if (a.n <= 16) return bed::launch_split16(a);
  if (a.n <= 24) return bed::launch_split24(a);
  if (a.n <= 32) return bed::launch_split32(a);
  return bed::launch_split64(a);
}

}  // namespace

namespace bed {

cudaError_t ensure_smem(const void* kern, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  struct Entry { const void* fn; int dev; };
  static std::mutex mu;
  static Entry done[512];
  static int ndone = 0;
  std::lock_guard<std::mutex> lock(mu);
  for (int i = 0; i < ndone; ++i)
    if (done[i].fn == kern && done[i].dev == dev) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess && ndone < 512) done[ndone++] = Entry{kern, dev};
  return e;
}

}  // namespace bed

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

size_t bed_forward_workspace_bytes(int64_t batch, int32_t n, const bed_config* cfg) {
  if (!cfg || batch <= 0 || n <= 8 || n > 64) return 0;
  const bed::KernelCfg k = kernel_cfg(cfg, n);
  const bool vecs = cfg->compute_vectors != 0;
  return bed::split_plan((batch + 31) / 32 * 32, n, vecs, k.max_steps).bytes;
}

int bed_forward_ws_f32(const float* A, int64_t batch, int32_t n, float* evals, float* evecs,
                       int32_t* status, int32_t* steps, int32_t* flags, int32_t* diag, float* resid,
                       const bed_config* cfg, void* workspace, size_t workspace_bytes, void* stream) {
  int rc = check_forward(A, batch, n, evals, evecs, cfg);
  if (rc) return rc;
  const bool vecs = cfg->compute_vectors != 0;
  const bed::KernelCfg k = kernel_cfg(cfg, n);
  if (batch > 0 && n > 8 &&
      (!workspace || bed::split_chunk(batch, n, vecs, k.max_steps, workspace_bytes) == 0))
    return BED_ERR_INVALID_ARGUMENT;  // below bed_forward_workspace_bytes(32, n, cfg)
  if ((reinterpret_cast<uintptr_t>(workspace) & 255) != 0 || !aligned4(diag) || !aligned4(resid))
    return BED_ERR_MISALIGNED;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (flags) {
    cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(int32_t), s);
    if (e != cudaSuccess) return cuda_fail(e, "bed_forward_ws_f32 memset(flags)");
  }
  if (batch == 0) return BED_SUCCESS;
  bed::FwdArgs a{A, batch, n, evals, vecs ? evecs : nullptr, status, steps, flags, k, s,
                 bed::DiagOut{diag, resid}, workspace, workspace_bytes};
  cudaError_t e = dispatch_forward(a);
  if (e != cudaSuccess) return cuda_fail(e, "bed_forward_ws_f32 launch");
  return BED_SUCCESS;
}

int bed_forward_f32(const float* A, int64_t batch, int32_t n, float* evals, float* evecs,
                    int32_t* status, int32_t* steps, int32_t* flags, const bed_config* cfg,
                    void* stream) {
  int rc = check_forward(A, batch, n, evals, evecs, cfg);
  if (rc) return rc;
  if (batch == 0 || n <= 8)
    return bed_forward_ws_f32(A, batch, n, evals, evecs, status, steps, flags, nullptr, nullptr, cfg,
                              nullptr, 0, stream);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool vecs = cfg->compute_vectors != 0;
  const int max_steps = kernel_cfg(cfg, n).max_steps;
  size_t bytes = std::min(bed_forward_workspace_bytes(batch, n, cfg), kWorkspaceCap);
  const size_t floor_bytes = bed::split_plan(32, n, vecs, max_steps).bytes;
  bytes = std::max(bytes, floor_bytes);
  void* ws = nullptr;
  cudaError_t e = pool_alloc(&ws, bytes, s);
  while (e == cudaErrorMemoryAllocation && bytes > floor_bytes) {
    cudaGetLastError();  // clear the allocation error and retry smaller
    bytes = std::max(floor_bytes, bytes / 2);
    e = pool_alloc(&ws, bytes, s);
  }
  if (e != cudaSuccess) return cuda_fail(e, "bed_forward_f32 workspace");
  rc = bed_forward_ws_f32(A, batch, n, evals, evecs, status, steps, flags, nullptr, nullptr, cfg, ws,
                          bytes, stream);
  e = cudaFreeAsync(ws, s);
  if (rc == BED_SUCCESS && e != cudaSuccess) return cuda_fail(e, "bed_forward_f32 free");
  return rc;
}

// Largest n whose spectral power is fused into the forward's epilogue; above it
// the per-thread row products of the fold lose to the tiled power kernel
// (measured 65536 x 32^2: 1.83 fused vs 1.49 ms composed; 8192 x 64^2: 2.12 vs 1.59).
constexpr int kFusedPowerMaxN = 24;

size_t bed_forward_power_workspace_bytes(int64_t batch, int32_t n, const bed_config* cfg) {
  if (!cfg || batch <= 0 || n <= 8 || n > 64) return 0;
  bed_config c = *cfg;
  c.compute_vectors = 1;
  // n > kFusedPowerMaxN: V in the workspace, then the tiled power kernel
  return (n > kFusedPowerMaxN ? align_up(sizeof(float) * (size_t)batch * n * n) : 0) +
         bed_forward_workspace_bytes(batch, n, &c);
}

int bed_forward_power_f32(const float* A, int64_t batch, int32_t n, float* evals, float* out,
                          int32_t* status, int32_t* flags, const bed_config* cfg, float p,
                          float floor, void* workspace, size_t workspace_bytes, void* stream) {
  if (!cfg || !(p == p)) return BED_ERR_INVALID_ARGUMENT;
  bed_config cv = *cfg;
  cv.compute_vectors = 1;
  int rc = check_forward(A, batch, n, evals, out, &cv);
  if (rc) return rc;
  if (!aligned4(status) || !aligned4(flags) || (reinterpret_cast<uintptr_t>(workspace) & 255) != 0)
    return BED_ERR_MISALIGNED;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (flags) {
    cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(int32_t), s);
    if (e != cudaSuccess) return cuda_fail(e, "bed_forward_power_f32 memset(flags)");
  }
  if (batch == 0) return BED_SUCCESS;
  const int needs_positive = (p < 0.0f || p != floorf(p)) ? 1 : 0;  // solver.py:133
  const bed::KernelCfg k = kernel_cfg(&cv, n);
  if (n > kFusedPowerMaxN) {  // V to the workspace, then the tiled power kernel
    const size_t vbytes = align_up(sizeof(float) * (size_t)batch * n * n);
    if (!workspace || workspace_bytes < vbytes) return BED_ERR_INVALID_ARGUMENT;
    float* V = static_cast<float*>(workspace);
    rc = bed_forward_ws_f32(A, batch, n, evals, V, status, nullptr, flags, nullptr, nullptr, &cv,
                            static_cast<char*>(workspace) + vbytes, workspace_bytes - vbytes, stream);
    if (rc) return rc;
    bed::PowArgs pa{V, evals, out, status, flags, batch, n, p, floor, needs_positive, s};
    pa.merge = 1;  // the forward's statuses win; flags keep its bits
    cudaError_t e = bed::launch_power(pa);
    if (e != cudaSuccess) return cuda_fail(e, "bed_forward_power_f32 power launch");
    return BED_SUCCESS;
  }
  // fused: n <= 8 forms the power from V in the thread that solved the matrix,
  // 9 <= n <= 24 in the eigenvector fold's epilogue -- V never reaches memory
  if (n > 8 && (!workspace || bed::split_chunk(batch, n, true, k.max_steps, workspace_bytes) == 0))
    return BED_ERR_INVALID_ARGUMENT;
  const bed::PowSpec spec{p, floor, needs_positive};
  bed::FwdArgs a{A, batch, n, evals, out, status, nullptr, flags, k, s,
                 bed::DiagOut{nullptr, nullptr}, workspace, workspace_bytes, &spec};
  cudaError_t e = dispatch_forward(a);
  if (e != cudaSuccess) return cuda_fail(e, "bed_forward_power_f32 launch");
  return BED_SUCCESS;
}

int bed_backward_f32(const float* V, const float* evals, const float* gV, const float* gL,
                     float* gA, int64_t batch, int32_t n, int32_t taylor_degree, int32_t* status,
                     int32_t* flags, void* stream) {
  if (batch < 0 || n < 1 || n > 64 || taylor_degree < 0) return BED_ERR_INVALID_ARGUMENT;
  if (batch > 0 && (!V || !evals || !gA)) return BED_ERR_INVALID_ARGUMENT;
  if (!aligned4(V) || !aligned4(evals) || !aligned4(gV) || !aligned4(gL) || !aligned4(gA) ||
      !aligned4(status) || !aligned4(flags))
    return BED_ERR_MISALIGNED;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (flags) {
    cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(int32_t), s);
    if (e != cudaSuccess) return cuda_fail(e, "bed_backward_f32 memset(flags)");
  }
  if (batch == 0) return BED_SUCCESS;
  bed::BwdArgs a{V, evals, gV, gL, gA, batch, n, taylor_degree, status, flags, s};
  cudaError_t e = bed::launch_backward(a);
  if (e != cudaSuccess) return cuda_fail(e, "bed_backward_f32 launch");
  return BED_SUCCESS;
}

int bed_matrix_power_f32(const float* V, const float* evals, float* out, int32_t* status,
                         int32_t* flags, int64_t batch, int32_t n, float p, float floor,
                         void* stream) {
  if (batch < 0 || n < 1 || n > 64 || !(p == p)) return BED_ERR_INVALID_ARGUMENT;
  if (batch > 0 && (!V || !evals || !out)) return BED_ERR_INVALID_ARGUMENT;
  if (!aligned4(V) || !aligned4(evals) || !aligned4(out) || !aligned4(status) || !aligned4(flags))
    return BED_ERR_MISALIGNED;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (flags) {
    cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(int32_t), s);
    if (e != cudaSuccess) return cuda_fail(e, "bed_matrix_power_f32 memset(flags)");
  }
  if (batch == 0) return BED_SUCCESS;
  const int needs_positive = (p < 0.0f || p != floorf(p)) ? 1 : 0;  // solver.py:133
  bed::PowArgs a{V, evals, out, status, flags, batch, n, p, floor, needs_positive, s};
  cudaError_t e = bed::launch_power(a);
  if (e != cudaSuccess) return cuda_fail(e, "bed_matrix_power_f32 launch");
  return BED_SUCCESS;
}

int bed_scatter_f32(const float* X, int64_t batch, int32_t n, int32_t m, float eps, float* out,
                    void* stream) {
  if (batch < 0 || n < 1 || n > 64 || m < 1 || !(eps >= 0.0f)) return BED_ERR_INVALID_ARGUMENT;
  if (batch > 0 && (!X || !out)) return BED_ERR_INVALID_ARGUMENT;
  if (!aligned4(X) || !aligned4(out)) return BED_ERR_MISALIGNED;
  if (batch == 0) return BED_SUCCESS;
  bed::ScatArgs a{X, out, batch, n, m, eps, static_cast<cudaStream_t>(stream)};
  cudaError_t e = bed::launch_scatter(a);
  if (e != cudaSuccess) return cuda_fail(e, "bed_scatter_f32 launch");
  return BED_SUCCESS;
}

size_t bed_scatter_forward_workspace_bytes(int64_t batch, int32_t n, int32_t m,
                                           const bed_config* cfg, int32_t power) {
  if (!cfg || batch <= 0 || n <= 8 || n > 64 || m < 1) return 0;
  return align_up(sizeof(float) * (size_t)batch * n * n) +
         (power ? bed_forward_power_workspace_bytes(batch, n, cfg)
                : bed_forward_workspace_bytes(batch, n, cfg));
}

int bed_scatter_forward_f32(const float* X, int64_t batch, int32_t n, int32_t m, float eps,
                            float* evals, float* out, int32_t* status, int32_t* flags,
                            const bed_config* cfg, int32_t power, float p, float floor,
                            void* workspace, size_t workspace_bytes, void* stream) {
  if (m < 1 || !(eps >= 0.0f) || (power && !(p == p))) return BED_ERR_INVALID_ARGUMENT;
  if (!cfg) return BED_ERR_INVALID_ARGUMENT;
  bed_config cv = *cfg;
  if (power) cv.compute_vectors = 1;
  int rc = check_forward(X, batch, n, evals, out, &cv);
  if (rc) return rc;
  if (!aligned4(status) || !aligned4(flags) || (reinterpret_cast<uintptr_t>(workspace) & 255) != 0)
    return BED_ERR_MISALIGNED;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n > 8) {  // composed: the scatter kernel writes S to the workspace, the forward reads it
    const size_t sbytes = align_up(sizeof(float) * (size_t)batch * n * n);
    if (batch > 0 && (!workspace || workspace_bytes < sbytes)) return BED_ERR_INVALID_ARGUMENT;
    float* S = static_cast<float*>(workspace);
    if (batch > 0) {
      bed::ScatArgs sa{X, S, batch, n, m, eps, s};
      cudaError_t e = bed::launch_scatter(sa);
      if (e != cudaSuccess) return cuda_fail(e, "bed_scatter_forward_f32 scatter launch");
    }
    void* rest = batch > 0 ? static_cast<char*>(workspace) + sbytes : workspace;
    const size_t rest_bytes = batch > 0 ? workspace_bytes - sbytes : workspace_bytes;
    return power ? bed_forward_power_f32(S, batch, n, evals, out, status, flags, &cv, p, floor, rest,
                                         rest_bytes, stream)
                 : bed_forward_ws_f32(S, batch, n, evals, out, status, nullptr, flags, nullptr,
                                      nullptr, &cv, rest, rest_bytes, stream);
  }
  if (flags) {
    cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(int32_t), s);
    if (e != cudaSuccess) return cuda_fail(e, "bed_scatter_forward_f32 memset(flags)");
  }
  if (batch == 0) return BED_SUCCESS;
  // n <= 8: one kernel -- each thread forms its covariance from X in registers,
  // solves it, and writes evals and V (or the power); S never reaches memory
  const bed::ScatSpec sc{X, m, eps};
  const bed::PowSpec spec{p, floor, (p < 0.0f || p != floorf(p)) ? 1 : 0};
  bed::FwdArgs a{X, batch, n, evals, cv.compute_vectors ? out : nullptr, status, nullptr, flags,
                 kernel_cfg(&cv, n), s, bed::DiagOut{nullptr, nullptr}, nullptr, 0,
                 power ? &spec : nullptr, &sc};
  cudaError_t e = dispatch_forward(a);
  if (e != cudaSuccess) return cuda_fail(e, "bed_scatter_forward_f32 launch");
  return BED_SUCCESS;
}

// Host-buffer entry: the batch streams through the device in chunks.  Three
// role streams -- host-to-device copies, solves, device-to-host copies --
// and a ring of kSlots device buffer sets ordered by events, so the copy
// engines of both directions run back to back (PCIe is full duplex) while
// the solves fit in between.  Copies are only asynchronous when the host
// buffers are page-locked; pageable buffers still give correct, serialised
// results.
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
  const int64_t chunk = std::max<int64_t>(1024, std::min<int64_t>(batch, host_chunk_bytes() / per));
  constexpr int kSlots = 4;
  enum { H, C, D };
  cudaStream_t st[3] = {};
  cudaEvent_t ev[3][kSlots] = {};
  char* pool = nullptr;
  const size_t szA = align_up(sizeof(float) * chunk * nn), szL = align_up(sizeof(float) * chunk * n);
  const size_t szV = vecs ? align_up(sizeof(float) * chunk * nn) : 0, szI = align_up(sizeof(int32_t) * chunk);
  const size_t slot = szA + szL + szV + 2 * szI;
  int out = BED_SUCCESS;
  for (int r = 0; r < 3 && out == BED_SUCCESS; ++r) {
    if ((e = cudaStreamCreateWithFlags(&st[r], cudaStreamNonBlocking)) != cudaSuccess) out = cuda_fail(e, "stream");
    for (int b = 0; b < kSlots && out == BED_SUCCESS; ++b)
      if ((e = cudaEventCreateWithFlags(&ev[r][b], cudaEventDisableTiming)) != cudaSuccess) out = cuda_fail(e, "event");
  }
  const size_t wsb = bed_forward_workspace_bytes(chunk, n, cfg);
  if (out == BED_SUCCESS && (e = pool_alloc(reinterpret_cast<void**>(&pool), slot * kSlots + wsb, st[C])) != cudaSuccess)
    out = cuda_fail(e, "bed_forward_host_f32 allocation");
  if (out == BED_SUCCESS && (e = cudaEventRecord(ev[C][0], st[C])) == cudaSuccess) {
    // the H2D stream must not touch the pool before it is allocated
    e = cudaStreamWaitEvent(st[H], ev[C][0], 0);
  }
  if (out == BED_SUCCESS && e != cudaSuccess) out = cuda_fail(e, "event order");
  bool used[kSlots] = {};
  for (int64_t off = 0, it = 0; off < batch && out == BED_SUCCESS; off += chunk, ++it) {
    const int b = (int)(it % kSlots);
    const int64_t m = std::min<int64_t>(chunk, batch - off);
    char* base = pool + slot * b;
    float* dA = reinterpret_cast<float*>(base);
    float* dL = reinterpret_cast<float*>(base + szA);
    float* dV = vecs ? reinterpret_cast<float*>(base + szA + szL) : nullptr;
    int32_t* dS = reinterpret_cast<int32_t*>(base + szA + szL + szV);
    int32_t* dK = reinterpret_cast<int32_t*>(base + szA + szL + szV + szI);
    // H2D: slot b's input is free once the solve of chunk it - kSlots is done
    if (used[b] && (e = cudaStreamWaitEvent(st[H], ev[C][b], 0)) != cudaSuccess) { out = cuda_fail(e, "wait"); break; }
    if ((e = cudaMemcpyAsync(dA, A + off * nn, sizeof(float) * m * nn, cudaMemcpyHostToDevice, st[H])) != cudaSuccess ||
        (e = cudaEventRecord(ev[H][b], st[H])) != cudaSuccess) { out = cuda_fail(e, "H2D"); break; }
    // solve: after this chunk's input arrived and slot b's outputs were read back
    if ((e = cudaStreamWaitEvent(st[C], ev[H][b], 0)) != cudaSuccess ||
        (used[b] && (e = cudaStreamWaitEvent(st[C], ev[D][b], 0)) != cudaSuccess)) { out = cuda_fail(e, "wait"); break; }
    bed::FwdArgs a{dA, m, n, dL, dV, dS, dK, nullptr, kernel_cfg(cfg, n), st[C], bed::DiagOut{nullptr, nullptr},
                   wsb ? pool + slot * kSlots : nullptr, wsb};
    if ((e = dispatch_forward(a)) != cudaSuccess) { out = cuda_fail(e, "bed_forward_host_f32 launch"); break; }
    if ((e = cudaEventRecord(ev[C][b], st[C])) != cudaSuccess) { out = cuda_fail(e, "record"); break; }
    // D2H
    if ((e = cudaStreamWaitEvent(st[D], ev[C][b], 0)) != cudaSuccess ||
        (vecs && (e = cudaMemcpyAsync(evecs + off * nn, dV, sizeof(float) * m * nn, cudaMemcpyDeviceToHost, st[D])) != cudaSuccess) ||
        (e = cudaMemcpyAsync(evals + off * n, dL, sizeof(float) * m * n, cudaMemcpyDeviceToHost, st[D])) != cudaSuccess ||
        (status && (e = cudaMemcpyAsync(status + off, dS, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, st[D])) != cudaSuccess) ||
        (steps && (e = cudaMemcpyAsync(steps + off, dK, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, st[D])) != cudaSuccess) ||
        (e = cudaEventRecord(ev[D][b], st[D])) != cudaSuccess) { out = cuda_fail(e, "D2H"); break; }
    used[b] = true;
  }
  for (int r = 0; r < 3; ++r) {
    if (!st[r]) continue;
    e = cudaStreamSynchronize(st[r]);
    if (e != cudaSuccess && out == BED_SUCCESS) out = cuda_fail(e, "bed_forward_host_f32 sync");
  }
  if (pool) cudaFreeAsync(pool, st[C]);
  if (st[C]) cudaStreamSynchronize(st[C]);
  for (int r = 0; r < 3; ++r) {
    for (int b = 0; b < kSlots; ++b)
      if (ev[r][b]) cudaEventDestroy(ev[r][b]);
    if (st[r]) cudaStreamDestroy(st[r]);
  }
  cudaSetDevice(prev);
  return out;
}

// ---------------------------------------------------------------------------
// Float64 host-buffer entry -- the call a reference user makes
// (batched_eig(BatchedSymmetric(float64 numpy)), solver.py:79-112).  The
// reference validates in float64 (core.py:286-309); here host threads do the
// same per matrix -- finiteness, max|a - a^T| <= symmetry_tol * max(1, ||A||_F),
// (A + A^T) / 2 -- and write the FP32 cast straight into a page-locked staging
// slot, so the validation, the casts and the PCIe copies all overlap.  Chunks
// cycle through kSlots slots, each with its own stream (H2D, solve, D2H in
// order); while the GPU works on chunks it-3..it-1 the host threads convert
// chunk it in and chunk it-kSlots out (FP32 -> float64 into the caller's
// arrays).  A matrix the host rejects is solved as the zero matrix (what the
// device kernels do with an invalid input) and keeps the host status.
namespace {

struct HostStage {
  std::mutex mu;  // one f64 host call per device at a time owns the staging memory
  char* buf = nullptr;
  size_t bytes = 0;
};

HostStage g_stage[64];

// Ask for transparent huge pages on a caller's freshly allocated result array:
// its first touch happens in the output conversion, and with 4 KB pages the
// page faults (one per 4 KB of float64 results) cost more than the conversion.
// Advisory only; errors are ignored.
void advise_huge(void* p, size_t bytes) {
  constexpr uintptr_t kHuge = uintptr_t(2) << 20;
  const uintptr_t b = (reinterpret_cast<uintptr_t>(p) + kHuge - 1) & ~(kHuge - 1);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes) & ~(kHuge - 1);
  if (p && e > b) madvise(reinterpret_cast<void*>(b), e - b, MADV_HUGEPAGE);
}

int host_threads(int32_t req) {
  if (req > 0) return std::min(req, 256);
  const unsigned hw = std::thread::hardware_concurrency();
  return (int)std::max(1u, std::min(hw, 64u));
}

// reference validate (core.py:286-309) for one matrix; returns the status and
// writes the symmetrised FP32 cast (zeros when rejected)
inline int32_t validate_cast(const double* a, int n, double sym_tol, float* o) {
  const int nn = n * n;
  bool finite = true;
  double fro2 = 0.0, asym = 0.0;
  for (int k = 0; k < nn; ++k) {
    finite = finite && std::isfinite(a[k]);
    fro2 += a[k] * a[k];
  }
  if (!finite) {
    memset(o, 0, sizeof(float) * nn);
    return BED_STATUS_NON_FINITE;
  }
  for (int r = 0; r < n; ++r)
    for (int c = 0; c < r; ++c) asym = std::max(asym, std::fabs(a[r * n + c] - a[c * n + r]));
  if (asym > sym_tol * std::max(1.0, std::sqrt(fro2))) {
    memset(o, 0, sizeof(float) * nn);
    return BED_STATUS_NON_SYMMETRIC;
  }
  for (int r = 0; r < n; ++r) {
    o[r * n + r] = (float)a[r * n + r];
    for (int c = 0; c < r; ++c) {
      const float v = (float)((a[r * n + c] + a[c * n + r]) / 2.0);
      o[r * n + c] = v;
      o[c * n + r] = v;
    }
  }
  return BED_STATUS_OK;
}

}  // namespace

int bed_forward_host_f64(const double* A, int64_t batch, int32_t n, double* evals, double* evecs,
                         int32_t* status, int32_t* steps, int32_t* diag, float* resid,
                         const bed_config* cfg, int32_t device, int32_t threads) {
  if (!cfg || batch < 0 || n < 1 || n > 64) return BED_ERR_INVALID_ARGUMENT;
  if (batch > 0 && (!A || !evals || (cfg->compute_vectors && !evecs))) return BED_ERR_INVALID_ARGUMENT;
  {
    // the FP32 checks of the shared validator (pointer alignment of the f64
    // buffers is 8 bytes, which implies the 4 the validator asks for)
    int rc = check_forward(reinterpret_cast<const float*>(A), batch, n,
                           reinterpret_cast<const float*>(evals), reinterpret_cast<const float*>(evecs), cfg);
    if (rc) return rc;
  }
  if ((reinterpret_cast<uintptr_t>(A) & 7) || (reinterpret_cast<uintptr_t>(evals) & 7) ||
      (reinterpret_cast<uintptr_t>(evecs) & 7) || !aligned4(status) || !aligned4(steps) ||
      !aligned4(diag) || !aligned4(resid))
    return BED_ERR_MISALIGNED;
  if (batch == 0) return BED_SUCCESS;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return BED_ERR_NO_DEVICE;
  if (device < 0 || device >= ndev || device >= 64) return BED_ERR_INVALID_ARGUMENT;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  const int nthr = host_threads(threads);
  advise_huge(evals, sizeof(double) * (size_t)batch * n);
  if (cfg->compute_vectors) advise_huge(evecs, sizeof(double) * (size_t)batch * n * n);

  const bool vecs = cfg->compute_vectors != 0;
  const int64_t nn = (int64_t)n * n;
  // page-locked bytes per matrix: FP32 input, evals, V, status, steps, diag (3), resid, host status
  const int64_t per = 4 * (nn + n + (vecs ? nn : 0) + 7);
  const int64_t chunk = std::max<int64_t>(1024, std::min<int64_t>(batch, host_chunk_bytes() / per));
  constexpr int kSlots = 4;
  const size_t szA = align_up(sizeof(float) * chunk * nn), szL = align_up(sizeof(float) * chunk * n);
  const size_t szV = vecs ? align_up(sizeof(float) * chunk * nn) : 0, szI = align_up(sizeof(int32_t) * chunk);
  const size_t slot = szA + szL + szV + 6 * szI;  // status, steps, diag x3, resid
  const size_t hslot = slot + szI;                 // + the host status
  const size_t wsb = bed_forward_workspace_bytes(chunk, n, cfg);

  HostStage& hs = g_stage[device];
  std::lock_guard<std::mutex> lock(hs.mu);
  int out = BED_SUCCESS;
  if (hs.bytes < hslot * kSlots) {
    if (hs.buf) cudaFreeHost(hs.buf);
    hs.buf = nullptr;
    hs.bytes = 0;
    if ((e = cudaHostAlloc(reinterpret_cast<void**>(&hs.buf), hslot * kSlots, cudaHostAllocPortable)) != cudaSuccess) {
      hs.buf = nullptr;
      cudaSetDevice(prev);
      return cuda_fail(e, "bed_forward_host_f64 staging");
    }
    hs.bytes = hslot * kSlots;
  }
  cudaStream_t st[kSlots] = {};
  cudaEvent_t done[kSlots] = {}, ready = nullptr;
  char* pool = nullptr;
  for (int b = 0; b < kSlots && out == BED_SUCCESS; ++b)
    if ((e = cudaStreamCreateWithFlags(&st[b], cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming)) != cudaSuccess)
      out = cuda_fail(e, "stream/event");
  if (out == BED_SUCCESS && (e = cudaEventCreateWithFlags(&ready, cudaEventDisableTiming)) != cudaSuccess)
    out = cuda_fail(e, "event");
  if (out == BED_SUCCESS && (e = pool_alloc(reinterpret_cast<void**>(&pool), (slot + wsb) * kSlots, st[0])) != cudaSuccess)
    out = cuda_fail(e, "bed_forward_host_f64 allocation");
  if (out == BED_SUCCESS && (e = cudaEventRecord(ready, st[0])) != cudaSuccess) out = cuda_fail(e, "record");
  for (int b = 1; b < kSlots && out == BED_SUCCESS; ++b)
    if ((e = cudaStreamWaitEvent(st[b], ready, 0)) != cudaSuccess) out = cuda_fail(e, "wait");

  const int64_t nchunks = (batch + chunk - 1) / chunk;
  const double sym_tol = cfg->symmetry_tol;
  auto hbase = [&](int b) { return hs.buf + hslot * b; };
  // results of chunk c (in slot c % kSlots) into the caller's float64 arrays
  auto drain = [&](int64_t c) {
    const int b = (int)(c % kSlots);
    const int64_t off = c * chunk, m = std::min<int64_t>(chunk, batch - off);
    char* h = hbase(b);
    const float* hL = reinterpret_cast<const float*>(h + szA);
    const float* hV = reinterpret_cast<const float*>(h + szA + szL);
    const int32_t* hS = reinterpret_cast<const int32_t*>(h + szA + szL + szV);
    const int32_t* hK = hS + szI / 4;
    const int32_t* hD = hK + szI / 4;  // diag, 3 per matrix (3 szI blocks)
    const float* hR = reinterpret_cast<const float*>(hD + 3 * (szI / 4));
    const int32_t* hH = reinterpret_cast<const int32_t*>(hR + szI / 4);
#pragma omp parallel for num_threads(nthr) schedule(static)
    for (int64_t i = 0; i < m; ++i) {
      for (int k = 0; k < n; ++k) evals[(off + i) * n + k] = (double)hL[i * n + k];
      if (vecs)
        for (int64_t k = 0; k < nn; ++k) evecs[(off + i) * nn + k] = (double)hV[i * nn + k];
      if (status) status[off + i] = hH[i] != BED_STATUS_OK ? hH[i] : hS[i];
      if (steps) steps[off + i] = hK[i];
      if (diag)
        for (int k = 0; k < 3; ++k) diag[(off + i) * 3 + k] = hD[i * 3 + k];
      if (resid) resid[off + i] = hR[i];
    }
  };
  for (int64_t it = 0; it < nchunks + kSlots && out == BED_SUCCESS; ++it) {
    const int b = (int)(it % kSlots);
    if (it >= kSlots) {  // slot b's previous chunk: wait for its read-back, convert it out
      if ((e = cudaEventSynchronize(done[b])) != cudaSuccess) { out = cuda_fail(e, "bed_forward_host_f64 sync"); break; }
      drain(it - kSlots);
    }
    if (it >= nchunks) continue;
    const int64_t off = it * chunk, m = std::min<int64_t>(chunk, batch - off);
    char* h = hbase(b);
    float* hA = reinterpret_cast<float*>(h);
    int32_t* hH = reinterpret_cast<int32_t*>(h + slot);
#pragma omp parallel for num_threads(nthr) schedule(static)
    for (int64_t i = 0; i < m; ++i) hH[i] = validate_cast(A + (off + i) * nn, n, sym_tol, hA + i * nn);
    char* d = pool + (slot + wsb) * b;
    float* dA = reinterpret_cast<float*>(d);
    float* dL = reinterpret_cast<float*>(d + szA);
    float* dV = vecs ? reinterpret_cast<float*>(d + szA + szL) : nullptr;
    int32_t* dS = reinterpret_cast<int32_t*>(d + szA + szL + szV);
    int32_t* dK = dS + szI / 4;
    int32_t* dD = dK + szI / 4;
    float* dR = reinterpret_cast<float*>(dD + 3 * (szI / 4));
    // D2H of the contiguous output block [evals .. resid] in one copy
    const size_t outb = szL + szV + 6 * szI;
    bed::FwdArgs a{dA, m, n, dL, dV, dS, dK, nullptr, kernel_cfg(cfg, n), st[b], bed::DiagOut{dD, dR},
                   wsb ? d + slot : nullptr, wsb};
    if ((e = cudaMemcpyAsync(dA, hA, sizeof(float) * m * nn, cudaMemcpyHostToDevice, st[b])) != cudaSuccess ||
        (e = dispatch_forward(a)) != cudaSuccess ||
        (e = cudaMemcpyAsync(h + szA, d + szA, outb, cudaMemcpyDeviceToHost, st[b])) != cudaSuccess ||
        (e = cudaEventRecord(done[b], st[b])) != cudaSuccess) {
      out = cuda_fail(e, "bed_forward_host_f64 chunk");
      break;
    }
  }
  for (int b = 0; b < kSlots; ++b)
    if (st[b]) {
      e = cudaStreamSynchronize(st[b]);
      if (e != cudaSuccess && out == BED_SUCCESS) out = cuda_fail(e, "bed_forward_host_f64 sync");
    }
  if (pool) cudaFreeAsync(pool, st[0]);
  if (st[0]) cudaStreamSynchronize(st[0]);
  for (int b = 0; b < kSlots; ++b) {
    if (done[b]) cudaEventDestroy(done[b]);
    if (st[b]) cudaStreamDestroy(st[b]);
  }
  if (ready) cudaEventDestroy(ready);
  cudaSetDevice(prev);
  return out;
}

}  // extern "C"
