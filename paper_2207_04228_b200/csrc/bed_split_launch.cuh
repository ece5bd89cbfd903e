// bed_split_launch.cuh -- host side of the three-kernel path: workspace
// sizing, chunking and launches (one stream, stream-ordered allocation).
#pragma once

#include <algorithm>

#include "bed_launch.h"
#include "bed_split.cuh"

namespace bed {

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// Workspace budget per call; chunks of the batch are solved in sequence.
constexpr size_t kSplitWorkspaceBytes = size_t(4) << 30;

template <typename K>
inline cudaError_t set_smem(K kern, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <int NMAX, bool EXACT>
cudaError_t run_split(const FwdArgs& a) {
  const bool vecs = a.evecs != nullptr;
  const int n = a.n;
  const int64_t nn = (int64_t)n * n;
  const int smax = 2 * a.cfg.max_steps + 1;
  const size_t per = 4 * (2 * (size_t)n) + 4 +
                     (vecs ? 4 * (size_t)nn + 4 * (size_t)n + (size_t)smax * (NMAX - 1) * 8 : 0);
  const size_t per_warp = vecs ? (size_t)smax * (4 + 32) + 4 : 0;
  const int64_t want = (a.batch + 31) / 32 * 32;
  const size_t need = (size_t)want * (per + per_warp / 32 + 1);
  // No per-call cudaMemGetInfo (it can take milliseconds and stalls the
  // stream's feed): try the full budget and shrink only if the pool refuses.
  size_t budget = kSplitWorkspaceBytes;
  int64_t Bc = 0, W = 0;
  size_t off = 0, oP = 0, oD = 0, oE = 0, oL = 0, oV = 0, oR = 0, oM = 0, oN = 0, oML = 0;
  auto plan = [&] {
    const int64_t cap = (int64_t)(budget / (per + per_warp / 32 + 1));
    Bc = std::max<int64_t>(32, std::min<int64_t>(cap, want) / 32 * 32);
    W = Bc / 32;
    off = 0;
    auto take = [&](size_t bytes) {
      size_t o = off;
      off += align256(bytes);
      return o;
    };
    oP = vecs ? take(4 * (size_t)Bc * nn) : 0;
    oD = take(4 * (size_t)Bc * n);
    oE = take(4 * (size_t)Bc * n);
    oL = vecs ? take(4 * (size_t)Bc * n) : 0;
    oV = take(4 * (size_t)Bc);
    oR = vecs ? take((size_t)W * smax * (NMAX - 1) * 32 * 8) : 0;
    oM = vecs ? take((size_t)W * smax * 4) : 0;
    oN = vecs ? take((size_t)W * 4) : 0;
    oML = vecs ? take((size_t)W * smax * 32) : 0;
  };
  plan();
  (void)need;
  char* base = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&base), off, a.stream);
  while (e == cudaErrorMemoryAllocation && Bc > 32) {
    cudaGetLastError();  // clear the allocation error
    size_t free_b = 0, total_b = 0;
    budget = (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) ? std::min(budget / 2, free_b / 2)
                                                                 : budget / 2;
    plan();
    e = cudaMallocAsync(reinterpret_cast<void**>(&base), off, a.stream);
  }
  if (e != cudaSuccess) return e;
  SplitWs ws;
  ws.P = vecs ? reinterpret_cast<float*>(base + oP) : nullptr;
  ws.D = reinterpret_cast<float*>(base + oD);
  ws.E = reinterpret_cast<float*>(base + oE);
  ws.lam = vecs ? reinterpret_cast<float*>(base + oL) : nullptr;
  ws.vstat = reinterpret_cast<int32_t*>(base + oV);
  ws.rot = vecs ? reinterpret_cast<float2*>(base + oR) : nullptr;
  ws.msw = vecs ? reinterpret_cast<int32_t*>(base + oM) : nullptr;
  ws.nsw = vecs ? reinterpret_cast<int32_t*>(base + oN) : nullptr;
  ws.mlane = vecs ? reinterpret_cast<uint8_t*>(base + oML) : nullptr;
  ws.Bc = Bc;
  ws.Smax = smax;

  using HP = HHParams<NMAX>;
  using FP = FoldParams<NMAX>;
  auto hk = vecs ? bed_hh_kernel<NMAX, EXACT, true> : bed_hh_kernel<NMAX, EXACT, false>;
  auto qk = vecs ? bed_qr_kernel<NMAX, EXACT, true> : bed_qr_kernel<NMAX, EXACT, false>;
  auto fk = bed_fold_kernel<NMAX, EXACT>;
  static bool attrs_set = false;  // idempotent; a benign race at worst repeats it
  if (!attrs_set) {
    if ((e = set_smem(bed_hh_kernel<NMAX, EXACT, true>, HP::BYTES)) != cudaSuccess ||
        (e = set_smem(bed_hh_kernel<NMAX, EXACT, false>, HP::BYTES)) != cudaSuccess ||
        (e = set_smem(fk, FP::BYTES)) != cudaSuccess) {
      cudaFreeAsync(base, a.stream);
      return e;
    }
    attrs_set = true;
  }

  for (int64_t c0 = 0; c0 < a.batch && e == cudaSuccess; c0 += Bc) {
    const int64_t bc = std::min<int64_t>(Bc, a.batch - c0);
    hk<<<(unsigned)((bc + HP::G - 1) / HP::G), HP::THREADS, HP::BYTES, a.stream>>>(
        a.A + c0 * nn, bc, n, ws, a.cfg);
    qk<<<(unsigned)((bc + kQThreads - 1) / kQThreads), kQThreads, 0, a.stream>>>(
        bc, c0, n, ws, a.evals, a.status, a.steps, a.flags, a.cfg);
    if (vecs)
      fk<<<(unsigned)((bc + FP::G - 1) / FP::G), FP::THREADS, FP::BYTES, a.stream>>>(
          bc, c0, n, ws, a.evals, a.evecs, a.cfg);
    e = cudaGetLastError();
  }
  cudaError_t ef = cudaFreeAsync(base, a.stream);
  return e != cudaSuccess ? e : ef;
}

}  // namespace bed
