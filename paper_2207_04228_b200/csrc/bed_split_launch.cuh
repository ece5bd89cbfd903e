// bed_split_launch.cuh -- host side of the medium path: workspace layout,
// chunking and launches (one stream; the workspace is the caller's).
#pragma once

#include <algorithm>

#include "bed_launch.h"
#include "bed_split_plan.h"
#include "bed_fold_tma.cuh"
#include "bed_split.cuh"

namespace bed {

template <int NMAX, bool EXACT>
cudaError_t run_split(const FwdArgs& a) {
  const bool vecs = a.evecs != nullptr;
  const int n = a.n;
  const int64_t nn = (int64_t)n * n;
  const int64_t Bc = split_chunk(a.batch, n, vecs, a.cfg.max_steps, a.ws_bytes);
  if (Bc == 0 || a.ws == nullptr) return cudaErrorInvalidValue;
  const SplitPlan pl = split_plan(Bc, n, vecs, a.cfg.max_steps);
  char* base = static_cast<char*>(a.ws);
  SplitWs ws;
  ws.P = vecs ? reinterpret_cast<float*>(base + pl.oP) : nullptr;
  ws.D = reinterpret_cast<float*>(base + pl.oD);
  ws.E = reinterpret_cast<float*>(base + pl.oE);
  ws.lam = vecs ? reinterpret_cast<float*>(base + pl.oL) : nullptr;
  ws.vstat = reinterpret_cast<int32_t*>(base + pl.oV);
  ws.rot = vecs ? reinterpret_cast<float2*>(base + pl.oR) : nullptr;
  ws.msw = vecs ? reinterpret_cast<int32_t*>(base + pl.oM) : nullptr;
  ws.nsw = vecs ? reinterpret_cast<int32_t*>(base + pl.oN) : nullptr;
  ws.mlane = vecs ? reinterpret_cast<uint8_t*>(base + pl.oML) : nullptr;
  ws.Bc = Bc;
  ws.Smax = 2 * a.cfg.max_steps + 1;
  cudaError_t e = cudaSuccess;

  using HP = HHParams<NMAX>;
  auto hk = vecs ? bed_hh_kernel<NMAX, EXACT, true> : bed_hh_kernel<NMAX, EXACT, false>;
  e = ensure_smem(hk, HP::BYTES);
  if (e == cudaSuccess && vecs) e = ensure_smem(bed_fold_tma_kernel<NMAX, EXACT>, FTParams<NMAX>::BYTES);
  for (int64_t c0 = 0; c0 < a.batch && e == cudaSuccess; c0 += Bc) {
    const int64_t bc = std::min<int64_t>(Bc, a.batch - c0);
    hk<<<(unsigned)((bc + HP::G - 1) / HP::G), HP::THREADS, HP::BYTES, a.stream>>>(
        a.A + c0 * nn, bc, n, ws, a.cfg);
    if (vecs) {
      using FP = FTParams<NMAX>;
      bed_qr_kernel<NMAX, EXACT, true><<<(unsigned)((bc + kQThreads - 1) / kQThreads), kQThreads, 0,
                                         a.stream>>>(bc, c0, n, ws, a.evals, a.status, a.steps,
                                                     a.flags, a.cfg, a.dg);
      bed_fold_tma_kernel<NMAX, EXACT><<<(unsigned)((bc + FP::MPC - 1) / FP::MPC), FP::THREADS, FP::BYTES,
                                         a.stream>>>(bc, c0, n, ws, a.evals, a.evecs, a.cfg);
    } else {
      bed_qr_kernel<NMAX, EXACT, false><<<(unsigned)((bc + kQThreads - 1) / kQThreads), kQThreads, 0,
                                          a.stream>>>(bc, c0, n, ws, a.evals, a.status, a.steps,
                                                      a.flags, a.cfg, a.dg);
    }
    e = cudaGetLastError();
  }
  return e;
}

}  // namespace bed
