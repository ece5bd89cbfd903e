// bed_split_launch.cuh -- host side of the medium path: workspace layout,
// chunking and launches (one stream; the workspace is the caller's).
#pragma once

#include <algorithm>

#include "bed_launch.h"
#include "bed_split_plan.h"
#include "bed_qf.cuh"
#include "bed_split.cuh"

namespace bed {

template <int NMAX, bool EXACT>
cudaError_t run_split(const FwdArgs& a) {
  const bool vecs = a.evecs != nullptr;
  constexpr bool kFused = NMAX <= 24;
  static_assert(!kFused || NMAX == 16 || NMAX == 24, "fused tiers");
  const int n = a.n;
  const int64_t nn = (int64_t)n * n;
  const int64_t Bc = split_chunk(a.batch, n, vecs, a.cfg.max_steps, a.ws_bytes);
  if (Bc == 0 || a.ws == nullptr) return cudaErrorInvalidValue;
  const SplitPlan pl = split_plan(Bc, n, vecs, a.cfg.max_steps);
  const bool rec = vecs && !kFused;
  char* base = static_cast<char*>(a.ws);
  SplitWs ws;
  ws.P = vecs ? reinterpret_cast<float*>(base + pl.oP) : nullptr;
  ws.D = reinterpret_cast<float*>(base + pl.oD);
  ws.E = reinterpret_cast<float*>(base + pl.oE);
  ws.lam = rec ? reinterpret_cast<float*>(base + pl.oL) : nullptr;
  ws.vstat = reinterpret_cast<int32_t*>(base + pl.oV);
  ws.rot = rec ? reinterpret_cast<float2*>(base + pl.oR) : nullptr;
  ws.msw = rec ? reinterpret_cast<int32_t*>(base + pl.oM) : nullptr;
  ws.nsw = rec ? reinterpret_cast<int32_t*>(base + pl.oN) : nullptr;
  ws.mlane = rec ? reinterpret_cast<uint8_t*>(base + pl.oML) : nullptr;
  ws.Bc = Bc;
  ws.Smax = 2 * a.cfg.max_steps + 1;
  cudaError_t e = cudaSuccess;

  using HP = HHParams<NMAX>;
  auto hk = vecs ? bed_hh_kernel<NMAX, EXACT, true> : bed_hh_kernel<NMAX, EXACT, false>;
  e = ensure_smem(hk, HP::BYTES);
  if constexpr (kFused) {
    using QP = QFParams<NMAX>;
    auto qfk = bed_qf_kernel<NMAX, EXACT>;
    if (e == cudaSuccess) e = ensure_smem(qfk, QP::BYTES);
    for (int64_t c0 = 0; c0 < a.batch && e == cudaSuccess; c0 += Bc) {
      const int64_t bc = std::min<int64_t>(Bc, a.batch - c0);
      hk<<<(unsigned)((bc + HP::G - 1) / HP::G), HP::THREADS, HP::BYTES, a.stream>>>(
          a.A + c0 * nn, bc, n, ws, a.cfg);
      if (vecs)
        qfk<<<(unsigned)((bc + QP::MPC - 1) / QP::MPC), QP::THREADS, QP::BYTES, a.stream>>>(
            bc, c0, n, ws, a.evals, a.evecs, a.status, a.steps, a.flags, a.cfg);
      else
        bed_qr_kernel<NMAX, EXACT, false><<<(unsigned)((bc + kQThreads - 1) / kQThreads), kQThreads, 0,
                                            a.stream>>>(bc, c0, n, ws, a.evals, a.status, a.steps,
                                                        a.flags, a.cfg);
      e = cudaGetLastError();
    }
  } else {
    using FP = FoldParams<NMAX>;
    auto qk = vecs ? bed_qr_kernel<NMAX, EXACT, true> : bed_qr_kernel<NMAX, EXACT, false>;
    auto fk = bed_fold_kernel<NMAX, EXACT>;
    if (e == cudaSuccess) e = ensure_smem(fk, FP::BYTES);
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
  }
  return e;
}

}  // namespace bed
