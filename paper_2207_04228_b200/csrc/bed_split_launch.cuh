// bed_split_launch.cuh -- host side of the medium path: workspace layout,
// chunking and launches (one stream; the workspace is the caller's).
#pragma once

#include <algorithm>

#include "bed_launch.h"
#include "bed_split_plan.h"
#include "bed_fold_tma.cuh"
#include "bed_split.cuh"

namespace bed {

inline SplitWs split_ws(char* base, const SplitPlan& pl, bool vecs, int max_steps) {
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
  ws.Bc = pl.Bc;
  ws.Smax = 2 * max_steps + 1;
  return ws;
}

// H for matrices [c0, c0 + bc) on stream st.
template <int NMAX, bool EXACT>
cudaError_t launch_h(const FwdArgs& a, const SplitWs& ws, int64_t c0, int64_t bc, cudaStream_t st) {
  const bool vecs = a.evecs != nullptr;
  using HP = HHParams<NMAX>;
  auto hk = vecs ? bed_hh_kernel<NMAX, EXACT, true> : bed_hh_kernel<NMAX, EXACT, false>;
  hk<<<(unsigned)((bc + HP::G - 1) / HP::G), HP::THREADS, HP::BYTES, st>>>(a.A + c0 * a.n * a.n, bc,
                                                                            a.n, ws, a.cfg);
  return cudaGetLastError();
}

// Q (+ F with vectors) for matrices [c0, c0 + bc) on stream st.
template <int NMAX, bool EXACT>
cudaError_t launch_qf(const FwdArgs& a, const SplitWs& ws, int64_t c0, int64_t bc, cudaStream_t st) {
  const int n = a.n;
  if (a.evecs != nullptr) {
    using FP = FTParams<NMAX, EXACT>;
    bed_qr_kernel<NMAX, EXACT, true><<<(unsigned)((bc + kQThreads - 1) / kQThreads), kQThreads, 0, st>>>(
        bc, c0, n, ws, a.evals, a.status, a.steps, a.flags, a.cfg, a.dg);
    if (a.pw)  // spectral power in the fold's epilogue (V never reaches memory)
      bed_fold_tma_kernel<NMAX, EXACT, true><<<(unsigned)((bc + FP::MPC - 1) / FP::MPC), FP::THREADS,
                                               FP::BYTES, st>>>(bc, c0, n, ws, a.evals, a.evecs, a.cfg,
                                                                *a.pw, a.status, a.flags);
    else
      bed_fold_tma_kernel<NMAX, EXACT><<<(unsigned)((bc + FP::MPC - 1) / FP::MPC), FP::THREADS, FP::BYTES,
                                         st>>>(bc, c0, n, ws, a.evals, a.evecs, a.cfg);
  } else {
    bed_qr_kernel<NMAX, EXACT, false><<<(unsigned)((bc + kQThreads - 1) / kQThreads), kQThreads, 0, st>>>(
        bc, c0, n, ws, a.evals, a.status, a.steps, a.flags, a.cfg, a.dg);
  }
  return cudaGetLastError();
}

template <int NMAX, bool EXACT>
cudaError_t run_split(const FwdArgs& a) {
  const bool vecs = a.evecs != nullptr;
  const int n = a.n;
  if (a.ws == nullptr) return cudaErrorInvalidValue;
  using HP = HHParams<NMAX>;
  cudaError_t e = ensure_smem(vecs ? bed_hh_kernel<NMAX, EXACT, true> : bed_hh_kernel<NMAX, EXACT, false>,
                              HP::BYTES);
  if (e == cudaSuccess && vecs) e = ensure_smem(bed_fold_tma_kernel<NMAX, EXACT>, FTParams<NMAX, EXACT>::BYTES);
  if (e == cudaSuccess && a.pw) e = ensure_smem(bed_fold_tma_kernel<NMAX, EXACT, true>, FTParams<NMAX, EXACT>::BYTES);
  if (e != cudaSuccess) return e;
  char* base = static_cast<char*>(a.ws);

  const int64_t Bc = split_chunk(a.batch, n, vecs, a.cfg.max_steps, a.ws_bytes);
  if (Bc == 0) return cudaErrorInvalidValue;
  const SplitWs ws = split_ws(base, split_plan(Bc, n, vecs, a.cfg.max_steps), vecs, a.cfg.max_steps);
  for (int64_t c0 = 0; c0 < a.batch && e == cudaSuccess; c0 += Bc) {
    const int64_t bc = std::min<int64_t>(Bc, a.batch - c0);
    e = launch_h<NMAX, EXACT>(a, ws, c0, bc, a.stream);
    if (e == cudaSuccess) e = launch_qf<NMAX, EXACT>(a, ws, c0, bc, a.stream);
  }
  return e;
}

}  // namespace bed
