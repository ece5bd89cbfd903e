// bed_split.cuh -- forward ED for 9 <= n <= 64 as three kernels per chunk.
//
// The band QR iteration is a long chain of dependent scalar rotations
// (~1.2 n^2 per matrix, each ~50 cycles of latency), while the eigenvector
// fold is wide, cheap arithmetic on n x n registers.  Running both in one
// kernel ties the number of matrices whose chains can overlap to how many
// V's fit in the register file.  So the work is split:
//
//   H (bed_hh_kernel)    lane group per matrix (lane r owns row r):
//                        validate + symmetrise (core.py:286-309), Householder
//                        reduction (_kernels.py:36-92) with reflectors as
//                        shared-memory broadcasts, P = H_0 H_1 ... formed row
//                        by row (householder.py:216-231).  Writes P (the
//                        initial V) and the band (position-major) to the
//                        workspace.
//   Q (bed_qr_kernel)    one THREAD per matrix, the band in registers:
//                        equilibration (qr.py:522-534), double-shift sweeps
//                        (_sweep_block, _kernels.py:221-300) with per-matrix
//                        deflation (qr_loop_kernel :321-398 with the gate of
//                        :381-388), 2x2 closeout (:401-417).  Thousands of
//                        independent chains per SM hide the latency.  Every
//                        rotation (c, s) is streamed to the workspace as
//                        [warp][sweep][position][lane] -- one coalesced
//                        256-byte store per warp and position.
//   F (bed_fold_tma_kernel, bed_fold_tma.cuh)  V := P in registers, the
//                        recorded rotations streamed in by bulk async copies
//                        and applied to V's rows (two column updates,
//                        _kernels.py:269-277), then stable sort + sign
//                        (solver.py:60-76) and coalesced stores.
//
// Values-only solves (solver.py:94-109) run H (band only) and Q, which sorts
// the eigenvalues itself.
#pragma once

#include "bed_f32x2.cuh"
#include "bed_hh.cuh"
#include "bed_split_ws.cuh"
#include "bed_tile.cuh"

namespace bed {

// ---------------------------------------------------------------------------
// Q: one thread per matrix, band in registers, warp-synchronous sweeps.

// Fused sweep of the leading m-block (_sweep_block), predicated straight-line
// code over the positions (rotations past a lane's block are exact
// identities; m = 0 is a no-op).  The warp runs positions in blocks of
// kSweepBlk, skipping the blocks no lane needs: mw is the warp's largest
// active size (warp-uniform), so the branch is uniform and each block is one
// basic block in which the compiler overlaps the retire of position i with
// the rotation of position i + 1 (a per-position vote would end a basic
// block at every position and serialise the whole chain).  Positions past
// mw - 1 inside the last block are identities for every lane.  With VECS
// every rotation is stored to rec[p * RSTRIDE].
constexpr int kSweepBlk = 4;

template <int NMAX, bool VECS, int RSTRIDE = 32>
__device__ __forceinline__ void qr_sweep(float (&d)[NMAX], float (&e)[NMAX], int m, float mu,
                                         float2* __restrict__ rec, int mw) {
  float dw = d[0] - mu, g = e[0];
  float c1 = 1.0f, s1 = 0.0f, c2 = 1.0f, r1 = 0.0f, u1 = 0.0f;
  static_for<0, (NMAX + kSweepBlk - 1) / kSweepBlk>([&](auto bc) {
    constexpr int b0 = decltype(bc)::value * kSweepBlk;
    constexpr int b1 = b0 + kSweepBlk < NMAX ? b0 + kSweepBlk : NMAX;
    if (b0 == 0 || b0 <= mw - 1) {
#pragma unroll
      for (int i = b0; i < b1; ++i) {
        const bool act = i < m - 1;
        const float ei = (i < NMAX - 1 && act) ? e[i] : 0.0f;
        float c, s, r;
        givens(dw, ei, c, s, r);
        if (VECS && i < NMAX - 1) rec[i * RSTRIDE] = make_float2(c, s);
        const float dn = (i + 1 < NMAX ? d[i + 1] : 0.0f) - mu;
        // (u, dw') = (c g - s dn, s g + c dn): one FMUL2 + one FFMA2
        const f2 ud = ffma2(f2_make(-s, c), f2_bc(dn), fmul2(f2_make(c, s), f2_bc(g)));
        const float un = f2_lo(ud);
        const float dwn = f2_hi(ud);
        if (i > 0) {
          const bool wr = i <= m - 1;  // rotation i-1 was a real one
          const float dret = (c1 * (c2 * r1) - s1 * u1) + mu;
          d[i - 1] = wr ? dret : d[i - 1];
          e[i - 1] = wr ? -s1 * r : e[i - 1];
        }
        d[i] = (i == m - 1) ? c1 * dw + mu : d[i];
        c2 = c1;
        c1 = c;
        s1 = s;
        r1 = r;
        u1 = un;
        dw = dwn;
        if (i + 1 < NMAX - 1) g = c1 * e[i + 1];
      }
    }
  });
}

template <int NMAX>
__device__ __forceinline__ int qr_deflate(const float (&e)[NMAX], int m, float eps) {
  unsigned long long small = 0ull;
#pragma unroll
  for (int j = 0; j < NMAX - 1; ++j) small |= (fabsf(e[j]) < eps ? 1ull : 0ull) << j;
  while (m > 2 && ((small >> (m - 2)) & 1ull)) --m;
  return m;
}

template <int NMAX, bool EXACT, bool VECS>
__global__ void __launch_bounds__(kQThreads)
    bed_qr_kernel(int64_t bc, int64_t c0, int n_rt, SplitWs ws, float* __restrict__ evals,
                  int32_t* __restrict__ status_out, int32_t* __restrict__ steps_out,
                  int32_t* __restrict__ flags, KernelCfg cfg, DiagOut dg) {
  const int n = EXACT ? NMAX : n_rt;
  const int64_t j = (int64_t)blockIdx.x * kQThreads + threadIdx.x;
  const bool live = j < bc;
  const int lane = threadIdx.x & 31;
  const int64_t w = j >> 5;  // warp of the chunk
  if (j - lane >= bc) return;  // whole warp past the chunk: it owns no records
  float d[NMAX], e[NMAX];
#pragma unroll
  for (int i = 0; i < NMAX; ++i) {
    d[i] = (live && i < n) ? ws.D[(int64_t)i * ws.Bc + j] : 0.0f;
    e[i] = (live && i < n - 1) ? ws.E[(int64_t)i * ws.Bc + j] : 0.0f;
  }
  int status = live ? ws.vstat[j] : kStatusOk;
  float top = 0.0f;
#pragma unroll
  for (int i = 0; i < NMAX; ++i) top = fmaxf(top, fmaxf(fabsf(d[i]), fabsf(e[i])));
  float iscale;
  const float scale = pow2_ceil(top, &iscale);  // exact powers of two
#pragma unroll
  for (int i = 0; i < NMAX; ++i) {
    d[i] *= iscale;
    e[i] *= iscale;
  }

  float2* recw = VECS ? ws.rot + (size_t)w * ws.Smax * (NMAX - 1) * 32 + lane : nullptr;
  int* mw_rec = VECS ? ws.msw + (size_t)w * ws.Smax : nullptr;
  uint8_t* ml_rec = VECS ? ws.mlane + (size_t)w * ws.Smax * 32 + lane : nullptr;
  int nrec = 0;
  // pad a recorded sweep with identities up to the fold block boundary
  auto pad = [&](int from, int upto) {
    for (int p = from; p < upto; ++p) recw[((size_t)nrec * (NMAX - 1) + p) * 32] = make_float2(1.0f, 0.0f);
  };
  // close a record: `written` positions were stored, the fold will run whole
  // blocks up to the one containing position mw - 2
  // blocks up to the one containing position mw - 2; mine is this lane's
  // active size (the fold skips a lane's no-op sweeps and positions)
  auto record_end = [&](int mw, int written, int mine) {
    if constexpr (VECS) {
      constexpr int kBlk = fold_blk<NMAX>();
      const int padded = min(NMAX - 1, ((mw - 1 + kBlk - 1) / kBlk) * kBlk);
      pad(min(written, NMAX - 1), padded);
      if (lane == 0) mw_rec[nrec] = mw;
      ml_rec[(size_t)nrec * 32] = (uint8_t)mine;
      ++nrec;
    }
  };

  int steps = 0, rot = 0, srs = 0;
  float res_out = 0.0f;
  int m = qr_deflate<NMAX>(e, n, cfg.eps);
  bool run = live && m > 2;
  while (__any_sync(0xffffffffu, run)) {
    if (run && steps >= cfg.max_steps) {  // budget exhausted: qr.py:604-612
      float resid = 0.0f;
#pragma unroll
      for (int i = 0; i < NMAX - 1; ++i) resid = fmaxf(resid, i < m - 1 ? fabsf(e[i]) : 0.0f);
      res_out = resid;
      if (resid >= cfg.eps && status == kStatusOk) status = kStatusNoConv;
      run = false;  // lock the diagonal; the leading 2x2 still closes below
    }
    if (!__any_sync(0xffffffffu, run)) break;
    // trailing 2x2 of the active block via an arithmetic blend
    float ta = 0.0f, tb = 0.0f, td = 0.0f;
#pragma unroll
    for (int i = 1; i < NMAX - 1; ++i) {
      const float wgt = (i == m - 2) ? 1.0f : 0.0f;
      ta = fmaf(wgt, d[i], ta);
      tb = fmaf(wgt, e[i], tb);
      td = fmaf(wgt, d[i + 1], td);
    }
    float lo, hi;
    wilkinson_shifts(ta, tb, td, lo, hi);
    // the two sweeps of the double step (shifts hi, then lo) share one copy
    // of the unrolled sweep code: a runtime loop of two halves the kernel's
    // size (instruction-cache misses stalled it at n = 64)
    srs += run ? n - m : 0;
    int mcur = run ? m : 0;
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      const int mw = __reduce_max_sync(0xffffffffu, mcur);
      if (h == 1 && mw <= 2) break;
      rot += mcur > 2 ? mcur - 1 : 0;
      qr_sweep<NMAX, VECS>(d, e, mcur, h ? lo : hi, VECS ? recw + (size_t)nrec * (NMAX - 1) * 32 : nullptr,
                           mw);
      record_end(mw, mw, mcur);
      if (run) m = qr_deflate<NMAX>(e, m, cfg.eps);
      mcur = (run && m > 2) ? m : 0;
    }
    if (run) {
      ++steps;
      run = m > 2;
    }
  }
  {  // exact 2x2 closeout (_kernels.py:401-417), recorded as a sweep of extent 2
    float lo, hi, c, s;
    wilkinson(d[0], e[0], d[1], lo, hi, c, s);
    d[0] = lo;
    d[1] = hi;
    if constexpr (VECS) {
      recw[(size_t)nrec * (NMAX - 1) * 32] = make_float2(c, s);
      record_end(2, 1, 2);
    }
  }
  if (VECS && lane == 0) ws.nsw[w] = nrec;

  if (live) {
    if constexpr (VECS) {
#pragma unroll
      for (int i = 0; i < NMAX; ++i)
        if (i < n) ws.lam[(int64_t)i * ws.Bc + j] = d[i] * scale;
    } else {  // values only: stable sort in the thread (solver.py:61-66)
#pragma unroll
      for (int c = 0; c < NMAX; ++c) {
        if (c >= n) continue;
        int rk = c;
        if (cfg.sort != 0) {
          rk = 0;
#pragma unroll
          for (int k = 0; k < NMAX; ++k)
            rk += (k < n && k != c && rank_before(d[k], k, d[c], c, cfg.sort)) ? 1 : 0;
        }
        evals[(c0 + j) * n + rk] = d[c] * scale;
      }
    }
    if (status_out) status_out[c0 + j] = status;
    if (steps_out) steps_out[c0 + j] = steps;
    dg.put(c0 + j, rot, n - m, srs, res_out);
  }
  if (flags) {
    unsigned bits = __reduce_or_sync(0xffffffffu, (live && status) ? (1u << status) : 0u);
    if (lane == 0 && bits) atomicOr(flags, (int)bits);
  }
}

}  // namespace bed
