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
//   F (bed_fold_kernel)  lane group per matrix: V := P, then the recorded
//                        rotations applied to V's rows in registers (two
//                        column updates, _kernels.py:269-277), then stable
//                        sort + sign (solver.py:60-76) and coalesced stores.
//
// Values-only solves (solver.py:94-109) run H (band only) and Q, which sorts
// the eigenvalues itself.
#pragma once

#include "bed_f32x2.cuh"
#include "bed_group.cuh"
#include "bed_hh.cuh"
#include "bed_split_ws.cuh"
#include "bed_tile.cuh"

namespace bed {

// ---------------------------------------------------------------------------
// Q: one thread per matrix, band in registers, warp-synchronous sweeps.

// Fused sweep of the leading m-block (_sweep_block), predicated straight-line
// code over all NMAX positions (rotations past a lane's block are exact
// identities; m = 0 is a no-op); positions no lane of the warp needs are
// skipped by a vote.  Returns the warp's processed extent.  With VECS every
// rotation is stored to rec[p * RSTRIDE].
template <int NMAX, bool VECS, int RSTRIDE = 32>
__device__ __forceinline__ int qr_sweep(float (&d)[NMAX], float (&e)[NMAX], int m, float mu,
                                        float2* __restrict__ rec) {
  float dw = d[0] - mu, g = e[0];
  float c1 = 1.0f, s1 = 0.0f, c2 = 1.0f, r1 = 0.0f, u1 = 0.0f;
  int extent = NMAX;
#pragma unroll
  for (int i = 0; i < NMAX; ++i) {
    if (i >= 2 && !__any_sync(0xffffffffu, i <= m - 1)) {
      extent = i;
      break;
    }
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
  return extent;
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
                  int32_t* __restrict__ flags, KernelCfg cfg) {
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
      const int padded = min(NMAX - 1, ((mw - 1 + kFoldBlk - 1) / kFoldBlk) * kFoldBlk);
      pad(min(written, NMAX - 1), padded);
      if (lane == 0) mw_rec[nrec] = mw;
      ml_rec[(size_t)nrec * 32] = (uint8_t)mine;
      ++nrec;
    }
  };

  int steps = 0;
  int m = qr_deflate<NMAX>(e, n, cfg.eps);
  bool run = live && m > 2;
  while (__any_sync(0xffffffffu, run)) {
    if (run && steps >= cfg.max_steps) {  // budget exhausted: qr.py:604-612
      float resid = 0.0f;
#pragma unroll
      for (int i = 0; i < NMAX - 1; ++i) resid = fmaxf(resid, i < m - 1 ? fabsf(e[i]) : 0.0f);
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
    const int ma = run ? m : 0;
    const int mwa = __reduce_max_sync(0xffffffffu, ma);
    qr_sweep<NMAX, VECS>(d, e, ma, hi, VECS ? recw + (size_t)nrec * (NMAX - 1) * 32 : nullptr);
    record_end(mwa, mwa, ma);
    if (run) m = qr_deflate<NMAX>(e, m, cfg.eps);
    const int mb = (run && m > 2) ? m : 0;
    const int mwb = __reduce_max_sync(0xffffffffu, mb);
    if (mwb > 2) {
      qr_sweep<NMAX, VECS>(d, e, mb, lo, VECS ? recw + (size_t)nrec * (NMAX - 1) * 32 : nullptr);
      record_end(mwb, mwb, mb);
    }
    if (run) {
      m = qr_deflate<NMAX>(e, m, cfg.eps);
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
  }
  if (flags) {
    unsigned bits = __reduce_or_sync(0xffffffffu, (live && status) ? (1u << status) : 0u);
    if (lane == 0 && bits) atomicOr(flags, (int)bits);
  }
}

// ---------------------------------------------------------------------------
// F: fold the recorded rotations into V = P, then sort + sign + store.
//
// A CTA holds G matrices of ONE band warp (G divides 32; small CTAs so the
// load / fold / store phases of neighbouring CTAs overlap), so all its
// groups replay the same sweep sequence.  The records are consumed in
// phases of K sweeps (one barrier per phase), copied by cp.async into a
// double-buffered, matrix-major shared buffer one phase ahead; each group
// skips its own no-op sweeps and positions and reads two rotations per
// 128-bit broadcast.
template <int NMAX>
struct FoldParams {
  static constexpr int L = GroupSize<NMAX>::L;
  static constexpr int G = NMAX <= 16 ? 8 : (NMAX <= 32 ? 4 : 8);
  static constexpr int THREADS = G * L;
  static constexpr int SROW = NMAX + 1;
  static constexpr int SMAT = NMAX * SROW;
  static constexpr int PADPOS = ((NMAX - 1 + kFoldBlk - 1) / kFoldBlk) * kFoldBlk;
  static constexpr int K = 4;                                      // sweeps per phase
  static constexpr int RROW = PADPOS + 2;                          // float2 per matrix row
  static constexpr int OFF_ROT = (G * SMAT + 3) / 4 * 4;           // float2 [2][K][G][RROW], 16-byte aligned
  static constexpr int OFF_MM = OFF_ROT + 2 * 2 * K * G * RROW;   // uint8 [2][K][G]
  static constexpr int OFF_FLIP = OFF_MM + (2 * K * G + 3) / 4;
  static constexpr int OFF_EV = OFF_FLIP + G * NMAX;
  static constexpr int OFF_RANK = OFF_EV + G * NMAX;
  static constexpr int OFF_LAM = OFF_RANK + G * NMAX;
  static constexpr int TOTAL = OFF_LAM + G * NMAX;
  static constexpr size_t BYTES = sizeof(float) * TOTAL;
  static constexpr int PER_THREAD = (PADPOS * G + THREADS - 1) / THREADS;  // prefetch slots
  static_assert(32 % G == 0, "a CTA must not straddle band warps");
};

template <int NMAX, bool EXACT>
__global__ void __launch_bounds__(FoldParams<NMAX>::THREADS)
    bed_fold_kernel(int64_t bc, int64_t c0, int n_rt, SplitWs ws, float* __restrict__ evals,
                    float* __restrict__ evecs, KernelCfg cfg) {
  using P = FoldParams<NMAX>;
  constexpr int L = P::L, G = P::G;
  const int n = EXACT ? NMAX : n_rt;
  const int nn = n * n;
  extern __shared__ __align__(16) float smem[];
  float2* rbuf = reinterpret_cast<float2*>(smem + P::OFF_ROT);
  float* flipv = smem + P::OFF_FLIP;
  float* evs = smem + P::OFF_EV;
  int* ranks = reinterpret_cast<int*>(smem + P::OFF_RANK);
  float* lams = smem + P::OFF_LAM;
  const int tid = threadIdx.x;
  const int mi = tid / L;
  const int r = tid % L;
  const int64_t j0 = (int64_t)blockIdx.x * G;
  const int count = (bc - j0) < G ? (int)(bc - j0) : G;
  const bool mlive = mi < count;
  const int64_t j = j0 + mi;
  float* st = smem + mi * P::SMAT;

  if (mlive && r < n) lams[mi * NMAX + r] = ws.lam[(int64_t)r * ws.Bc + j];
  tile_to_stage<NMAX, P::THREADS, P::SROW, P::SMAT>(ws.P + j0 * nn, count, n, smem);
  __syncthreads();
  float v[NMAX];
#pragma unroll
  for (int c = 0; c < NMAX; ++c) v[c] = (mlive && r < n && c < n) ? st[r * P::SROW + c] : 0.0f;

  // rotation stream of this CTA's band warp
  const int64_t w = j0 >> 5;
  const int lane0 = (int)(j0 & 31);
  const int nrec = ws.nsw[w];
  const int* mws = ws.msw + (size_t)w * ws.Smax;
  const float2* recw = ws.rot + (size_t)w * ws.Smax * (NMAX - 1) * 32 + lane0;
  // The stream is consumed in phases of K sweeps with one barrier per
  // phase: while a phase is folded, the next phase's records travel
  // global -> shared by cp.async (no register staging), each thread moving
  // the (position, lane) rotations it covers into the matrix-major buffer
  // [G][RROW], so a group reads two consecutive rotations with one 128-bit
  // broadcast.  Positions past a sweep's padded warp extent are never read
  // (every group's blocks end at or before it), so they are not copied.
  constexpr int K = P::K;
  uint8_t* mbuf = reinterpret_cast<uint8_t*>(smem + P::OFF_MM);  // [2][K][G] active sizes
  const uint8_t* mls = ws.mlane + (size_t)w * ws.Smax * 32 + lane0;
  constexpr int REC = (NMAX - 1) * 32;  // float2 per sweep record
  int q_pos[P::PER_THREAD], q_goff[P::PER_THREAD], q_soff[P::PER_THREAD];
#pragma unroll
  for (int q = 0; q < P::PER_THREAD; ++q) {
    const int e = tid + q * P::THREADS;
    const int pp = e / G, g = e - pp * G;
    q_pos[q] = e < P::PADPOS * G ? pp : NMAX;
    q_goff[q] = pp * 32 + g;
    q_soff[q] = g * P::RROW + pp;
  }
  auto fetch = [&](int ph, int buf) {
    const float2* rs = recw + (size_t)ph * K * REC;
#pragma unroll
    for (int kk = 0; kk < K; ++kk) {
      const int s2 = ph * K + kk;
      if (s2 < nrec) {
        const int mw = __ldg(mws + s2);
        const int npos = min(NMAX - 1, ((mw - 1 + kFoldBlk - 1) / kFoldBlk) * kFoldBlk);
        float2* rb = rbuf + (buf * K + kk) * G * P::RROW;
#pragma unroll
        for (int q = 0; q < P::PER_THREAD; ++q)
          if (q_pos[q] < npos) cp_async8(rb + q_soff[q], rs + kk * REC + q_goff[q]);
        if (tid == 0) cp_async_bytes<G>(mbuf + (buf * K + kk) * G, mls + (size_t)s2 * 32);
      }
    }
    cp_async_commit();
  };
  const int nph = (nrec + K - 1) / K;
  if (nph > 0) fetch(0, 0);
  cp_async_wait_all();
  __syncthreads();
#pragma unroll 1
  for (int ph = 0; ph < nph; ++ph) {
    const int buf = ph & 1;
    if (ph + 1 < nph) fetch(ph + 1, buf ^ 1);  // lands while this phase is folded
#pragma unroll 1
    for (int kk = 0; kk < K; ++kk) {
      // this matrix's active size in the sweep (0: no-op; past nrec: 0)
      const int mm = ph * K + kk < nrec ? mbuf[(buf * K + kk) * G + mi] : 0;
      if (mlive && mm > 1) {
        const float2* rs = rbuf + ((buf * K + kk) * G + mi) * P::RROW;
        static_for<0, (NMAX - 1 + kFoldBlk - 1) / kFoldBlk>([&](auto bcst) {
          constexpr int b0 = decltype(bcst)::value * kFoldBlk;
          constexpr int b1 = b0 + kFoldBlk < NMAX - 1 ? b0 + kFoldBlk : NMAX - 1;
          if (b0 < mm - 1) {
#pragma unroll
            for (int p = b0; p < b1; p += 2) {
              // two rotations per 128-bit broadcast; scalar FMAs on purpose:
              // the packed form (FMUL2 -> FFMA2) lengthens the position-to-
              // position dependency chain and doubles the row's register
              // footprint, which measured slower here
              const float4 c2 = *reinterpret_cast<const float4*>(rs + p);
              {
                const float x = v[p], y = v[p + 1];
                v[p] = c2.x * x - c2.y * y;
                v[p + 1] = fmaf(c2.y, x, c2.x * y);
              }
              if (p + 1 < b1) {
                const float x = v[p + 1], y = v[p + 2];
                v[p + 1] = c2.z * x - c2.w * y;
                v[p + 2] = fmaf(c2.w, x, c2.z * y);
              }
            }
          }
        });
      }
    }
    cp_async_wait_all();
    __syncthreads();
  }

  // stable sort + sign (solver.py:60-76), transposed staging, coalesced store
  if (mlive && r < n) {
    const float lr = lams[mi * NMAX + r];
    int rk = r;
    if (cfg.sort != 0) {
      rk = 0;
      for (int k2 = 0; k2 < n; ++k2)
        rk += (k2 != r && rank_before(lams[mi * NMAX + k2], k2, lr, r, cfg.sort)) ? 1 : 0;
    }
    ranks[mi * NMAX + r] = rk;
    evs[mi * NMAX + rk] = lr;
  }
  __syncthreads();
  if (mlive && r < n) {
#pragma unroll
    for (int c = 0; c < NMAX; ++c)
      if (c < n) st[r * P::SROW + ranks[mi * NMAX + c]] = v[c];
  }
  __syncthreads();
  if (mlive && r < n) {  // sign: largest-magnitude entry of column r >= 0
    float best = -1.0f, lead = 0.0f;
    for (int rr = 0; rr < n; ++rr) {
      const float x = st[rr * P::SROW + r];
      if (fabsf(x) > best) {
        best = fabsf(x);
        lead = x;
      }
    }
    flipv[mi * NMAX + r] = lead < 0.0f ? -1.0f : 1.0f;
  }
  __syncthreads();
  {
    stage_to_tile<NMAX, P::THREADS, P::SROW, P::SMAT>(smem, count, n, evecs + (c0 + j0) * nn, flipv);
    float* dstl = evals + (c0 + j0) * n;
    for (int g = tid; g < count * n; g += P::THREADS) {
      int mat = g / n, c = g - mat * n;
      dstl[g] = evs[mat * NMAX + c];
    }
  }
}

}  // namespace bed
