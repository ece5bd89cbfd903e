// bed_qf.cuh -- fused band QR + eigenvector fold for 9 <= n <= 24 (the "QF"
// kernel).  It replaces the Q and F kernels of bed_split.cuh on the vectors
// path: the rotations of every sweep pass from the band warp to the fold warps
// through a shared-memory ring instead of a record in HBM.
//
// A CTA owns MPC matrices:
//   * one band warp (the last warp): lane k runs matrix k's band QR exactly as
//     bed_qr_kernel does -- equilibration (qr.py:522-534), double-shift sweeps
//     (_sweep_block, _kernels.py:221-300) with per-matrix deflation
//     (qr_loop_kernel :321-398 with the gate of :381-388), 2x2 closeout
//     (:401-417) -- and writes each sweep's rotations into a ring slot;
//   * MPC * LF fold threads: LF threads per matrix, R rows of V each, held in
//     registers as packed row pairs so a rotation of two columns costs
//     2 FMUL2 + 2 FFMA2 per two rows (the column update of _kernels.py:
//     269-277); V starts as P = H_0 H_1 ... written by bed_hh_kernel, so
//     V = P Q (solver.py:93) needs no GEMM.
// Slots are handed over with named barriers (FULL: band warp arrives, fold
// threads wait; EMPTY: the reverse), NB slots deep, so the band warp runs up
// to NB sweeps ahead of the fold.  A slot holds, per matrix, the rotations of
// positions 0 .. ext-2 (ext = the warp's largest active size in that sweep;
// a matrix whose block is smaller, or that has finished, recorded exact
// identities there), read by the fold two at a time with 128-bit broadcasts.
// ext = 2 is the closeout, ext = 0 ends the stream.  Then stable sort + sign
// (solver.py:60-76) through a shared stage that reuses the ring, and
// coalesced stores.
#pragma once

#include "bed_split.cuh"

namespace bed {

template <int NMAX>
struct QFParams {
  static constexpr int LF = NMAX <= 16 ? 4 : (NMAX <= 24 ? 6 : 16);    // fold threads per matrix
  static constexpr int R = NMAX / LF;                                  // rows per fold thread
  static constexpr int RP = R / 2;                                     // packed row pairs
  static constexpr int MPC = NMAX <= 16 ? 32 : 16;                     // matrices per CTA
  static constexpr int FT = MPC * LF;                                  // fold threads
  static constexpr int THREADS = FT + 32;                              // + the band warp
  static constexpr int MINB = NMAX <= 24 ? 4 : 2;                      // CTAs per SM
  static constexpr int NB = 4;                                         // ring slots (sweeps)
  static constexpr int PADPOS = NMAX;                                  // positions per slot row (even)
  static constexpr int RROW = PADPOS + 2;                              // float2 per matrix row
  static constexpr int RING = NB * 32 * RROW * 2;                      // floats (32 rows: every band lane)
  static constexpr int SROW = NMAX + 1;
  static constexpr int SMAT = NMAX * SROW;
  static constexpr int STAGE = MPC * SMAT;
  static constexpr int U = ((RING > STAGE ? RING : STAGE) + 3) / 4 * 4;
  static constexpr int OFF_LAM = U;                 // [MPC][NMAX] unsorted eigenvalues
  static constexpr int OFF_EV = OFF_LAM + MPC * NMAX;
  static constexpr int OFF_RANK = OFF_EV + MPC * NMAX;
  static constexpr int OFF_FLIP = OFF_RANK + MPC * NMAX;
  static constexpr int OFF_EXT = OFF_FLIP + MPC * NMAX;
  static constexpr int TOTAL = OFF_EXT + NB;
  static constexpr size_t BYTES = sizeof(float) * (size_t)TOTAL;
  static_assert(R % 2 == 0 && R * LF == NMAX, "rows come in packed pairs");
  static_assert(FT % 32 == 0 && MPC <= 32, "fold threads fill whole warps");
  static_assert(2 + 2 * NB <= 16, "named barrier ids");
};

__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <int NMAX, bool EXACT>
__global__ void __launch_bounds__(QFParams<NMAX>::THREADS, QFParams<NMAX>::MINB)
    bed_qf_kernel(int64_t bc, int64_t c0, int n_rt, SplitWs ws, float* __restrict__ evals,
                  float* __restrict__ evecs, int32_t* __restrict__ status_out,
                  int32_t* __restrict__ steps_out, int32_t* __restrict__ flags, KernelCfg cfg) {
  using P = QFParams<NMAX>;
  constexpr int LF = P::LF, R = P::R, RP = P::RP, MPC = P::MPC, NB = P::NB, RROW = P::RROW;
  constexpr int FULL = 1, EMPTY = 1 + NB;  // named barrier ids (0 is __syncthreads)
  const int n = EXACT ? NMAX : n_rt;
  const int nn = n * n;
  extern __shared__ __align__(16) float smem[];
  float2* ring = reinterpret_cast<float2*>(smem);
  float* lams = smem + P::OFF_LAM;
  float* evs = smem + P::OFF_EV;
  int* ranks = reinterpret_cast<int*>(smem + P::OFF_RANK);
  float* flipv = smem + P::OFF_FLIP;
  int* ext_s = reinterpret_cast<int*>(smem + P::OFF_EXT);
  const int tid = threadIdx.x;
  const int64_t j0 = (int64_t)blockIdx.x * MPC;
  const int count = (bc - j0) < MPC ? (int)(bc - j0) : MPC;

  f2 v[RP][NMAX];  // fold threads: rows (l + LF * 2rp, l + LF * (2rp + 1)) of V
  const int mi = tid / LF, l = tid % LF;
  const bool mlive = tid < P::FT && mi < count;

  if (tid >= P::FT) {
    // ------------------------------------------------------------ band warp
    const int lane = tid & 31;
    const int64_t j = j0 + lane;
    const bool live = lane < count;
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
    int slot = 0;
    auto acquire = [&]() -> float2* {
      const int b = slot % NB;
      if (slot >= NB) named_sync(EMPTY + b, P::THREADS);
      return ring + (b * 32 + lane) * RROW;
    };
    auto publish = [&](int ext) {
      const int b = slot % NB;
      if (lane == 0) ext_s[b] = ext;
      __syncwarp();
      named_arrive(FULL + b, P::THREADS);
      ++slot;
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
      float ta = 0.0f, tb = 0.0f, td = 0.0f;  // trailing 2x2 via an arithmetic blend
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
      qr_sweep<NMAX, true, 1>(d, e, ma, hi, acquire());
      publish(mwa);
      if (run) m = qr_deflate<NMAX>(e, m, cfg.eps);
      const int mb = (run && m > 2) ? m : 0;
      const int mwb = __reduce_max_sync(0xffffffffu, mb);
      if (mwb > 2) {
        qr_sweep<NMAX, true, 1>(d, e, mb, lo, acquire());
        publish(mwb);
      }
      if (run) {
        m = qr_deflate<NMAX>(e, m, cfg.eps);
        ++steps;
        run = m > 2;
      }
    }
    {  // exact 2x2 closeout (_kernels.py:401-417): a slot of extent 2
      float lo, hi, c, s;
      wilkinson(d[0], e[0], d[1], lo, hi, c, s);
      d[0] = lo;
      d[1] = hi;
      float2* rec = acquire();
      rec[0] = make_float2(c, s);
      rec[1] = make_float2(1.0f, 0.0f);  // the pair partner the fold reads
      publish(2);
    }
    acquire();
    publish(0);  // end of stream
    for (int k = slot > NB ? slot - NB : 0; k < slot; ++k) named_sync(EMPTY + k % NB, P::THREADS);
    if (live) {
#pragma unroll
      for (int i = 0; i < NMAX; ++i)
        if (i < n) lams[lane * NMAX + i] = d[i] * scale;
      if (status_out) status_out[c0 + j] = status;
      if (steps_out) steps_out[c0 + j] = steps;
    }
    if (flags) {
      unsigned bits = __reduce_or_sync(0xffffffffu, (live && status) ? (1u << status) : 0u);
      if (lane == 0 && bits) atomicOr(flags, (int)bits);
    }
  } else {
    // ------------------------------------------------------------ fold threads
    // V := P, rows straight from the workspace (each row is n contiguous floats)
    const float* pm = ws.P + (j0 + mi) * nn;
#pragma unroll
    for (int rp = 0; rp < RP; ++rp) {
      const int r0 = l + LF * (2 * rp), r1 = r0 + LF;
      const bool ok0 = mlive && r0 < n, ok1 = mlive && r1 < n;
      if (EXACT && NMAX % 4 == 0) {
#pragma unroll
        for (int c4 = 0; c4 < NMAX / 4; ++c4) {
          const float4 x = ok0 ? __ldg(reinterpret_cast<const float4*>(pm + r0 * NMAX) + c4)
                               : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
          const float4 y = ok1 ? __ldg(reinterpret_cast<const float4*>(pm + r1 * NMAX) + c4)
                               : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
          v[rp][4 * c4] = f2_make(x.x, y.x);
          v[rp][4 * c4 + 1] = f2_make(x.y, y.y);
          v[rp][4 * c4 + 2] = f2_make(x.z, y.z);
          v[rp][4 * c4 + 3] = f2_make(x.w, y.w);
        }
      } else {
#pragma unroll
        for (int c = 0; c < NMAX; ++c) {
          const float x = (ok0 && c < n) ? __ldg(pm + r0 * n + c) : 0.0f;
          const float y = (ok1 && c < n) ? __ldg(pm + r1 * n + c) : 0.0f;
          v[rp][c] = f2_make(x, y);
        }
      }
    }
    // apply the stream of sweeps
#pragma unroll 1
    for (int slot = 0;; ++slot) {
      const int b = slot % NB;
      named_sync(FULL + b, P::THREADS);
      const int ext = ext_s[b];
      if (ext == 0) {
        named_arrive(EMPTY + b, P::THREADS);
        break;
      }
      const float2* rs = ring + (b * 32 + mi) * RROW;
      static_for<0, NMAX / 2>([&](auto qc) {
        constexpr int p = 2 * decltype(qc)::value;
        if (p < ext - 1) {
          const float4 cs = *reinterpret_cast<const float4*>(rs + p);
#pragma unroll
          for (int rp = 0; rp < RP; ++rp) rot2(v[rp][p], v[rp][p + 1], cs.x, cs.y, -cs.y);
          if constexpr (p + 1 < NMAX - 1) {
#pragma unroll
            for (int rp = 0; rp < RP; ++rp) rot2(v[rp][p + 1], v[rp][p + 2], cs.z, cs.w, -cs.w);
          }
        }
      });
      named_arrive(EMPTY + b, P::THREADS);
    }
  }
  __syncthreads();  // eigenvalues are in lams; the ring is free for the stage

  // ---- stable sort + sign (solver.py:60-76): fold thread l ranks columns l + LF * rr
  float* st = smem + (tid < P::FT ? mi : 0) * P::SMAT;
  if (mlive) {
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const int c = l + LF * rr;
      if (c < n) {
        const float lc = lams[mi * NMAX + c];
        int rk = c;
        if (cfg.sort != 0) {
          rk = 0;
          for (int k = 0; k < n; ++k)
            rk += (k != c && rank_before(lams[mi * NMAX + k], k, lc, c, cfg.sort)) ? 1 : 0;
        }
        ranks[mi * NMAX + c] = rk;
        evs[mi * NMAX + rk] = lc;
      }
    }
  }
  __syncthreads();
  if (mlive) {
#pragma unroll
    for (int rp = 0; rp < RP; ++rp) {
      const int r0 = l + LF * (2 * rp), r1 = r0 + LF;
#pragma unroll
      for (int c = 0; c < NMAX; ++c) {
        if (c < n) {
          const int rk = ranks[mi * NMAX + c];
          if (r0 < n) st[r0 * P::SROW + rk] = f2_lo(v[rp][c]);
          if (r1 < n) st[r1 * P::SROW + rk] = f2_hi(v[rp][c]);
        }
      }
    }
  }
  __syncthreads();
  if (mlive) {  // sign: the largest-magnitude entry of each column is >= 0
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const int c = l + LF * rr;
      if (c < n) {
        float best = -1.0f, lead = 0.0f;
        for (int r = 0; r < n; ++r) {
          const float x = st[r * P::SROW + c];
          if (fabsf(x) > best) {
            best = fabsf(x);
            lead = x;
          }
        }
        flipv[mi * NMAX + c] = lead < 0.0f ? -1.0f : 1.0f;
      }
    }
  }
  __syncthreads();
  stage_to_tile<NMAX, P::THREADS, P::SROW, P::SMAT>(smem, count, n, evecs + (c0 + j0) * nn, flipv);
  float* dstl = evals + (c0 + j0) * n;
  for (int g = tid; g < count * n; g += P::THREADS) {
    const int mat = g / n, c = g - mat * n;
    dstl[g] = evs[mat * NMAX + c];
  }
}

}  // namespace bed
