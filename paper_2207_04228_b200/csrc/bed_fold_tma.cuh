// bed_fold_tma.cuh -- F stage of the split medium path: fold the rotation
// record of bed_qr_kernel into V = P (the column updates of _kernels.py:
// 269-277; V starts as P = H_0 H_1 ..., so V = P Q of solver.py:93 needs no
// GEMM), then stable sort + sign (solver.py:60-76) and coalesced stores.
//
// A CTA owns MPC consecutive matrices of one band warp.  A producer warp
// streams that warp's sweep records global -> shared with bulk async copies
// (TMA engine, cp.async.bulk: one copy per sweep of the rows its extent
// covers, all 32 lanes -- the CTAs sharing a band warp read it from L2) into
// an NB-deep ring; each slot completes an mbarrier by transaction count.  The fold
// threads -- LF per matrix, R rows of V each, held in registers (packed row
// pairs for R even, so a rotation of two columns costs 2 FMUL2 + 2 FFMA2 per
// two rows) -- wait on the slot's barrier, apply the sweep, and release the
// slot through a second mbarrier.  Each fold warp applies only the
// positions its own matrices need (the largest active size among them, put
// in the slot header by the producer; the record holds exact identities past
// a matrix's block), in blocks of BLK positions whose rotations are loaded
// ahead of the arithmetic, and skips sweeps in which all of them sit out.
#pragma once

#include "bed_mbar.cuh"
#include "bed_f32x2.cuh"
#include "bed_split_ws.cuh"
#include "bed_tile.cuh"

namespace bed {

// EXACT = n equals the tier's NMAX.  At n = 32 four rows per fold thread
// (LF = 8) beat two (65 536 matrices: 1.121 -> 1.096 ms) but not for the padded
// n = 25..31 (1.124 -> 1.152 ms at n = 26), which keep two.
template <int NMAX, bool EXACT = true>
struct FTParams {
  static constexpr int LF = NMAX <= 16 ? 4 : (NMAX <= 24 ? 6 : (NMAX <= 32 ? (EXACT ? 8 : 16) : 32));
  static constexpr int R = NMAX / LF;     // rows per fold thread: 4, 4, 4 (2 padded), 2
  static constexpr int RP = (R + 1) / 2;  // packed row pairs (R = 1: scalar rows)
  static constexpr int MPC = NMAX <= 16 ? 32 : (NMAX <= 32 ? 16 : 8);
  static constexpr int FT = MPC * LF;
  static constexpr int THREADS = FT + 32;  // + the producer warp
  static constexpr int MINB = NMAX <= 24 ? 4 : (NMAX <= 32 ? 2 : 1);
  static constexpr int NB = NMAX >= 32 ? 8 : 6;  // 8 fits inside the sort stage at n >= 32
  static constexpr int NW = FT / 32;   // fold warps
  static constexpr int BLK = fold_blk<NMAX>();  // positions per fold block (one branch, loads hoisted)
  static constexpr int POS = NMAX - 1;
  static constexpr int SLOT = POS * 32;  // float2 per ring slot: a whole sweep record [position][lane]
  static constexpr int RING = NB * SLOT * 2;
  static constexpr int SROW = NMAX + 1;
  static constexpr int SMAT = NMAX * SROW;
  static constexpr int STAGE = MPC * SMAT;
  static constexpr int U = ((RING > STAGE ? RING : STAGE) + 3) / 4 * 4;
  static constexpr int OFF_LAM = U;
  static constexpr int OFF_EV = OFF_LAM + MPC * NMAX;
  static constexpr int OFF_RANK = OFF_EV + MPC * NMAX;
  static constexpr int OFF_FLIP = OFF_RANK + MPC * NMAX;
  static constexpr int OFF_BAR = (OFF_FLIP + MPC * NMAX + 1) / 2 * 2;  // 8-byte aligned
  static constexpr int OFF_HDR = OFF_BAR + 2 * 2 * NB;                 // full[NB], empty[NB]
  static constexpr int TOTAL = OFF_HDR + NB * NW;                      // per slot: each fold warp's extent
  static constexpr size_t BYTES = sizeof(float) * (size_t)TOTAL;
  static_assert(R * LF == NMAX && (R % 2 == 0 || R == 1), "row split");
  static_assert(FT % 32 == 0 && 32 % MPC == 0, "CTA = whole warps, one band warp's lanes");
  static_assert(MPC % 4 == 0 && NW <= 8, "active sizes read as words; fold-warp extents packed in 8 bytes");
};

// POW: instead of V, write the spectral power V diag(max(lambda, floor)^p) V^T
// (matrix_power, solver.py:115-143) to `evecs` -- formed from V in registers
// and a shared copy of it, so V never reaches memory.
// Each entry sums fma(V[r][k] V[c][k], f_k) in k order, which is symmetric in
// (r, c), so the output is exactly symmetric (solver.py:141).
template <int NMAX, bool EXACT, bool POW = false>
__global__ void __launch_bounds__(FTParams<NMAX, EXACT>::THREADS, FTParams<NMAX, EXACT>::MINB)
    bed_fold_tma_kernel(int64_t bc, int64_t c0, int n_rt, SplitWs ws, float* __restrict__ evals,
                        float* __restrict__ evecs, KernelCfg cfg, PowSpec pw = PowSpec{},
                        int32_t* __restrict__ status_out = nullptr, int32_t* __restrict__ flags = nullptr) {
  using P = FTParams<NMAX, EXACT>;
  constexpr int LF = P::LF, R = P::R, RP = P::RP, MPC = P::MPC, NB = P::NB, POS = P::POS;
  const int n = EXACT ? NMAX : n_rt;
  const int nn = n * n;
  extern __shared__ __align__(16) float smem[];
  float2* ring = reinterpret_cast<float2*>(smem);
  float* lams = smem + P::OFF_LAM;
  float* evs = smem + P::OFF_EV;
  int* ranks = reinterpret_cast<int*>(smem + P::OFF_RANK);
  float* flipv = smem + P::OFF_FLIP;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + P::OFF_BAR);
  uint64_t* empty = full + NB;
  const int tid = threadIdx.x;
  const int64_t j0 = (int64_t)blockIdx.x * MPC;
  const int count = (bc - j0) < MPC ? (int)(bc - j0) : MPC;
  const int64_t w = j0 >> 5;            // band warp of the chunk
  const int lane0 = (int)(j0 & 31);     // its first lane in this CTA
  const int nrec = ws.nsw[w];
  const int* msw = ws.msw + (size_t)w * ws.Smax;
  const uint8_t* mls = ws.mlane + (size_t)w * ws.Smax * 32 + lane0;
  const float2* recw = ws.rot + (size_t)w * ws.Smax * POS * 32;  // the band warp's record

  if (tid == 0) {
    for (int b = 0; b < NB; ++b) {
      mbar_init(full + b, 1);
      mbar_init(empty + b, P::FT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int mi = tid / LF, l = tid % LF;
  const bool mlive = tid < P::FT && mi < count;
  if (mlive) {
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const int c = l + LF * rr;
      if (c < n) lams[mi * NMAX + c] = ws.lam[(int64_t)c * ws.Bc + j0 + mi];
    }
  }
  __syncthreads();

  // V rows: packed pairs (rows l + LF * 2rp, l + LF * (2rp + 1)) or, for
  // R = 1, one scalar row l
  f2 v[RP][NMAX];
  float vs[R == 1 ? NMAX : 1];

  if (tid >= P::FT) {
    // ------------------------------------------------------------ producer warp
    // Per sweep: the warp's extent (msw) bounds the rows to copy -- Q wrote
    // every row up to the fold-block boundary past it (identities beyond a
    // lane's block) -- and each fold warp's extent (the largest active size
    // among its matrices, from mlane) goes into the slot header.
    const int lane = tid & 31;
    int* hdr = reinterpret_cast<int*>(smem + P::OFF_HDR);
#pragma unroll 1
    for (int s0 = 0; s0 < nrec; s0 += 32) {
      // lane k fetches sweep s0 + k's metadata once per 32 sweeps: the warp's
      // extent and the active sizes of this CTA's MPC matrices, from which it
      // forms each fold warp's extent (NW bytes packed in two words)
      const int sk = s0 + lane;
      const int mw_l = sk < nrec ? __ldg(msw + sk) : 0;
      uint32_t wpk[2] = {0u, 0u};
      if (sk < nrec) {
        uint8_t ml[MPC];
#pragma unroll
        for (int q = 0; q < MPC; q += 4) {
          const uint32_t wd = __ldg(reinterpret_cast<const uint32_t*>(mls + (size_t)sk * 32 + q));
          ml[q] = wd & 0xff; ml[q + 1] = (wd >> 8) & 0xff; ml[q + 2] = (wd >> 16) & 0xff; ml[q + 3] = wd >> 24;
        }
#pragma unroll
        for (int f = 0; f < P::NW; ++f) {
          int mx = 0;
#pragma unroll
          for (int k = 0; k < MPC; ++k)
            if (k >= (32 * f) / LF && k <= (32 * f + 31) / LF) mx = max(mx, (int)ml[k]);
          wpk[f / 4] |= (uint32_t)mx << (8 * (f % 4));
        }
      }
#pragma unroll 1
      for (int s = s0; s < min(nrec, s0 + 32); ++s) {
        const int b = s % NB;
        const int mw = __shfl_sync(0xffffffffu, mw_l, s - s0);
        const int np = min(POS, (mw - 1 + P::BLK - 1) / P::BLK * P::BLK);
        if (s >= NB) mbar_wait(empty + b, ((s / NB) & 1) ^ 1);
        if (lane == s - s0) {
#pragma unroll
          for (int f = 0; f < P::NW; ++f) hdr[b * P::NW + f] = (wpk[f / 4] >> (8 * (f % 4))) & 0xff;
        }
        __syncwarp();
        if (lane == 0) {  // rows 0 .. np-1 of the sweep record: one contiguous bulk copy
          mbar_arrive_tx(full + b, (unsigned)(np * 32 * 8));
          bulk_g2s(ring + b * P::SLOT, recw + (size_t)s * POS * 32, np * 32 * 8, full + b);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ fold threads
    const float* pm = ws.P + (j0 + mi) * nn;
    if constexpr (R == 1) {
      const bool ok = mlive && l < n;
#pragma unroll
      for (int c = 0; c < NMAX; ++c) vs[c] = (ok && c < n) ? __ldg(pm + l * n + c) : 0.0f;
    } else {
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
    }
    const int* hdr = reinterpret_cast<const int*>(smem + P::OFF_HDR) + (tid >> 5);
#pragma unroll 1
    for (int s = 0; s < nrec; ++s) {
      const int b = s % NB;
      mbar_wait(full + b, (s / NB) & 1);
      const int wm = hdr[b * P::NW];  // positions 0 .. wm - 2 hold this warp's rotations
      const float2* rs = ring + b * P::SLOT + lane0 + mi;
      static_for<0, (POS + P::BLK - 1) / P::BLK>([&](auto bcst) {
        constexpr int p0 = decltype(bcst)::value * P::BLK;
        constexpr int p1 = p0 + P::BLK < POS ? p0 + P::BLK : POS;
        if (p0 < wm - 1) {  // the block's rows were copied (whole fold blocks)
          float2 cs[P::BLK];
#pragma unroll
          for (int p = p0; p < p1; ++p) cs[p - p0] = rs[p * 32];
#pragma unroll
          for (int p = p0; p < p1; ++p) {
            if constexpr (R == 1) {
              const float x = vs[p], y = vs[p + 1];
              vs[p] = cs[p - p0].x * x - cs[p - p0].y * y;
              vs[p + 1] = fmaf(cs[p - p0].y, x, cs[p - p0].x * y);
            } else {
#pragma unroll
              for (int rp = 0; rp < RP; ++rp)
                rot2_ip(v[rp][p], v[rp][p + 1], cs[p - p0].x, cs[p - p0].y, -cs[p - p0].y);
            }
          }
        }
      });
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(empty + b);
    }
  }
  __syncthreads();  // every slot was consumed: the ring is free for the stage

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
  if constexpr (POW) {
    static_assert(R % 2 == 0, "power epilogue on packed row pairs");
    float* fv = flipv;  // f_k per matrix, unsorted order (as V's columns)
    if (mlive) {
#pragma unroll
      for (int rp = 0; rp < RP; ++rp) {
        const int r0 = l + LF * (2 * rp), r1 = r0 + LF;
#pragma unroll
        for (int c = 0; c < NMAX; ++c) {
          if (r0 < NMAX) st[r0 * P::SROW + c] = f2_lo(v[rp][c]);
          if (r1 < NMAX) st[r1 * P::SROW + c] = f2_hi(v[rp][c]);
        }
      }
      if (l == 0) {  // floor, positivity check, f (solver.py:127-139)
        float lmax = lams[mi * NMAX];
        for (int k = 1; k < n; ++k) lmax = fmaxf(lmax, lams[mi * NMAX + k]);
        const float fl = pw.floor_abs < 0.0f ? 1e-12f * lmax : pw.floor_abs;
        bool bad = false;
        for (int k = 0; k < n; ++k) {
          const float x = fmaxf(lams[mi * NMAX + k], fl);
          bad = bad || (pw.needs_positive && !(x > 0.0f));
          fv[mi * NMAX + k] = x;
        }
        for (int k = 0; k < NMAX; ++k) fv[mi * NMAX + k] = (bad || k >= n) ? 0.0f : spectral_pow(fv[mi * NMAX + k], pw.p);
        const int64_t j = c0 + j0 + mi;
        if (bad && (!status_out || status_out[j] == kStatusOk)) {  // the forward's status wins
          if (status_out) status_out[j] = kStatusNonPositive;
          if (flags) atomicOr(flags, 1 << kStatusNonPositive);
        }
      }
    }
    __syncthreads();
    if (mlive) {
      const float* fk = fv + mi * NMAX;
      float* om = evecs + (c0 + j0 + mi) * nn;
#pragma unroll
      for (int rp = 0; rp < RP; ++rp) {
        const int r0 = l + LF * (2 * rp), r1 = r0 + LF;
        for (int c = 0; c < n; ++c) {
          const float* vc = st + c * P::SROW;
          f2 acc = f2_bc(0.0f);
#pragma unroll
          for (int k = 0; k < NMAX; ++k) acc = ffma2(fmul2(v[rp][k], f2_bc(vc[k])), f2_bc(fk[k]), acc);
          if (r0 < n) om[r0 * n + c] = f2_lo(acc);
          if (r1 < n) om[r1 * n + c] = f2_hi(acc);
        }
      }
    }
  } else if (mlive) {
    if constexpr (R == 1) {
#pragma unroll
      for (int c = 0; c < NMAX; ++c)
        if (c < n && l < n) st[l * P::SROW + ranks[mi * NMAX + c]] = vs[c];
    } else {
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
  }
  if constexpr (!POW) {
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
  }
  float* dstl = evals + (c0 + j0) * n;
  for (int g = tid; g < count * n; g += P::THREADS) {
    const int mat = g / n, c = g - mat * n;
    dstl[g] = evs[mat * NMAX + c];
  }
}

}  // namespace bed
