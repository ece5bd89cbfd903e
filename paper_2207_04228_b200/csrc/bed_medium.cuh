// bed_medium.cuh -- forward ED for 9 <= n <= 64 (templated on NMAX >= n).
//
// A CTA solves T matrices.  Every matrix gets a lane group of L lanes
// (L = 16 for NMAX <= 16, 32 for NMAX <= 32, 64 = two warps above that);
// lane l of the group owns row l of the matrix and, later, row l of V.
//
//   1. tile load     T*n*n floats, coalesced, into a padded shared stage
//   2. validate      symmetrise + finiteness + asymmetry, group reductions
//                    (core.py:286-309)
//   3. Householder   lane-row form: the lane's matrix row in registers,
//                    reflector u_i written to shared memory and read back as
//                    broadcasts, group reductions for the norms and dots
//                    (_kernels.py:36-92)
//   4. P             V := H_0 H_1 ... row by row in registers (= P of
//                    householder.py:216-231); V is then folded in place, so
//                    V = P Q (solver.py:93) costs no GEMM
//   5. band QR       decoupled from V: lane k of warp 0 runs matrix k's band
//                    recurrence (qr_loop_kernel _kernels.py:321-398 with the
//                    deflation gate applied per matrix, _sweep_block
//                    _kernels.py:221-300) out of shared memory and records
//                    every rotation (c, s) into a ring of S sweeps; one
//                    warp-instruction stream thereby carries T matrices'
//                    scalar chains instead of every lane of every group
//                    repeating its matrix's chain
//   6. fold          each lane applies the recorded rotations to its V row
//                    in registers (two-column updates, _kernels.py:269-277);
//                    steps 5 and 6 alternate chunk by chunk
//   7. sort + sign   ranks and column signs via shared memory, coalesced
//                    stores (solver.py:60-76)
#pragma once

#include "bed_common.cuh"

namespace bed {

constexpr int kFoldBlk = 8;  // fold granularity (positions per static block)

template <int NMAX, int T_, int S_>
struct MedParams {
  static constexpr int L = NMAX <= 16 ? 16 : (NMAX <= 32 ? 32 : 64);
  static constexpr int T = T_;
  static constexpr int S = S_;  // sweeps per band chunk
  static constexpr int THREADS = T * L;
  static_assert(THREADS % 32 == 0, "lane groups must tile whole warps");
  static_assert(T <= 32, "one band lane per matrix in warp 0");
  static_assert(L != 64 || T <= 15, "one named barrier per two-warp group");
  static constexpr int SROW = NMAX + 1;     // padded row stride (odd)
  static constexpr int SMAT = NMAX * SROW;  // per-matrix stage
  // shared memory carve-up, in 4-byte words
  static constexpr int OFF_STAGE = 0;
  static constexpr int OFF_Q = OFF_STAGE + T * SMAT;
  static constexpr int OFF_D = OFF_Q + T * NMAX;
  static constexpr int OFF_E = OFF_D + NMAX * T;
  static constexpr int OFF_EV = OFF_E + NMAX * T;
  static constexpr int OFF_FLIP = OFF_EV + T * NMAX;
  static constexpr int OFF_SCALE = OFF_FLIP + T * NMAX;
  static constexpr int OFF_RED = OFF_SCALE + T;       // [T][4] cross-warp scratch
  static constexpr int OFF_RANK = OFF_RED + 4 * T;    // int [T][NMAX]
  static constexpr int OFF_MS = OFF_RANK + T * NMAX;  // int [S][T]
  static constexpr int OFF_ROT = ((OFF_MS + S * T + 1) / 2) * 2;  // float2 [S][NMAX-1][T]
  static constexpr int TOTAL = OFF_ROT + 2 * S * (NMAX - 1) * T;
  static constexpr size_t BYTES = sizeof(float) * TOTAL;
};

// Communication inside one matrix's lane group.  L <= 32: shuffles within
// the group's lanes.  L == 64: two warps -- warp shuffles, then a two-slot
// exchange through shared memory ordered by a named barrier per group.
template <int L>
struct Group {
  unsigned mask;  // lanes of this warp in the group
  int bar;        // named barrier id (L == 64)
  float* red;     // 4-word scratch (L == 64)
  int gl;         // lane in group

  __device__ __forceinline__ void sync() const {
    if constexpr (L <= 32) __syncwarp(mask);
    else asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(64) : "memory");
  }
  template <bool IS_MAX>
  __device__ __forceinline__ float reduce(float x) const {
    constexpr int W = L <= 32 ? L : 32;
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) {
      float y = __shfl_xor_sync(mask, x, o, W);
      x = IS_MAX ? fmaxf(x, y) : x + y;
    }
    if constexpr (L == 64) {
      if ((gl & 31) == 0) red[gl >> 5] = x;
      sync();
      x = IS_MAX ? fmaxf(red[0], red[1]) : red[0] + red[1];
      sync();
    }
    return x;
  }
  __device__ __forceinline__ float max(float x) const { return reduce<true>(x); }
  __device__ __forceinline__ float sum(float x) const { return reduce<false>(x); }
  // value held by group lane `src` (a compile-time constant at every call)
  __device__ __forceinline__ float bcast(float x, int src) const {
    if constexpr (L <= 32) {
      return __shfl_sync(mask, x, src, L);
    } else {
      if (gl == src) red[2] = x;
      sync();
      float res = red[2];
      sync();
      return res;
    }
  }
};

template <int NMAX, bool EXACT, bool VECS, int T_, int S_>
__global__ void __launch_bounds__(MedParams<NMAX, T_, S_>::THREADS, 1)
    bed_medium_kernel(const float* __restrict__ A, int64_t batch, int n_rt,
                      float* __restrict__ evals, float* __restrict__ evecs,
                      int32_t* __restrict__ status_out, int32_t* __restrict__ steps_out,
                      int32_t* __restrict__ flags, KernelCfg cfg) {
  using P = MedParams<NMAX, T_, S_>;
  constexpr int L = P::L, T = P::T, S = P::S;
  const int n = EXACT ? NMAX : n_rt;
  const int nn = n * n;

  extern __shared__ __align__(16) float smem[];
  float* stage = smem + P::OFF_STAGE;
  float* Dg = smem + P::OFF_D;  // [pos][T]
  float* Eg = smem + P::OFF_E;  // [pos][T]
  float* evs = smem + P::OFF_EV;
  float* flipv = smem + P::OFF_FLIP;
  float* scales = smem + P::OFF_SCALE;
  int* ranks = reinterpret_cast<int*>(smem + P::OFF_RANK);
  int* msw = reinterpret_cast<int*>(smem + P::OFF_MS);
  float2* rot = reinterpret_cast<float2*>(smem + P::OFF_ROT);

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int mi = tid / L;  // matrix slot in the CTA
  const int r = tid % L;   // lane in the group == owned row
  Group<L> grp;
  grp.mask = L >= 32 ? 0xffffffffu : (((1u << L) - 1u) << (lane & ~(L - 1)));
  grp.bar = 1 + mi;
  grp.red = smem + P::OFF_RED + 4 * mi;
  grp.gl = r;
  const int64_t base = (int64_t)blockIdx.x * T;
  const int count = (batch - base) < T ? (int)(batch - base) : T;
  const bool mlive = mi < count;
  float* st = stage + mi * P::SMAT;
  float* qrow = smem + P::OFF_Q + mi * NMAX;

  // ---- 1. coalesced tile load into the padded stage
  {
    const float* src = A + base * nn;
    const int total = count * nn;
    for (int g = tid; g < total; g += P::THREADS) {
      int mat = g / nn, off = g - mat * nn;
      int rr = off / n, c = off - rr * n;
      stage[mat * P::SMAT + rr * P::SROW + c] = __ldg(src + g);
    }
  }
  __syncthreads();

  // ---- 2. validate + symmetrise (core.py:286-309)
  float a[NMAX];
  int status = kStatusOk;
  {
    bool finite = true;
    float fro2 = 0.0f, asym = 0.0f;
#pragma unroll
    for (int c = 0; c < NMAX; ++c) {
      float x = 0.0f, y = 0.0f;
      if (mlive && r < n && c < n) {
        x = st[r * P::SROW + c];
        y = st[c * P::SROW + r];
      }
      finite = finite && isfinite(x);
      fro2 = fmaf(x, x, fro2);
      asym = fmaxf(asym, fabsf(x - y));
      a[c] = 0.5f * (x + y);
    }
    finite = grp.max(finite ? 0.0f : 1.0f) == 0.0f;
    fro2 = grp.sum(fro2);
    asym = grp.max(asym);
    if (!finite) status = kStatusNonFinite;
    else if (asym > cfg.sym_tol * fmaxf(1.0f, sqrtf(fro2))) status = kStatusNonSym;
    if (status != kStatusOk) {
#pragma unroll
      for (int c = 0; c < NMAX; ++c) a[c] = 0.0f;
    }
  }
  grp.sync();  // stage rows are about to be reused for reflectors

  // ---- 3. Householder tridiagonalisation (reflector i stored in st[i][*])
  static_for<0, NMAX - 2>([&](auto ic) {
    constexpr int i = decltype(ic)::value;
    if (!EXACT && i >= n - 2) return;
    const float x = r > i ? a[i] : 0.0f;
    const float scale = grp.max(fabsf(x));
    float* urow = st + i * P::SROW;
    if (scale > kZeroTail) {
      // reflector of the scaled tail xs = tail/scale (householder.py:97-118):
      // sigma = sign(xs_0) ||xs||, u0 = xs_0 + sigma, ||u||^2 = 2 sigma u0
      const float xs = x * rcp_fast(scale);
      const float ss = grp.sum(xs * xs);
      const float pivot = grp.bcast(xs, i + 1);
      const float nrm = ss * rsqrt_nr(ss);
      const float sigma = pivot >= 0.0f ? nrm : -nrm;
      const float u0 = pivot + sigma;
      const float iu = rsqrt_nr(2.0f * sigma * u0);  // sigma, u0 share a sign
      const float u = (r == i + 1 ? u0 : xs) * iu;  // xs = 0 for r <= i
      if (r < NMAX) urow[r] = u;
      grp.sync();
      // p = 2 A u, K = u^T p, q = p - K u (zero above row i)
      float p = 0.0f;
#pragma unroll
      for (int c = i + 1; c < NMAX; ++c) p = fmaf(a[c], urow[c], p);
      p *= 2.0f;
      const float kk = grp.sum(u * p);
      const float q = r >= i ? fmaf(-kk, u, p) : 0.0f;
      if (r < NMAX) qrow[r] = q;
      grp.sync();
      if (r >= i) {
#pragma unroll
        for (int c = i; c < NMAX; ++c) {
          const float uc = c > i ? urow[c] : 0.0f;
          a[c] -= fmaf(q, uc, u * qrow[c]);
        }
      }
    } else if (r < NMAX) {
      urow[r] = 0.0f;
    }
    grp.sync();
  });
  // band: D[r] = a(r, r), E[r-1] = a(r, r-1).  The row's own diagonal sits at
  // a register index equal to the lane's row -- extracted with an arithmetic
  // blend so no register array is ever indexed at run time.
  {
    float dv = 0.0f, ev = 0.0f;
#pragma unroll
    for (int c = 0; c < NMAX; ++c) {
      dv = fmaf(r == c ? 1.0f : 0.0f, a[c], dv);
      ev = fmaf(r == c + 1 ? 1.0f : 0.0f, a[c], ev);
    }
    if (r < n) Dg[r * T + mi] = dv;
    if (r >= 1 && r < n) Eg[(r - 1) * T + mi] = ev;
  }

  // ---- 4. V := P, row by row
  float v[NMAX];
  if constexpr (VECS) {
#pragma unroll
    for (int c = 0; c < NMAX; ++c) v[c] = (r == c) ? 1.0f : 0.0f;
    static_for<0, NMAX - 2>([&](auto ic) {
      constexpr int i = decltype(ic)::value;
      if (!EXACT && i >= n - 2) return;
      const float* urow = st + i * P::SROW;
      float t = 0.0f;
#pragma unroll
      for (int c = i + 1; c < NMAX; ++c) t = fmaf(v[c], urow[c], t);
      t *= -2.0f;
#pragma unroll
      for (int c = i + 1; c < NMAX; ++c) v[c] = fmaf(t, urow[c], v[c]);
    });
  }
  if (r == 0 && mi < T) ranks[mi] = status;  // handed to the band lane
  __syncthreads();

  // ---- 5/6. band QR in warp 0 (lane k = matrix k), folds in every group
  const bool band_lane = tid < T;
  int bm = n, bsteps = 0, bstatus = kStatusOk;
  bool bfin = !(tid < count);
  float bscale = 1.0f;
  if (band_lane) {
    const int k = tid;
    bstatus = ranks[k];
    float top = 0.0f;
    for (int c = 0; c < n; ++c) {
      top = fmaxf(top, fabsf(Dg[c * T + k]));
      if (c + 1 < n) top = fmaxf(top, fabsf(Eg[c * T + k]));
    }
    float inv;
    bscale = pow2_ceil(top, &inv);  // exact powers of two
    for (int c = 0; c < n; ++c) {
      Dg[c * T + k] *= inv;
      if (c + 1 < n) Eg[c * T + k] *= inv;
    }
    while (bm > 2 && fabsf(Eg[(bm - 2) * T + k]) < cfg.eps) --bm;  // initial deflation
  }

  // One explicit shifted sweep of the leading m-block (_sweep_block), run by
  // the band lane of matrix k out of shared memory.  The loads of d[i+2] and
  // e[i+2] are issued one iteration ahead so only the register recurrence
  // (dw -> rotation -> dw) is on the critical path.  Rotations past the
  // active block, up to the next multiple of kFoldBlk, are recorded as the
  // identity so the fold runs whole static blocks.
  auto sweep = [&](int k, int m, float mu, int slot) {
    float2* rs = rot + (size_t)slot * (NMAX - 1) * T + k;
    float dw = Dg[k] - mu, g = Eg[k];
    float ei = g;
    float dnx = Dg[T + k];
    float en = m > 2 ? Eg[T + k] : 0.0f;
    float c1 = 1.0f, s1 = 0.0f, c2 = 1.0f, r1 = 0.0f, u1 = 0.0f;
    for (int i = 0; i < m - 1; ++i) {
      const float dnx2 = i + 2 < m ? Dg[(i + 2) * T + k] : 0.0f;
      const float en2 = i + 2 < m - 1 ? Eg[(i + 2) * T + k] : 0.0f;
      float c, s, rr;
      givens(dw, ei, c, s, rr);
      const float dn = dnx - mu;
      const float un = c * g - s * dn;
      dw = fmaf(s, g, c * dn);
      if (i > 0) {
        Dg[(i - 1) * T + k] = (c1 * (c2 * r1) - s1 * u1) + mu;
        Eg[(i - 1) * T + k] = -s1 * rr;
      }
      if (VECS) rs[i * T] = make_float2(c, s);
      c2 = c1;
      c1 = c;
      s1 = s;
      r1 = rr;
      u1 = un;
      g = c1 * en;
      ei = en;
      dnx = dnx2;
      en = en2;
    }
    Dg[(m - 2) * T + k] = (c1 * (c2 * r1) - s1 * u1) + mu;
    Eg[(m - 2) * T + k] = -s1 * dw;
    Dg[(m - 1) * T + k] = c1 * dw + mu;
    if (VECS) {
      const int padded = min(NMAX - 1, ((m - 1 + kFoldBlk - 1) / kFoldBlk) * kFoldBlk);
      for (int i = m - 1; i < padded; ++i) rs[i * T] = make_float2(1.0f, 0.0f);
      msw[slot * T + k] = m;
    }
  };

  for (;;) {
    if (band_lane && tid < count) {
      const int k = tid;
      int slot = 0;
      while (!bfin) {
        if (bm > 2 && bsteps < cfg.max_steps) {
          if (VECS && slot + 2 > S) break;
          float lo, hi;
          wilkinson_shifts(Dg[(bm - 2) * T + k], Eg[(bm - 2) * T + k], Dg[(bm - 1) * T + k], lo,
                           hi);
          sweep(k, bm, hi, slot++);
          while (bm > 2 && fabsf(Eg[(bm - 2) * T + k]) < cfg.eps) --bm;
          if (bm > 2) {
            sweep(k, bm, lo, slot++);
            while (bm > 2 && fabsf(Eg[(bm - 2) * T + k]) < cfg.eps) --bm;
          }
          ++bsteps;
          if (!VECS) slot = 0;
        } else {
          if (VECS && slot + 1 > S) break;
          if (bm > 2) {  // budget exhausted: qr.py:604-612
            float resid = 0.0f;
            for (int c = 0; c < bm - 1; ++c) resid = fmaxf(resid, fabsf(Eg[c * T + k]));
            if (resid >= cfg.eps && bstatus == kStatusOk) bstatus = kStatusNoConv;
          }
          float lo, hi, c, s;  // 2x2 closeout (_kernels.py:401-417)
          wilkinson(Dg[k], Eg[k], Dg[T + k], lo, hi, c, s);
          Dg[k] = lo;
          Dg[T + k] = hi;
          if (VECS) {
            float2* rs = rot + (size_t)slot * (NMAX - 1) * T + k;
            rs[0] = make_float2(c, s);
            for (int i = 1; i < min(NMAX - 1, kFoldBlk); ++i) rs[i * T] = make_float2(1.0f, 0.0f);
            msw[slot * T + k] = 2;
            ++slot;
          }
          bfin = true;
        }
      }
      if (VECS)
        for (int s2 = slot; s2 < S; ++s2) msw[s2 * T + k] = 0;
    } else if (band_lane && VECS) {
      for (int s2 = 0; s2 < S; ++s2) msw[s2 * T + tid] = 0;
    }
    if (!VECS) break;
    __syncthreads();
    // fold the chunk's rotations into the owned V row, kFoldBlk positions at
    // a time (static register indices; the band lane padded each sweep with
    // identity rotations up to a block boundary)
    if (mlive) {
#pragma unroll 1
      for (int s2 = 0; s2 < S; ++s2) {
        const int m = msw[s2 * T + mi];
        if (m == 0) break;
        const float2* rs = rot + (size_t)s2 * (NMAX - 1) * T + mi;
        static_for<0, (NMAX - 1 + kFoldBlk - 1) / kFoldBlk>([&](auto bc) {
          constexpr int b0 = decltype(bc)::value * kFoldBlk;
          if (b0 < m - 1) {
#pragma unroll
            for (int p = b0; p < (b0 + kFoldBlk < NMAX - 1 ? b0 + kFoldBlk : NMAX - 1); ++p) {
              const float2 cs = rs[p * T];
              const float x = v[p], y = v[p + 1];
              v[p] = cs.x * x - cs.y * y;
              v[p + 1] = fmaf(cs.y, x, cs.x * y);
            }
          }
        });
      }
    }
    const int more = __syncthreads_or(band_lane && !bfin);
    if (!more) break;
  }
  if (band_lane) {
    scales[tid] = bscale;
    if (tid < count) {
      if (status_out) status_out[base + tid] = bstatus;
      if (steps_out) steps_out[base + tid] = bsteps;
    }
  }
  if (flags && tid < 32) {
    unsigned bits =
        __reduce_or_sync(0xffffffffu, (band_lane && tid < count && bstatus) ? (1u << bstatus) : 0u);
    if (tid == 0 && bits) atomicOr(flags, (int)bits);
  }
  __syncthreads();

  // ---- 7. sort + sign + store
  const float myscale = scales[mi];
  if (mlive && r < n) {  // rank of slot r (stable, solver.py:60-76)
    const float lr = Dg[r * T + mi];
    int rk = r;
    if (cfg.sort != 0) {
      rk = 0;
      for (int k2 = 0; k2 < n; ++k2)
        rk += (k2 != r && rank_before(Dg[k2 * T + mi], k2, lr, r, cfg.sort)) ? 1 : 0;
    }
    ranks[mi * NMAX + r] = rk;
    evs[mi * NMAX + rk] = lr * myscale;
  }
  __syncthreads();
  if constexpr (VECS) {
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
    float* dst = evecs + base * nn;
    const int total = count * nn;
    for (int g = tid; g < total; g += P::THREADS) {
      int mat = g / nn, off = g - mat * nn;
      int rr = off / n, c = off - rr * n;
      dst[g] = stage[mat * P::SMAT + rr * P::SROW + c] * flipv[mat * NMAX + c];
    }
  }
  {
    float* dstl = evals + base * n;
    for (int g = tid; g < count * n; g += P::THREADS) {
      int mat = g / n, c = g - mat * n;
      dstl[g] = evs[mat * NMAX + c];
    }
  }
}

}  // namespace bed
