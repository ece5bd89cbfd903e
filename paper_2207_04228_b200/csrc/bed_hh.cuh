// bed_hh.cuh -- H stage of the medium path (9 <= n <= 64): validation,
// Householder tridiagonalisation and P = H_0 H_1 ... H_{n-3}.
//
// A group of L lanes owns a matrix (4 lanes at n <= 16, 16 at n <= 32, two
// warps at n = 64); lane l holds rows l, l + L, ... of A in registers as
// packed column pairs (bed_f32x2.cuh), so every p = A u product and every symmetric rank-2
// update runs as FFMA2 on two columns at once, with the reflector u and the
// vector q read back from shared memory as 128-bit broadcasts.  All group
// communication is warp shuffles -- no named barriers, no shared-memory
// reductions -- so a CTA holds several independent matrices and the SM
// keeps 8-16 of them in flight.
//
// Reference (/root/reference/pkg/src/batchedeig):
//   validate + symmetrise      core.py:286-309
//   reflector                  householder.py:97-118 / _kernels.py:47-68
//   rank-2 update              householder.py:121-126 / _kernels.py:70-92
//   band                       householder.py:207-213
//   P (accumulate reflectors)  householder.py:216-231
//
// The reference scales every reflector's tail by its max |.| before the
// norm (householder.py:97-118), which guards float64 over/underflow.  Here
// the whole matrix is scaled once by the power of two 2^-ceil(log2 max|a|)
// (exact; Householder steps preserve the Frobenius norm, so every tail then
// has |x| <= n and its square sum cannot overflow), and the band is scaled
// back exactly.  Tails whose square sum underflows (below ~1e-19 of the
// matrix norm) count as already reduced -- the reference's zero-tail rule
// (householder.py:37-39) at FP32 resolution.
#pragma once

#include <type_traits>

#include "bed_f32x2.cuh"
#include "bed_split_ws.cuh"
#include "bed_tile.cuh"

#ifndef HH_GROUP_MIN
#define HH_GROUP_MIN 32
#endif

namespace bed {

// Householder steps as runtime loops over groups of four (bed_hh_kernel)
template <int NMAX>
constexpr bool kHHGroupSteps = NMAX >= HH_GROUP_MIN;

template <int NMAX>
struct HHParams {
  // n <= 32: several rows per lane (l, l + L, ...; four at n <= 16, three at
  // n = 24, two at n <= 32): every shuffle reduction serves 32 / L matrices at once and each
  // lane carries R times the FMA work between them.
  // n = 64: one row per lane over two warps (64 lanes), so a matrix needs
  // ~100 registers per thread instead of ~250 and twice the warps are in
  // flight; the two warps meet through shared memory and a named barrier.
  static constexpr int L = NMAX <= 16 ? 4 : (NMAX <= 24 ? 8 : (NMAX <= 32 ? 16 : 64));  // lanes per matrix
  static constexpr int R = (NMAX + L - 1) / L;                      // rows per lane
  static constexpr int MINB = 4;  // CTAs per SM the register cap must allow (128 registers)
  static constexpr int NP = NMAX / 2;              // column pairs per row
  static constexpr int G = NMAX == 64 ? 2 : 128 / L;  // matrices per CTA (shared stage per matrix)
  static constexpr int THREADS = G * L;
  static constexpr int SROW = NMAX + 4;            // 16-byte rows, conflict-free row reads
  static constexpr int SMAT = NMAX * SROW + NMAX + 8;  // stage / reflectors + q + scratch
  static constexpr size_t BYTES = sizeof(float) * (size_t)G * SMAT;
};

// Communication inside a matrix's lane group.  L <= 32: warp shuffles.
// L = 64 (two warps): a warp reduction, then the two partials through
// shared memory behind a named barrier (id 1 + matrix); two scratch slots
// alternate so one barrier per reduction suffices.
template <int L>
struct HHGroup {
  unsigned mask;
  int bar;
  float* red;  // 8 floats: [2 slots][2 warps] partials, [2 slots] broadcast
  int slot = 0;
  int l;
  __device__ __forceinline__ void init(int tid, int mi, float* scratch) {
    l = tid % L;
    mask = L >= 32 ? 0xffffffffu : (((1u << L) - 1u) << ((tid & 31) & ~(L - 1)));
    bar = 1 + mi;
    red = scratch;
  }
  __device__ __forceinline__ void sync() const {
    if constexpr (L <= 32) __syncwarp(mask);
    else asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(64) : "memory");
  }
  template <bool IS_MAX>
  __device__ __forceinline__ float reduce(float x) {
    constexpr int W = L <= 32 ? L : 32;
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) {
      const float y = __shfl_xor_sync(mask, x, o, W);
      x = IS_MAX ? fmaxf(x, y) : x + y;
    }
    if constexpr (L == 64) {
      float* rs = red + 2 * slot;
      if ((l & 31) == 0) rs[l >> 5] = x;
      sync();
      x = IS_MAX ? fmaxf(rs[0], rs[1]) : rs[0] + rs[1];
      slot ^= 1;
    }
    return x;
  }
  __device__ __forceinline__ float sum(float x) { return reduce<false>(x); }
  __device__ __forceinline__ float max(float x) { return reduce<true>(x); }
  // value x held by group lane src (compile-time at every call)
  __device__ __forceinline__ float bcast(float x, int src) {
    if constexpr (L <= 32) {
      return __shfl_sync(mask, x, src, L);
    } else {
      float* rb = red + 4 + slot;
      if (l == src) *rb = x;
      sync();
      const float v = *rb;
      slot ^= 1;
      return v;
    }
  }
};

// component c of a packed row (c a compile-time constant at every call)
template <int NP>
__device__ __forceinline__ float col_of(const f2 (&row)[NP], int c) {
  return (c & 1) ? f2_hi(row[c >> 1]) : f2_lo(row[c >> 1]);
}

template <int NMAX, bool EXACT, bool VECS>
__global__ void __launch_bounds__(HHParams<NMAX>::THREADS, HHParams<NMAX>::MINB)
    bed_hh_kernel(const float* __restrict__ A, int64_t bc, int n_rt, SplitWs ws, KernelCfg cfg) {
  using P = HHParams<NMAX>;
  constexpr int L = P::L, R = P::R, NP = P::NP, G = P::G, SROW = P::SROW;
  const int n = EXACT ? NMAX : n_rt;
  const int nn = n * n;
  extern __shared__ __align__(16) float smem[];
  const int tid = threadIdx.x;
  const int mi = tid / L;
  const int l = tid % L;
  const int64_t j0 = (int64_t)blockIdx.x * G;
  const int count = (bc - j0) < G ? (int)(bc - j0) : G;
  const bool mlive = mi < count;
  const int64_t j = j0 + mi;
  float* st = smem + mi * P::SMAT;  // rows of A, later reflector rows, later P rows
  float* qv = st + NMAX * SROW;     // q of the current step
  HHGroup<L> grp;
  grp.init(tid, mi, qv + NMAX);

  {  // coalesced tile load into the 16-byte-row stage (padding zero-filled)
    if (!EXACT) {
      for (int g = tid; g < G * P::SMAT; g += P::THREADS) smem[g] = 0.0f;
      __syncthreads();
    }
    if (tile_to_stage_async<NMAX, P::THREADS, SROW, P::SMAT>(A + j0 * nn, count, n, smem)) {
      cp_async_commit();
      cp_async_wait_all();
    } else {
      tile_to_stage<NMAX, P::THREADS, SROW, P::SMAT>(A + j0 * nn, count, n, smem);
    }
  }
  __syncthreads();

  // ---- validate + symmetrise (core.py:286-309); rows via 128-bit reads,
  // the transposed entries via conflict-free column reads
  f2 a[R][NP];
  int status = kStatusOk;
  float prescale = 1.0f, unscale = 1.0f;
  {
    bool finite = true;
    float amax = 0.0f, asym = 0.0f;
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const int row = l + L * rr;
      const bool ok = mlive && row < NMAX;  // NMAX = 24: lanes 24..31 hold no row
      const float4* r4 = reinterpret_cast<const float4*>(st + (ok ? row : 0) * SROW);
#pragma unroll
      for (int k4 = 0; k4 < NMAX / 4; ++k4) {
        const float4 x = ok ? r4[k4] : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        const float xs[4] = {x.x, x.y, x.z, x.w};
        float ys[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          ys[t] = ok ? st[(4 * k4 + t) * SROW + row] : 0.0f;
          finite = finite && isfinite(xs[t]);
          amax = fmaxf(amax, fabsf(xs[t]));
          asym = fmaxf(asym, fabsf(xs[t] - ys[t]));
        }
        a[rr][2 * k4] = f2_make(0.5f * (xs[0] + ys[0]), 0.5f * (xs[1] + ys[1]));
        a[rr][2 * k4 + 1] = f2_make(0.5f * (xs[2] + ys[2]), 0.5f * (xs[3] + ys[3]));
      }
    }
    finite = grp.max(finite ? 0.0f : 1.0f) == 0.0f;
    amax = grp.max(amax);
    asym = grp.max(asym);
    prescale = 1.0f;
    if (finite) unscale = pow2_ceil(amax, &prescale);
    // ||A||_F of the prescaled matrix (entries <= 1: no overflow)
    float fro2 = 0.0f;
#pragma unroll
    for (int rr = 0; rr < R; ++rr)
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const f2 y = fmul2(a[rr][k], f2_bc(prescale));
        fro2 = fmaf(f2_lo(y), f2_lo(y), fmaf(f2_hi(y), f2_hi(y), fro2));
      }
    fro2 = grp.sum(fro2);
    if (!finite) {
      status = kStatusNonFinite;
    } else if (asym > cfg.sym_tol * fmaxf(1.0f, sqrtf(fro2) * unscale)) {
      status = kStatusNonSym;
    }
    const float f = status == kStatusOk ? prescale : 0.0f;
#pragma unroll
    for (int rr = 0; rr < R; ++rr)
#pragma unroll
      for (int k = 0; k < NP; ++k) a[rr][k] = fmul2(a[rr][k], f2_bc(f));
  }
  grp.sync();  // stage rows are about to be reused for reflectors

  // ---- Householder reduction; reflector i stored in st row i.  The step
  // loop is expanded by template recursion so every column index is a
  // compile-time constant (NVVM's unroller gives up on the n = 64 body).
  // One step for reflector i: K0 / K1 are the (compile-time) first column
  // pairs of p = A u and of the update -- at most the step's own -- and the
  // pivot column is picked among NC compile-time candidates from C0.
  auto hh_step = [&](const int i, auto k0c, auto k1c, auto c0c, auto ncc) {
    constexpr int K0 = decltype(k0c)::value, K1 = decltype(k1c)::value;
    constexpr int C0 = decltype(c0c)::value, NC = decltype(ncc)::value;
    // row groups rr < RR0 hold only rows < C0 <= i: u, p, q vanish there and
    // the update leaves them unchanged, so their FMA work is skipped
    constexpr int RR0 = C0 / L;
    // n = 64 (one row per lane, two warps): warp 0's rows drop out from i = 32
    const bool wdead = L == 64 && C0 >= 32 && l < 32;
    float x[R];
    float ss = 0.0f;
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      float c = col_of<NP>(a[rr], C0);
#pragma unroll
      for (int q = 1; q < NC; ++q)
        if (C0 + q < NMAX) c = (i == C0 + q) ? col_of<NP>(a[rr], C0 + q) : c;
      x[rr] = (l + L * rr > i) ? c : 0.0f;
      ss = fmaf(x[rr], x[rr], ss);
    }
    ss = grp.sum(ss);
    float* urow = st + i * SROW;
    float u[R];
    if (ss > 0x1p-120f) {
      // sigma = sign(x_0) ||x||, u0 = x_0 + sigma, ||u||^2 = 2 sigma u0
      // (householder.py:97-118; the tail is already at unit scale)
      const int pr = (i + 1) / L, pl = (i + 1) % L;
      float xp = x[0];
#pragma unroll
      for (int rr = 1; rr < R; ++rr) xp = (rr == pr) ? x[rr] : xp;
      const float pivot = grp.bcast(xp, pl);
      const float nrm = ss * rsqrt_nr(ss);
      const float sigma = pivot >= 0.0f ? nrm : -nrm;
      const float u0 = pivot + sigma;
      const float iu = rsqrt_nr(2.0f * sigma * u0);  // sigma, u0 share a sign
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        u[rr] = (l + L * rr == i + 1 ? u0 : x[rr]) * iu;  // x = 0 for rows <= i
        if (l + L * rr < NMAX) urow[l + L * rr] = u[rr];
      }
      grp.sync();
      // p = 2 A u (two accumulators per row for ILP), K = u^T p, q = p - K u
      constexpr int k0 = K0;  // 16-byte aligned start; u = 0 below i+1
      float p[R];
      float kk = 0.0f;
      {
        f2 acc0[R], acc1[R];
#pragma unroll
        for (int rr = 0; rr < R; ++rr) acc0[rr] = acc1[rr] = f2_bc(0.0f);
        if (!wdead) {
#pragma unroll
          for (int k = k0; k < NP; k += 2) {
            const float4 u4 = *reinterpret_cast<const float4*>(urow + 2 * k);
#pragma unroll
            for (int rr = RR0; rr < R; ++rr) {
              acc0[rr] = ffma2(a[rr][k], f2_make(u4.x, u4.y), acc0[rr]);
              if (k + 1 < NP) acc1[rr] = ffma2(a[rr][k + 1], f2_make(u4.z, u4.w), acc1[rr]);
            }
          }
        }
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          if (rr < RR0 || wdead) {
            p[rr] = 0.0f;
            continue;
          }
          const f2 acc = fadd2(acc0[rr], acc1[rr]);
          p[rr] = 2.0f * (f2_lo(acc) + f2_hi(acc));
          kk = fmaf(u[rr], p[rr], kk);
        }
      }
      kk = grp.sum(kk);
      float q[R];
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        q[rr] = (rr >= RR0 && !wdead && l + L * rr >= i) ? fmaf(-kk, u[rr], p[rr]) : 0.0f;
        if (l + L * rr < NMAX) qv[l + L * rr] = q[rr];
      }
      grp.sync();
      // A <- A - q u^T - u q^T on columns >= i (u, q vanish on the rest)
      constexpr int k1 = K1;
#pragma unroll
      for (int k = k1; k < NP && !wdead; k += 2) {
        const float4 u4 = *reinterpret_cast<const float4*>(urow + 2 * k);
        const float4 q4 = *reinterpret_cast<const float4*>(qv + 2 * k);
#pragma unroll
        for (int rr = RR0; rr < R; ++rr) {
          a[rr][k] = ffma2(f2_bc(-u[rr]), f2_make(q4.x, q4.y),
                           ffma2(f2_bc(-q[rr]), f2_make(u4.x, u4.y), a[rr][k]));
          if (k + 1 < NP)
            a[rr][k + 1] = ffma2(f2_bc(-u[rr]), f2_make(q4.z, q4.w),
                                 ffma2(f2_bc(-q[rr]), f2_make(u4.z, u4.w), a[rr][k + 1]));
        }
      }
    } else {
#pragma unroll
      for (int rr = 0; rr < R; ++rr)
        if (l + L * rr < NMAX) urow[l + L * rr] = 0.0f;
    }
    grp.sync();
  };
  if constexpr (kHHGroupSteps<NMAX>) {
    // four steps per group in a runtime loop, their columns picked by selects:
    // ~4x less code than one expanded body per step (the unrolled form leaves
    // the SM 11-20 % of cycles without instructions at n >= 32)
    static_for<0, (NMAX - 2 + 3) / 4>([&](auto gc) {
      constexpr int g = decltype(gc)::value;
#pragma unroll 1
      for (int t = 0; t < 4; ++t) {
        const int i = 4 * g + t;
        if (i >= NMAX - 2 || (!EXACT && i >= n - 2)) break;
        hh_step(i, std::integral_constant<int, 2 * g>{}, std::integral_constant<int, 2 * g>{},
                std::integral_constant<int, 4 * g>{}, std::integral_constant<int, 4>{});
      }
    });
  } else {
    static_for<0, NMAX - 2>([&](auto ic) {
      constexpr int i = decltype(ic)::value;
      if (!EXACT && i >= n - 2) return;
      hh_step(i, std::integral_constant<int, ((i + 1) / 2) & ~1>{}, std::integral_constant<int, (i / 2) & ~1>{},
              std::integral_constant<int, i>{}, std::integral_constant<int, 1>{});
    });
  }

  // ---- band: D[r] = a(r, r), E[r-1] = a(r, r-1), picked with compares on
  // the lane index so no register array is indexed at run time
  if (mlive) {
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const int row = l + L * rr;
      float dv = 0.0f, ev = 0.0f;
#pragma unroll
      for (int c = 0; c < NMAX; ++c) {
        const float x = col_of<NP>(a[rr], c);
        dv = row == c ? x : dv;
        ev = row == c + 1 ? x : ev;
      }
      if (row < n) ws.D[(int64_t)row * ws.Bc + j] = dv * unscale;
      if (row >= 1 && row < n) ws.E[(int64_t)(row - 1) * ws.Bc + j] = ev * unscale;
    }
    if (l == 0) ws.vstat[j] = status;
  }

  if constexpr (VECS) {
    // ---- P = H_0 H_1 ... H_{n-3} (householder.py:216-231), accumulated as
    // W = P^T = H_{n-3} ... H_0 in reverse order, rows in registers:
    // W <- W (I - 2 u u^T).  With the later reflectors applied first, W is the
    // identity outside rows / columns > i when H_i arrives, so only those rows
    // (row groups rr >= RR0) and columns change -- ~2/3 of the forward
    // accumulation's FMA work; W^T is written to the stage below.  At one row
    // per lane (n = 64) warp 0's rows drop out from i = 31.
    constexpr bool REV = true;
    f2 v[R][NP];
#pragma unroll
    for (int rr = 0; rr < R; ++rr)
#pragma unroll
      for (int k = 0; k < NP; ++k)
        v[rr][k] = f2_make(l + L * rr == 2 * k ? 1.0f : 0.0f, l + L * rr == 2 * k + 1 ? 1.0f : 0.0f);
    auto p_step = [&](const int i, auto k0c, auto rr0c, bool wdead) {
      if (wdead) return;
      const float* urow = st + i * SROW;
      constexpr int k0 = decltype(k0c)::value;
      constexpr int RR0 = decltype(rr0c)::value;  // row groups below: rows <= i, unchanged
      f2 acc0[R], acc1[R];
#pragma unroll
      for (int rr = RR0; rr < R; ++rr) acc0[rr] = acc1[rr] = f2_bc(0.0f);
#pragma unroll
      for (int k = k0; k < NP; k += 2) {
        const float4 u4 = *reinterpret_cast<const float4*>(urow + 2 * k);
#pragma unroll
        for (int rr = RR0; rr < R; ++rr) {
          acc0[rr] = ffma2(v[rr][k], f2_make(u4.x, u4.y), acc0[rr]);
          if (k + 1 < NP) acc1[rr] = ffma2(v[rr][k + 1], f2_make(u4.z, u4.w), acc1[rr]);
        }
      }
      float t[R];
#pragma unroll
      for (int rr = RR0; rr < R; ++rr) {
        const f2 acc = fadd2(acc0[rr], acc1[rr]);
        t[rr] = -2.0f * (f2_lo(acc) + f2_hi(acc));
      }
#pragma unroll
      for (int k = k0; k < NP; k += 2) {
        const float4 u4 = *reinterpret_cast<const float4*>(urow + 2 * k);
#pragma unroll
        for (int rr = RR0; rr < R; ++rr) {
          v[rr][k] = ffma2(f2_bc(t[rr]), f2_make(u4.x, u4.y), v[rr][k]);
          if (k + 1 < NP) v[rr][k + 1] = ffma2(f2_bc(t[rr]), f2_make(u4.z, u4.w), v[rr][k + 1]);
        }
      }
    };
    if constexpr (kHHGroupSteps<NMAX>) {
      constexpr int NG = (NMAX - 2 + 3) / 4;
      static_for<0, NG>([&](auto gc) {
        constexpr int g = REV ? NG - 1 - decltype(gc)::value : decltype(gc)::value;
#pragma unroll 1
        for (int tt = 0; tt < 4; ++tt) {
          const int i = 4 * g + (REV ? 3 - tt : tt);
          if (i >= NMAX - 2 || (!EXACT && i >= n - 2)) continue;
          p_step(i, std::integral_constant<int, 2 * g>{}, std::integral_constant<int, REV ? (4 * g + 1) / L : 0>{},
                 L == 64 && 4 * g >= 31 && l < 32);
        }
      });
    } else {
      static_for<0, NMAX - 2>([&](auto ic) {
        constexpr int i = REV ? NMAX - 3 - decltype(ic)::value : decltype(ic)::value;
        if (!EXACT && i >= n - 2) return;
        p_step(i, std::integral_constant<int, ((i + 1) / 2) & ~1>{}, std::integral_constant<int, REV ? (i + 1) / L : 0>{},
               L == 64 && i >= 31 && l < 32);
      });
    }
    grp.sync();  // every lane is done reading reflectors
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      if (l + L * rr >= NMAX) continue;
      if constexpr (REV) {  // P = W^T: row r of W is column r of P
        float* col = st + l + L * rr;
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          col[(2 * k) * SROW] = f2_lo(v[rr][k]);
          col[(2 * k + 1) * SROW] = f2_hi(v[rr][k]);
        }
      } else {
        float4* r4 = reinterpret_cast<float4*>(st + (l + L * rr) * SROW);
#pragma unroll
        for (int k4 = 0; k4 < NMAX / 4; ++k4)
          r4[k4] = make_float4(f2_lo(v[rr][2 * k4]), f2_hi(v[rr][2 * k4]), f2_lo(v[rr][2 * k4 + 1]),
                               f2_hi(v[rr][2 * k4 + 1]));
      }
    }
    __syncthreads();
    stage_to_tile<NMAX, P::THREADS, SROW, P::SMAT>(smem, count, n, ws.P + j0 * nn);
  }
}

}  // namespace bed
