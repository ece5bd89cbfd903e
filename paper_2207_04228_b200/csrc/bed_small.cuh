// bed_small.cuh -- forward ED for n <= 8: one thread owns one matrix.
//
// Layout: a CTA of 128 threads solves 128 consecutive matrices.  The tile
// (128 * n^2 floats, contiguous in HBM) is staged through shared memory
// with coalesced 128-bit loads into an odd per-matrix stride, so every
// thread's private reads are bank-conflict free; outputs leave the same
// way.  Everything else -- the symmetric lower triangle, the band, V and
// the loop state -- lives in registers; every array index is a
// compile-time constant (loops fully unrolled on N, the per-matrix active
// size m is a runtime predicate), so nothing spills to local memory.
//
// The kernel is limited by instruction issue (n = 4: ~90 % issue-active,
// FMA pipe ~50 %), so V is held as packed row pairs (bed_f32x2.cuh): a
// Givens fold on two columns costs 2 FFMA2 + 2 FMUL2 per two rows instead
// of 8 scalar ops, and the band recurrence computes its (u, dw) pair with
// one FMUL2 + one FFMA2.
//
// The QR loop runs warp-synchronously: all 32 lanes stay in the loop until
// every lane's matrix has deflated; finished lanes run exact no-op sweeps.
// n <= 4 sweeps all positions unmasked (locked couplings are exact zeros,
// small_sweep_full); 5 <= n <= 8 masks positions past each lane's block and
// skips positions no lane needs by a warp vote.  That keeps the code
// straight-line (no per-lane control flow the compiler could fold into
// dynamically indexed, local-memory register arrays).
//
// Per-matrix pipeline (reference /root/reference/pkg/src/batchedeig):
//   validate + symmetrise        core.py:286-309
//   Householder reduction        _kernels.py:36-92, with V <- V H_i folded
//                                in as each reflector is made (= P of
//                                householder.py:216-231, V starts as P so
//                                V = P Q of solver.py:93 needs no GEMM)
//   power-of-two equilibration   qr.py:522-534, :596-598, :624
//   double-shift QR loop         _kernels.py:321-398 with the deflation
//                                gate applied per matrix (the reference's
//                                own per-matrix bookkeeping :381-388)
//   fused sweep                  _kernels.py:221-300
//   2x2 closeout                 _kernels.py:401-417
//   sort + sign                  solver.py:60-76
#pragma once

#include "bed_common.cuh"
#include "bed_scatter_regs.cuh"
#include "bed_f32x2.cuh"

namespace bed {

constexpr int kSmallThreads = 128;

// largest n whose QR loop sweeps every position unmasked (small_sweep_full)
constexpr int kUnmaskedMaxN = 4;  // n = 8 measured equal either way

template <int N>
struct SmallLayout {
  static constexpr int NN = N * N;
  static constexpr int NP = (N + 1) / 2;                 // packed row pairs of V
  static constexpr int STRIDE = (NN % 2) ? NN : NN + 1;  // odd => conflict free
  static constexpr int LSTRIDE = (N % 2) ? N : N + 1;
};

// A(r, c) of the symmetric lower-triangle store.
template <int N>
BED_HD float sym_at(const float (&a)[N][N], int r, int c) {
  return c <= r ? a[r][c] : a[c][r];
}

// V(r, c) of the packed row-pair store.
template <int NP, int N>
__device__ __forceinline__ float v_at(const f2 (&v)[NP][N], int r, int c) {
  return (r & 1) ? f2_hi(v[r >> 1][c]) : f2_lo(v[r >> 1][c]);
}

// V <- V R on columns (p, p+1), all rows; an identity rotation (c = 1,
// s = 0) leaves V bit-identical.
template <int N, bool VECS>
__device__ __forceinline__ void small_fold(f2 (&v)[SmallLayout<N>::NP][N], int p, float c,
                                           float s, float ns) {
  if constexpr (VECS) {
#pragma unroll
    for (int rp = 0; rp < SmallLayout<N>::NP; ++rp) rot2(v[rp][p], v[rp][p + 1], c, s, ns);
  }
}

__device__ __forceinline__ bool warp_any(bool p) { return __any_sync(0xffffffffu, p); }

// Givens rotation of the fused sweep with the identity rule folded into the
// inputs: a dead target (|e| < 2^-60, or a position past the active block,
// passed as e = 0) runs on (1, 0), giving c = 1, s = 0 exactly; r is then
// the unrotated dw (_kernels.py:247, :256-258).
//
// For n <= 8 the reciprocal square root is the raw MUFU value (relative
// error < 2^-22): a rotation is then orthogonal up to a scale 1 + O(2^-22),
// and the few dozen rotations a small solve applies keep V orthogonal and
// the eigenvalues within a few 1e-7 of the spectral radius (the parity
// gates are 1e-5).  The medium kernels, which fold thousands of rotations,
// refine it (rsqrt_nr).
template <bool REFINE>
__device__ __forceinline__ void small_givens(float dw, float e, float& c, float& s, float& ns,
                                             float& r) {
  const bool live = fabsf(e) >= 0x1p-60f;
  const float x = live ? dw : 1.0f;
  const float y = live ? e : 0.0f;
  const float h2 = fmaf(x, x, y * y);
  const float ih = REFINE ? rsqrt_nr(h2) : rsqrt_approx(h2);
  c = x * ih;
  s = -y * ih;
  ns = -s;
  const float rr = h2 * ih;
  r = live ? rr : dw;
}

// One explicit shifted QR sweep of the leading m-block, fused exactly like
// _sweep_block (rotation i-1 retires once rotation i exists), written as
// predicated straight-line code: rotations at positions >= m-1 degenerate to
// the identity and writes past the active block are masked with selects.
// m = 0 makes the whole sweep a no-op (used for lanes whose matrix has
// finished).  Positions no lane of the warp needs are skipped by a vote
// (n > 4; for n <= 4 the branch would cost register moves of the packed V
// at every join, see small_sweep_full).
template <int N, bool VECS>
__device__ __forceinline__ void small_sweep(float (&d)[N], float (&e)[N],
                                            f2 (&v)[SmallLayout<N>::NP][N], int m, float mu) {
  float dw = d[0] - mu, g = e[0];
  float c1 = 1.0f, s1 = 0.0f, ns1 = 0.0f, c2 = 1.0f, r1 = 0.0f, u1 = 0.0f;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    if (i >= 2 && !warp_any(i <= m - 1)) break;
    const bool act = i < m - 1;
    const float ei = (i < N - 1 && act) ? e[i] : 0.0f;
    float c, s, ns, r;
    small_givens<false>(dw, ei, c, s, ns, r);
    const float dn = (i + 1 < N ? d[i + 1] : 0.0f) - mu;
    // (u, dw') = (c g - s dn, s g + c dn)
    const f2 ud = ffma2(f2_make(-s, c), f2_bc(dn), fmul2(f2_make(c, s), f2_bc(g)));
    if (i > 0) {
      const bool wr = i <= m - 1;  // rotation i-1 was a real one
      const float dret = (c1 * (c2 * r1) - s1 * u1) + mu;
      d[i - 1] = wr ? dret : d[i - 1];
      e[i - 1] = wr ? ns1 * r : e[i - 1];
      small_fold<N, VECS>(v, i - 1, c1, s1, ns1);  // identity once past the block
    }
    d[i] = (i == m - 1) ? c1 * dw + mu : d[i];
    c2 = c1;
    c1 = c;
    s1 = s;
    ns1 = ns;
    r1 = r;
    u1 = f2_lo(ud);
    dw = f2_hi(ud);
    if (i + 1 < N - 1) g = c1 * e[i + 1];
  }
}

// Trailing deflation: while m > 2 and |e[m-2]| < eps, m -= 1 -- unrolled
// from the top so no array is indexed by m, in integer arithmetic so it
// compiles without branches.  Idempotent (a finished lane's m stays put).
template <int N>
__device__ __forceinline__ int small_deflate(const float (&e)[N], int m, float eps) {
#pragma unroll
  for (int j = N - 2; j >= 1; --j) m -= (int)(m == j + 2) & (int)(fabsf(e[j]) < eps);
  return m;
}

// n <= 4: a sweep over all N positions with no per-position masks.  A
// lane's deflated couplings are exact zeros (small_deflate_zero), so its
// rotations there are exact identities and the reduced block is swept as in
// the masked form (bitwise: the retire formula with an identity rotation
// reduces to the tail formula); positions past the block only see the
// shift added and removed again, a rounding-level change of an already
// locked diagonal entry.  A lane that is off (finished, or budget spent)
// sweeps with mu = 0 and its leading coupling masked, which is an exact
// no-op, so results never depend on the warp's other lanes.
template <int N, bool VECS>
__device__ __forceinline__ void small_sweep_full(float (&d)[N], float (&e)[N],
                                                 f2 (&v)[SmallLayout<N>::NP][N], bool on,
                                                 float mu) {
  float dw = d[0] - mu, g = on ? e[0] : 0.0f;
  float c1 = 1.0f, s1 = 0.0f, ns1 = 0.0f, c2 = 1.0f, r1 = 0.0f, u1 = 0.0f;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const float ei = i == 0 ? g : (i < N - 1 ? e[i] : 0.0f);
    float c, s, ns, r;
    small_givens<false>(dw, ei, c, s, ns, r);
    const float dn = (i + 1 < N ? d[i + 1] : 0.0f) - mu;
    // (u, dw') = (c g - s dn, s g + c dn)
    const f2 ud = ffma2(f2_make(-s, c), f2_bc(dn), fmul2(f2_make(c, s), f2_bc(g)));
    if (i > 0) {
      d[i - 1] = (c1 * (c2 * r1) - s1 * u1) + mu;
      e[i - 1] = (i == 1 && !on) ? e[0] : ns1 * r;
      small_fold<N, VECS>(v, i - 1, c1, s1, ns1);
    }
    if (i == N - 1) d[i] = c1 * dw + mu;  // tail of the last position
    c2 = c1;
    c1 = c;
    s1 = s;
    ns1 = ns;
    r1 = r;
    u1 = f2_lo(ud);
    dw = f2_hi(ud);
    if (i + 1 < N - 1) g = c1 * e[i + 1];
  }
}

// Deflation that also zeroes the couplings it locks (see small_sweep_full).
template <int N>
__device__ __forceinline__ int small_deflate_zero(float (&e)[N], int m, float eps) {
#pragma unroll
  for (int j = N - 2; j >= 1; --j) {
    const bool dec = (m == j + 2) && (fabsf(e[j]) < eps);
    m -= dec ? 1 : 0;
    e[j] = dec ? 0.0f : e[j];
  }
  return m;
}

// POW: the spectral power V diag(max(lambda, floor)^p) V^T (matrix_power,
// solver.py:115-143) is formed from V in registers and written to `evecs` in
// place of V -- the fused epilogue of SURVEY.md 8(f) row 1; V never leaves
// the thread.
// SCAT: the thread forms its matrix from X (n channels x m samples) as the
// scatter (X - mu)(X - mu)^T + eps I (zca_whiten, solver.py:161-166; the
// covariance producer of SURVEY.md 8(f) row 3) in registers, in one pass
// shifted by each channel's first sample (as bed_scatter.cu), instead of
// reading A: the covariance never reaches memory.
// CTAs per SM the register allocation must allow: 0 = no constraint (ptxas's
// own choice -- an explicit 1 is NOT the same and gave the n = 4 kernel 80
// registers instead of 54); n = 7 at five CTAs (102 registers, a 48-byte spill
// outside the loop): 1 M matrices 0.298 -> 0.284 ms.  n = 5, 6 and 8 measured
// best unconstrained (n = 8 capped at five spills inside the QR loop).
template <int N>
constexpr int small_min_blocks() { return N == 7 ? 5 : 0; }

template <int N, bool VECS, bool POW = false, bool SCAT = false>
__global__ void __launch_bounds__(kSmallThreads, small_min_blocks<N>())
    bed_small_kernel(const float* __restrict__ A, int64_t batch, float* __restrict__ evals,
                     float* __restrict__ evecs, int32_t* __restrict__ status_out,
                     int32_t* __restrict__ steps_out, int32_t* __restrict__ flags, KernelCfg cfg,
                     DiagOut dg, PowSpec pw = PowSpec{}, ScatSpec sc = ScatSpec{}) {
  static_assert(!POW || VECS, "the power is formed from the eigenvectors");
  using Lay = SmallLayout<N>;
  constexpr int NN = Lay::NN;
  constexpr int NP = Lay::NP;
  __shared__ float tile[kSmallThreads * Lay::STRIDE];
  __shared__ float ltile[kSmallThreads * Lay::LSTRIDE];

  const int64_t base = (int64_t)blockIdx.x * kSmallThreads;
  const int count = (batch - base) < kSmallThreads ? (int)(batch - base) : kSmallThreads;
  const int tid = threadIdx.x;
  const bool live = tid < count;

  // ---- load.  n^2 % 4 == 0 with a 16-byte aligned batch: each thread reads
  // its own matrix with 128-bit loads (the warp's n^2/4 loads cover one
  // contiguous span; L1 merges the sectors).  Otherwise a coalesced tile
  // load into the odd-stride shared stage.  The branch is CTA-uniform.
  float a[N][N];
  int status = kStatusOk;
  {
    float x[N][N];
    const bool direct = (NN % 4 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
    if constexpr (SCAT) {
      scatter_regs<N>(sc.X + (base + (live ? tid : 0)) * (int64_t)N * sc.m, sc.m, sc.eps, live,
                      (reinterpret_cast<uintptr_t>(sc.X) & 15) == 0, x);
    } else if (direct) {
      if constexpr (NN % 4 == 0) {
        const float4* p = reinterpret_cast<const float4*>(A + (base + (live ? tid : 0)) * NN);
#pragma unroll
        for (int q = 0; q < NN / 4; ++q) {
          float4 t = __ldg(p + q);
          if (!live) t = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
          x[(4 * q) / N][(4 * q) % N] = t.x;
          x[(4 * q + 1) / N][(4 * q + 1) % N] = t.y;
          x[(4 * q + 2) / N][(4 * q + 2) % N] = t.z;
          x[(4 * q + 3) / N][(4 * q + 3) % N] = t.w;
        }
      }
    } else {
      const float* src = A + base * NN;
      for (int g = tid; g < count * NN; g += kSmallThreads)
        tile[(g / NN) * Lay::STRIDE + (g % NN)] = __ldg(src + g);
      __syncthreads();
      const float* my = tile + tid * Lay::STRIDE;
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int c = 0; c < N; ++c) x[r][c] = live ? my[r * N + c] : 0.0f;
    }

    // ---- validate + symmetrise (core.py:286-309).  A NaN or Inf entry makes
    // the square sum non-finite, so the per-entry scan runs only then (or
    // when a finite entry's square overflows, where it finds nothing)
    float fro2 = 0.0f, asym = 0.0f;
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int c = 0; c < N; ++c) fro2 = fmaf(x[r][c], x[r][c], fro2);
    bool finite = isfinite(fro2);
    if (!finite) {
      finite = true;
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int c = 0; c < N; ++c) finite = finite && isfinite(x[r][c]);
    }
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int c = 0; c < r; ++c) asym = fmaxf(asym, fabsf(x[r][c] - x[c][r]));
    float limit = cfg.sym_tol * fmaxf(1.0f, sqrtf(fro2));
    if (!finite) status = kStatusNonFinite;
    else if (asym > limit) status = kStatusNonSym;
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int c = 0; c <= r; ++c)
        a[r][c] = status == kStatusOk ? 0.5f * (x[r][c] + x[c][r]) : 0.0f;
  }

  // ---- Householder tridiagonalisation with V <- V H_i accumulated in place
  // (V as packed row pairs; the odd-N padding row stays zero)
  f2 v[NP][N];
#pragma unroll
  for (int rp = 0; rp < NP; ++rp)
#pragma unroll
    for (int c = 0; c < N; ++c)
      v[rp][c] = f2_make((VECS && 2 * rp == c) ? 1.0f : 0.0f, (VECS && 2 * rp + 1 == c) ? 1.0f : 0.0f);

#pragma unroll
  for (int i = 0; i < N - 2; ++i) {
    float scale = 0.0f;
#pragma unroll
    for (int r = i + 1; r < N; ++r) scale = fmaxf(scale, fabsf(a[r][i]));
    if (scale > kZeroTail) {
      // reflector of the scaled tail xs = tail/scale (householder.py:97-118):
      // sigma_s = sign(xs_0) ||xs||, u0 = xs_0 + sigma_s, ||u||^2 = 2 sigma_s u0
      const float is = rcp_fast(scale);
      float u[N];
      float sumsq = 0.0f;
#pragma unroll
      for (int r = 0; r < N; ++r) {
        u[r] = r <= i ? 0.0f : a[r][i] * is;
        sumsq = fmaf(u[r], u[r], sumsq);
      }
      const float pivot = u[i + 1];
      const float nrm = sumsq * rsqrt_nr(sumsq);
      const float sigma = pivot >= 0.0f ? nrm : -nrm;
      const float u0 = pivot + sigma;
      const float iu = rsqrt_nr(2.0f * sigma * u0);  // sigma, u0 share a sign
      u[i + 1] = u0;
#pragma unroll
      for (int r = i + 1; r < N; ++r) u[r] *= iu;
      // p = 2 A u on rows i.., K = u^T p, q = p - K u  (u_i = 0)
      float q[N];
      float kk = 0.0f;
#pragma unroll
      for (int r = i; r < N; ++r) {
        float acc = 0.0f;
#pragma unroll
        for (int c = i + 1; c < N; ++c) acc = fmaf(sym_at<N>(a, r, c), u[c], acc);
        q[r] = 2.0f * acc;
        if (r > i) kk = fmaf(u[r], q[r], kk);
      }
#pragma unroll
      for (int r = i + 1; r < N; ++r) q[r] = fmaf(-kk, u[r], q[r]);
      // A <- A - q u^T - u q^T on the trailing lower triangle (two FMAs)
#pragma unroll
      for (int r = i; r < N; ++r)
#pragma unroll
        for (int c = i; c <= r; ++c) a[r][c] = fmaf(-q[r], u[c], fmaf(-u[r], q[c], a[r][c]));
      if constexpr (VECS) {
        if (i == 0) {
          // V = I - 2 u u^T directly (u_0 = 0: row and column 0 stay e_0)
#pragma unroll
          for (int rp = 0; rp < NP; ++rp)
#pragma unroll
            for (int c = 1; c < N; ++c) {
              const int r0 = 2 * rp, r1 = 2 * rp + 1;
              const float w = -2.0f * u[c];
              const float lo = r0 >= 1 ? fmaf(w, u[r0], r0 == c ? 1.0f : 0.0f) : 0.0f;
              const float hi = (r1 >= 1 && r1 < N) ? fmaf(w, u[r1], r1 == c ? 1.0f : 0.0f) : 0.0f;
              v[rp][c] = f2_make(lo, hi);
            }
        } else {
          // V <- V (I - 2 u u^T): columns before i+1 are untouched
#pragma unroll
          for (int rp = 0; rp < NP; ++rp) {
            f2 t = fmul2(v[rp][i + 1], f2_bc(u[i + 1]));
#pragma unroll
            for (int c = i + 2; c < N; ++c) t = ffma2(v[rp][c], f2_bc(u[c]), t);
            t = fmul2(t, f2_bc(-2.0f));
#pragma unroll
            for (int c = i + 1; c < N; ++c) v[rp][c] = ffma2(t, f2_bc(u[c]), v[rp][c]);
          }
        }
      }
    }
  }

  // ---- band, equilibration
  float d[N], e[N];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    d[j] = a[j][j];
    e[j] = j + 1 < N ? a[j + 1][j] : 0.0f;
  }
  float top = 0.0f;
#pragma unroll
  for (int j = 0; j < N; ++j) top = fmaxf(top, fmaxf(fabsf(d[j]), fabsf(e[j])));
  float iscale;
  const float scale = pow2_ceil(top, &iscale);  // exact powers of two
#pragma unroll
  for (int j = 0; j < N; ++j) {
    d[j] *= iscale;
    e[j] *= iscale;
  }

  // ---- double-shift QR with per-matrix deflation, warp-synchronous
  int steps = 0, rot = 0, srs = 0, mfin = N < 2 ? 2 : N;
  float res_out = 0.0f;
  if constexpr (N >= 3) {
    if constexpr (N <= kUnmaskedMaxN) {
      int m = small_deflate_zero<N>(e, N, cfg.eps);
      bool run = m > 2;
      while (warp_any(run)) {
        if (warp_any(run && steps >= cfg.max_steps)) {  // budget exhausted: qr.py:604-612
          if (run && steps >= cfg.max_steps) {
            float resid = 0.0f;
#pragma unroll
            for (int j = 0; j < N - 1; ++j) resid = fmaxf(resid, j < m - 1 ? fabsf(e[j]) : 0.0f);
            res_out = resid;
            if (resid >= cfg.eps && status == kStatusOk) status = kStatusNoConv;
            run = false;  // lock the diagonal; the leading 2x2 still closes below
#pragma unroll
            for (int j = 1; j < N - 1; ++j) e[j] = 0.0f;  // off lanes sweep as exact no-ops
          }
        }
        float ta = 0.0f, tb = 0.0f, td = 0.0f;
#pragma unroll
        for (int j = 1; j < N - 1; ++j) {
          const float w = (j == m - 2) ? 1.0f : 0.0f;
          ta = fmaf(w, d[j], ta);
          tb = fmaf(w, e[j], tb);
          td = fmaf(w, d[j + 1], td);
        }
        float lo, hi;
        wilkinson_shifts(ta, tb, td, lo, hi);
        small_sweep_full<N, VECS>(d, e, v, run, run ? hi : 0.0f);
        srs += run ? N - m : 0;
        rot += run ? m - 1 : 0;
        m = small_deflate_zero<N>(e, m, cfg.eps);
        const bool on2 = run && m > 2;
        small_sweep_full<N, VECS>(d, e, v, on2, on2 ? lo : 0.0f);
        rot += on2 ? m - 1 : 0;
        m = small_deflate_zero<N>(e, m, cfg.eps);
        steps += run ? 1 : 0;
        run = run && m > 2;
      }
      mfin = m;
    } else {
      int m = small_deflate<N>(e, N, cfg.eps);
      bool run = m > 2;
      while (warp_any(run)) {
        if (warp_any(run && steps >= cfg.max_steps)) {  // budget exhausted: qr.py:604-612
          if (run && steps >= cfg.max_steps) {
            float resid = 0.0f;
#pragma unroll
            for (int j = 0; j < N - 1; ++j) resid = fmaxf(resid, j < m - 1 ? fabsf(e[j]) : 0.0f);
            res_out = resid;
            if (resid >= cfg.eps && status == kStatusOk) status = kStatusNoConv;
            run = false;  // lock the diagonal; the leading 2x2 still closes below
          }
        }
        // trailing 2x2 of the active block; an arithmetic blend, not a
        // select chain, so the compiler cannot fold it into a dynamically
        // indexed (local-memory) load of d[m-2]
        float ta = 0.0f, tb = 0.0f, td = 0.0f;
#pragma unroll
        for (int j = 1; j < N - 1; ++j) {
          const float w = (j == m - 2) ? 1.0f : 0.0f;
          ta = fmaf(w, d[j], ta);
          tb = fmaf(w, e[j], tb);
          td = fmaf(w, d[j + 1], td);
        }
        float lo, hi;
        wilkinson_shifts(ta, tb, td, lo, hi);
        // finished lanes sweep nothing (m = 0); their couplings do not
        // move, so the unconditional deflations leave their m unchanged
        if constexpr (N >= 8) {
          // both sweeps through one copy of the sweep code (a runtime loop of
          // two): n = 8 spent ~10 % of cycles waiting for instructions with two
          // expanded copies (1 M: 0.322 -> 0.312 ms); at n = 5..7 the loop
          // costs more than it saves
          srs += run ? N - m : 0;
#pragma unroll 1
          for (int h = 0; h < 2; ++h) {
            const int mm = (run && (h == 0 || m > 2)) ? m : 0;
            small_sweep<N, VECS>(d, e, v, mm, h ? lo : hi);
            rot += mm > 2 ? mm - 1 : 0;
            m = small_deflate<N>(e, m, cfg.eps);
          }
        } else {
          small_sweep<N, VECS>(d, e, v, run ? m : 0, hi);
          srs += run ? N - m : 0;
          rot += run ? m - 1 : 0;
          m = small_deflate<N>(e, m, cfg.eps);
          small_sweep<N, VECS>(d, e, v, (run && m > 2) ? m : 0, lo);
          rot += (run && m > 2) ? m - 1 : 0;
          m = small_deflate<N>(e, m, cfg.eps);
        }
        steps += run ? 1 : 0;
        run = run && m > 2;
      }
      mfin = m;
    }
  }
  if constexpr (N >= 2) {
    float lo, hi, c, s;  // exact 2x2 closeout (_kernels.py:401-417)
    wilkinson(d[0], e[0], d[1], lo, hi, c, s);
    d[0] = lo;
    d[1] = hi;
    small_fold<N, VECS>(v, 0, c, s, -s);
  }

  // ---- sort (stable) + sign, staged back through shared memory.  Ranks
  // from one comparison per pair: with x = d (descending) or -d
  // (ascending), k < c sorts first iff x_k >= x_c (ties keep index order,
  // solver.py:60-76).
  int rank[N];
#pragma unroll
  for (int c = 0; c < N; ++c) rank[c] = cfg.sort != 0 ? 0 : c;
  if (cfg.sort != 0) {
    const float sg = cfg.sort == 1 ? 1.0f : -1.0f;
#pragma unroll
    for (int c = 1; c < N; ++c)
#pragma unroll
      for (int k = 0; k < c; ++k) {
        const int kb = (sg * d[k] >= sg * d[c]) ? 1 : 0;
        rank[c] += kb;
        rank[k] += 1 - kb;
      }
  }
  __syncthreads();  // every thread is done reading its input tile
  if (live) {
    float* lrow = ltile + tid * Lay::LSTRIDE;
#pragma unroll
    for (int c = 0; c < N; ++c) lrow[rank[c]] = d[c] * scale;
    if constexpr (POW) {
      // f_k = max(lambda_k, floor)^p with the per-matrix floor (solver.py:127-139)
      float lmax = d[0] * scale;
#pragma unroll
      for (int k = 1; k < N; ++k) lmax = fmaxf(lmax, d[k] * scale);
      const float fl = pw.floor_abs < 0.0f ? 1e-12f * lmax : pw.floor_abs;
      float f[N];
      bool bad = false;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const float x = fmaxf(d[k] * scale, fl);
        bad = bad || (pw.needs_positive && !(x > 0.0f));
        f[k] = x;
      }
#pragma unroll
      for (int k = 0; k < N; ++k) f[k] = bad ? 0.0f : spectral_pow(f[k], pw.p);
      if (bad && status == kStatusOk) status = kStatusNonPositive;
      float* my = tile + tid * Lay::STRIDE;
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int c = r; c < N; ++c) {  // symmetric by construction (solver.py:141)
          float acc = 0.0f;
#pragma unroll
          for (int k = 0; k < N; ++k) acc = fmaf(v_at<NP, N>(v, r, k) * f[k], v_at<NP, N>(v, c, k), acc);
          my[r * N + c] = acc;
          my[c * N + r] = acc;
        }
    } else if constexpr (VECS) {
      float* my = tile + tid * Lay::STRIDE;
#pragma unroll
      for (int c = 0; c < N; ++c) {
        float best = -1.0f, lead = 0.0f;
#pragma unroll
        for (int r = 0; r < N; ++r) {
          const float x = v_at<NP, N>(v, r, c);
          const float mag = fabsf(x);
          if (mag > best) { best = mag; lead = x; }
        }
        const float flip = lead < 0.0f ? -1.0f : 1.0f;
#pragma unroll
        for (int r = 0; r < N; ++r) my[r * N + rank[c]] = v_at<NP, N>(v, r, c) * flip;
      }
    }
    if (status_out) status_out[base + tid] = status;
    if (steps_out) steps_out[base + tid] = steps;
    dg.put(base + tid, rot, N >= 2 ? N - mfin : 0, srs, res_out);
  }
  if (flags) {
    unsigned bits = __reduce_or_sync(0xffffffffu, (live && status) ? (1u << status) : 0u);
    if ((tid & 31) == 0 && bits) atomicOr(flags, (int)bits);
  }
  __syncthreads();
  {
    float* dstl = evals + base * N;
    for (int g = tid; g < count * N; g += kSmallThreads) dstl[g] = ltile[(g / N) * Lay::LSTRIDE + g % N];
    if constexpr (VECS) {
      float* dst = evecs + base * NN;
      const int total = count * NN;
      if ((NN % 4 == 0) && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
        float4* dst4 = reinterpret_cast<float4*>(dst);
        for (int g4 = tid; g4 < total / 4; g4 += kSmallThreads) {
          int g = 4 * g4;
          const float* s = tile + (g / NN) * Lay::STRIDE + (g % NN);
          dst4[g4] = make_float4(s[0], s[1], s[2], s[3]);
        }
      } else {
        for (int g = tid; g < total; g += kSmallThreads) dst[g] = tile[(g / NN) * Lay::STRIDE + (g % NN)];
      }
    }
  }
}

}  // namespace bed
