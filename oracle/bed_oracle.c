/*
 * bed_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain-C, float64 restatement of the reference CPU eigensolver
 * (`batchedeig.batched_eig`, /root/reference/pkg/src/batchedeig/solver.py:79-112)
 * used only as the parity checker for the CUDA path and as the CPU baseline
 * leg of bench.py.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product path
 * (paper_2207_04228_b200) never links or calls anything in oracle/.
 *
 * Every stage cites the reference function it restates:
 *   validate            core.py:286-309
 *   tridiagonalize      _kernels.py:36-92 (tridiagonalize_kernel); values-only
 *                       path reduce_band_kernel _kernels.py:95-202 is the same
 *                       per-matrix arithmetic
 *   band scale          qr.py:522-534 (_band_scale), applied qr.py:596-598
 *   wilkinson pair      _kernels.py:205-218 (_wilkinson_scalar)
 *   sweep               _kernels.py:221-300 (_sweep_block)
 *   deflation gate      _kernels.py:303-318 (_deflate_scan, batch-wide max)
 *   QR loop             _kernels.py:321-398 (qr_loop_kernel)
 *   no-convergence      qr.py:385-389, qr.py:604-612
 *   2x2 closeout        _kernels.py:401-417 (finalize_kernel)
 *   reflector product   householder.py:216-231 (accumulate_reflectors; the
 *                       WY route householder.py:234-271 is the same product)
 *   V = P Q             solver.py:93
 *   sort and sign       solver.py:60-76 (_sort_and_sign)
 *
 * gate = BEDO_GATE_BATCH reproduces the reference's batch-wide deflation
 * gate exactly (results depend on the batch).  gate =
 * BEDO_GATE_MATRIX runs the same loop on every matrix as a batch of one
 * (the reference applied matrix by matrix), which is the per-matrix
 * deflation the CUDA path implements.
 *
 * Build: see oracle/Makefile (gcc -O2 -ffp-contract=off, no fast-math, so the
 * arithmetic is IEEE double like numba's default).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define BEDO_OK 0
#define BEDO_NOCONV 1
#define BEDO_NONFINITE 2
#define BEDO_NONSYM 3

#define BEDO_GATE_BATCH 0
#define BEDO_GATE_MATRIX 1

#define BEDO_SORT_NONE 0
#define BEDO_SORT_DESC 1
#define BEDO_SORT_ASC 2

typedef struct {
  double deflation_tol;   /* core.py:249 default 1e-5 */
  double symmetry_tol;    /* core.py:254 default 1e-12 */
  int32_t max_double_steps; /* resolved (core.py:270-271): caller passes 2n for None */
  int32_t sort;           /* BEDO_SORT_* ; core.py:252 default descending */
  int32_t compute_vectors;
  int32_t strict;         /* core.py:255 */
  int32_t gate;           /* BEDO_GATE_* */
  int32_t threads;        /* worker threads (>=1) */
  int64_t chunk;          /* matrices per gate group for GATE_BATCH (0 = whole batch) */
} bedo_config;

/* Per-matrix outputs beyond values/vectors; any pointer may be NULL. */
typedef struct {
  int32_t* status;          /* (b) BEDO_* */
  int32_t* converged_steps; /* (b) qr.py:101-118 converged_steps */
  int32_t* double_steps;    /* (b) double steps of the loop that solved this matrix */
  int64_t* rotations;       /* (b) rotations of the loop that solved this matrix */
  double* residual;         /* (b) max |e| left in the active block at exhaustion */
} bedo_outputs;

/* ------------------------------------------------------------------ */
/* validate: core.py:286-309.  Returns status; out = (A + A^T)/2.       */
static int validate_one(const double* a, int n, double sym_tol, double* out) {
  for (int i = 0; i < n * n; ++i)
    if (!isfinite(a[i])) return BEDO_NONFINITE;
  double asym = 0.0, fro2 = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double d = fabs(a[i * n + j] - a[j * n + i]);
      if (d > asym) asym = d;
      fro2 += a[i * n + j] * a[i * n + j];
    }
  double fro = sqrt(fro2);
  double limit = sym_tol * (fro > 1.0 ? fro : 1.0);
  if (asym > limit) return BEDO_NONSYM;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) out[i * n + j] = (a[i * n + j] + a[j * n + i]) / 2.0;
  return BEDO_OK;
}

/* ------------------------------------------------------------------ */
/* tridiagonalize_kernel, _kernels.py:36-92, one matrix.               */
/* w: (n,n) in place; vec: (n-2, n) unit reflectors (zeroed by caller). */
static void tridiagonalize_one(double* w, int n, double* vec, double* p) {
  for (int i = 0; i < n - 2; ++i) {
    int tail = n - i - 1;
    double scale = 0.0;
    for (int t = 0; t < tail; ++t) {
      double v = fabs(w[(i + 1 + t) * n + i]);
      if (v > scale) scale = v;
    }
    if (scale <= 1e-300) continue; /* householder.py:37-39 _ZERO_TAIL */
    double sumsq = 0.0;
    for (int t = 0; t < tail; ++t) {
      double v = w[(i + 1 + t) * n + i] / scale;
      sumsq += v * v;
    }
    double norm = scale * sqrt(sumsq);
    double pivot = w[(i + 1) * n + i];
    double sigma = pivot >= 0 ? norm : -norm;
    double u0 = pivot + sigma;
    double unorm = sqrt(2.0 * fabs(sigma)) * sqrt(fabs(u0));
    double* u = vec + (size_t)i * n;
    u[i + 1] = u0 / unorm;
    for (int t = 1; t < tail; ++t) u[i + 1 + t] = w[(i + 1 + t) * n + i] / unorm;

    int m = n - i;
    for (int r = 0; r < m; ++r) {
      double acc = 0.0;
      for (int c = 1; c < m; ++c) acc += w[(i + r) * n + i + c] * u[i + c];
      p[r] = 2.0 * acc;
    }
    double kk = 0.0;
    for (int r = 1; r < m; ++r) kk += u[i + r] * p[r];
    for (int r = 1; r < m; ++r) p[r] = p[r] - kk * u[i + r];
    double q0 = p[0];
    for (int c = 1; c < m; ++c) w[i * n + i + c] -= q0 * u[i + c];
    for (int r = 1; r < m; ++r) {
      double ur = u[i + r];
      double qr = p[r];
      w[(i + r) * n + i] -= ur * q0;
      for (int c = 1; c < m; ++c) w[(i + r) * n + i + c] -= qr * u[i + c] + ur * p[c];
    }
  }
}

/* ------------------------------------------------------------------ */
/* _band_scale, qr.py:522-534 (numpy exp2(ceil(log2(top)))).            */
static double band_scale(const double* d, const double* e, int n) {
  double top = 0.0;
  for (int i = 0; i < n; ++i)
    if (fabs(d[i]) > top) top = fabs(d[i]);
  for (int i = 0; i < n - 1; ++i)
    if (fabs(e[i]) > top) top = fabs(e[i]);
  double safe = top > 0 ? top : 1.0;
  return exp2(ceil(log2(safe)));
}

/* _wilkinson_scalar, _kernels.py:205-218. */
static void wilkinson(double a, double bb, double d, double* lo, double* hi, double* c_out,
                      double* s_out) {
  if (bb == 0.0) {
    *lo = a; *hi = d; *c_out = 1.0; *s_out = 0.0;
    return;
  }
  double m = (a - d) / (2.0 * bb);
  double sign = m >= 0 ? 1.0 : -1.0;
  double t = -sign / (fabs(m) + hypot(1.0, m));
  double c = 1.0 / sqrt(1.0 + t * t);
  double s = c * t;
  double bcs2 = 2.0 * bb * c * s;
  *lo = a * c * c - bcs2 + d * s * s;
  *hi = a * s * s + bcs2 + d * c * c;
  *c_out = c;
  *s_out = s;
}

/* Right-multiply q (n x n, row-major) by the rotation at (pos, pos+1). */
static void fold(double* q, int n, int pos, double c, double s) {
  if (!q) return;
  for (int row = 0; row < n; ++row) {
    double qp = q[row * n + pos];
    double qn = q[row * n + pos + 1];
    q[row * n + pos] = c * qp - s * qn;
    q[row * n + pos + 1] = s * qp + c * qn;
  }
}

/* _sweep_block, _kernels.py:221-300, one matrix: d (n), e (n-1). */
static void sweep_one(double* d, double* e, double* q, int n, int m, double mu) {
  double dw = d[0] - mu, g = e[0];
  double c1 = 1.0, s1 = 0.0, c2 = 1.0, r1 = 0.0, u1 = 0.0;
  for (int i = 0; i < m - 1; ++i) {
    double ei = e[i];
    int live = ei != 0.0;
    double adw = fabs(dw), aei = fabs(ei);
    double am = adw >= aei ? adw : aei;
    double ams = am > 0.0 ? am : 1.0;
    double t1 = dw / ams, t2 = ei / ams;
    double hh = sqrt(t1 * t1 + t2 * t2);
    double ih = 1.0 / (hh > 0.0 ? hh : 1.0);
    double c = live ? t1 * ih : 1.0;
    double s = live ? -t2 * ih : 0.0;
    double r = live ? am * hh : dw;
    double dn = d[i + 1] - mu;
    double cn = c, sn = s, rn = r;
    double un = c * g - s * dn;
    dw = s * g + c * dn;
    if (i > 0) {
      d[i - 1] = c1 * (c2 * r1) - s1 * u1 + mu;
      e[i - 1] = -s1 * rn;
      fold(q, n, i - 1, c1, s1);
    }
    c2 = c1; c1 = cn; s1 = sn; r1 = rn; u1 = un;
    if (i < m - 2) g = c1 * e[i + 1];
  }
  d[m - 2] = c1 * (c2 * r1) - s1 * u1 + mu;
  e[m - 2] = -s1 * dw;
  d[m - 1] = c1 * dw + mu;
  fold(q, n, m - 2, c1, s1);
}

/* ------------------------------------------------------------------ */
/* qr_loop_kernel (_kernels.py:321-398) + finalize (_kernels.py:401-417)
 * over a group of `b` matrices sharing one batch-wide gate.  d: (b,n),
 * e: (b,n-1) matrix-major; q: (b,n,n) or NULL.  Returns the loop status
 * (1 = budget exhausted with the active block above 2).                 */
static int deflate_scan(const double* e, int b, int n, int active, double eps) {
  int shrink = 0;
  while (active - shrink > 2) {
    int pos = active - shrink - 2;
    double worst = 0.0;
    for (int k = 0; k < b; ++k) {
      double v = fabs(e[(size_t)k * (n - 1) + pos]);
      if (v > worst) worst = v;
    }
    if (worst >= eps) break;
    shrink += 1;
  }
  return shrink;
}

static int qr_group(double* d, double* e, double* q, int b, int n, double eps, int max_steps,
                    int strict, const bedo_outputs* out, int64_t base) {
  int active = n, double_steps = 0, status = 0;
  int64_t rotations = 0;
  int* converged = (int*)malloc(sizeof(int) * (size_t)b);
  int* vact = (int*)malloc(sizeof(int) * (size_t)b);
  double* los = (double*)malloc(sizeof(double) * (size_t)b);
  double* his = (double*)malloc(sizeof(double) * (size_t)b);
  for (int k = 0; k < b; ++k) { converged[k] = -1; vact[k] = n; }

  if (n >= 3) {
    active -= deflate_scan(e, b, n, active, eps);
    for (int k = 0; k < b; ++k) {
      const double* ek = e + (size_t)k * (n - 1);
      int va = vact[k];
      while (va > 2 && fabs(ek[va - 2]) < eps) va -= 1;
      vact[k] = va;
      if (va <= 2) converged[k] = 0;
    }
    while (active > 2) {
      if (double_steps >= max_steps) { status = 1; break; }
      for (int k = 0; k < b; ++k) {
        double c, s;
        wilkinson(d[(size_t)k * n + active - 2], e[(size_t)k * (n - 1) + active - 2],
                  d[(size_t)k * n + active - 1], &los[k], &his[k], &c, &s);
      }
      for (int k = 0; k < b; ++k)
        sweep_one(d + (size_t)k * n, e + (size_t)k * (n - 1), q ? q + (size_t)k * n * n : NULL,
                  n, active, his[k]);
      rotations += active - 1;
      active -= deflate_scan(e, b, n, active, eps);
      for (int k = 0; k < b; ++k) {
        if (converged[k] < 0) {
          const double* ek = e + (size_t)k * (n - 1);
          int va = vact[k];
          while (va > 2 && fabs(ek[va - 2]) < eps) va -= 1;
          vact[k] = va;
          if (va <= 2) converged[k] = double_steps + 1;
        }
      }
      if (active > 2) {
        for (int k = 0; k < b; ++k)
          sweep_one(d + (size_t)k * n, e + (size_t)k * (n - 1),
                    q ? q + (size_t)k * n * n : NULL, n, active, los[k]);
        rotations += active - 1;
        active -= deflate_scan(e, b, n, active, eps);
      }
      double_steps += 1;
    }
  }
  /* qr.py:604-612: strict exhaustion raises NoConvergence naming every
   * matrix whose active-block couplings are still >= eps (qr.py:385-389). */
  for (int k = 0; k < b; ++k) {
    int st = BEDO_OK;
    double resid = 0.0;
    if (status) {
      const double* ek = e + (size_t)k * (n - 1);
      for (int j = 0; j < active - 1; ++j)
        if (fabs(ek[j]) > resid) resid = fabs(ek[j]);
      if (strict && resid >= eps) st = BEDO_NOCONV;
    }
    if (out->status) out->status[base + k] = st;
    if (out->residual) out->residual[base + k] = resid;
    if (out->converged_steps)
      out->converged_steps[base + k] = converged[k] < 0 ? double_steps : converged[k];
    if (out->double_steps) out->double_steps[base + k] = double_steps;
    if (out->rotations) out->rotations[base + k] = rotations;
  }
  /* finalize: _kernels.py:401-417, qr.py:610-612 (exhausted -> active=2). */
  int final_active = status ? 2 : active;
  if (n >= 2 && final_active == 2) {
    for (int k = 0; k < b; ++k) {
      double lo, hi, c, s;
      double* dk = d + (size_t)k * n;
      double* ek = e + (size_t)k * (n - 1);
      wilkinson(dk[0], ek[0], dk[1], &lo, &hi, &c, &s);
      dk[0] = lo; dk[1] = hi; ek[0] = 0.0;
      fold(q ? q + (size_t)k * n * n : NULL, n, 0, c, s);
    }
  }
  free(converged); free(vact); free(los); free(his);
  return status;
}

/* ------------------------------------------------------------------ */
/* Solve one gate group of matrices [k0, k0+b).                          */
typedef struct {
  const double* a;
  int n;
  int64_t k0, b;
  const bedo_config* cfg;
  double* evals;
  double* evecs;
  const bedo_outputs* out;
} group_job;

static void solve_group(const group_job* job) {
  const int n = job->n;
  const int64_t b = job->b;
  const bedo_config* cfg = job->cfg;
  const size_t nn = (size_t)n * n;
  double* w = (double*)calloc((size_t)b * nn, sizeof(double));
  double* vec = (double*)calloc((size_t)b * (n > 2 ? n - 2 : 1) * n, sizeof(double));
  double* d = (double*)calloc((size_t)b * n, sizeof(double));
  double* e = (double*)calloc((size_t)b * (n > 1 ? n - 1 : 1), sizeof(double));
  double* scale = (double*)calloc((size_t)b, sizeof(double));
  double* q = cfg->compute_vectors ? (double*)calloc((size_t)b * nn, sizeof(double)) : NULL;
  double* p = (double*)calloc((size_t)n + 1, sizeof(double));
  int32_t* vstat = (int32_t*)calloc((size_t)b, sizeof(int32_t));
  int nbad = 0;

  for (int64_t k = 0; k < b; ++k) {
    const double* ak = job->a + (size_t)(job->k0 + k) * nn;
    vstat[k] = validate_one(ak, n, cfg->symmetry_tol, w + k * nn);
    if (vstat[k]) {
      nbad++;
      /* a rejected matrix is solved as the zero matrix so the group runs on */
      memset(w + k * nn, 0, nn * sizeof(double));
    }
  }
  for (int64_t k = 0; k < b; ++k) {
    tridiagonalize_one(w + k * nn, n, vec + (size_t)k * (n > 2 ? n - 2 : 1) * n, p);
    for (int i = 0; i < n; ++i) d[k * n + i] = w[k * nn + (size_t)i * n + i];
    for (int i = 0; i + 1 < n; ++i) e[k * (n - 1) + i] = w[k * nn + (size_t)(i + 1) * n + i];
    scale[k] = band_scale(d + k * n, e + k * (n - 1), n);
    for (int i = 0; i < n; ++i) d[k * n + i] /= scale[k];
    for (int i = 0; i + 1 < n; ++i) e[k * (n - 1) + i] /= scale[k];
    if (q) {
      double* qk = q + k * nn;
      for (int i = 0; i < n; ++i) qk[(size_t)i * n + i] = 1.0;
    }
  }
  (void)nbad;
  /* batch gate: the whole group shares one gate; matrix gate: each matrix
   * is its own group of one */
  int64_t gsize = cfg->gate == BEDO_GATE_MATRIX ? 1 : b;
  for (int64_t g0 = 0; g0 < b; g0 += gsize) {
    int64_t gb = g0 + gsize <= b ? gsize : b - g0;
    qr_group(d + g0 * n, e + g0 * (n > 1 ? n - 1 : 0), q ? q + g0 * nn : NULL, (int)gb, n,
             cfg->deflation_tol, cfg->max_double_steps, cfg->strict, job->out, job->k0 + g0);
  }

  double* vals = (double*)malloc(sizeof(double) * (size_t)n);
  int* perm = (int*)malloc(sizeof(int) * (size_t)n);
  double* pm = (double*)malloc(sizeof(double) * nn);
  double* vk = (double*)malloc(sizeof(double) * nn);
  for (int64_t k = 0; k < b; ++k) {
    int64_t gk = job->k0 + k;
    if (vstat[k] && job->out->status) job->out->status[gk] = vstat[k];
    for (int i = 0; i < n; ++i) vals[i] = d[k * n + i] * scale[k];
    if (q) {
      /* P = H_0 H_1 ... (householder.py:216-231) */
      memset(pm, 0, nn * sizeof(double));
      for (int i = 0; i < n; ++i) pm[(size_t)i * n + i] = 1.0;
      const double* vk_refl = vec + (size_t)k * (n > 2 ? n - 2 : 1) * n;
      for (int i = 0; i < n - 2; ++i) {
        const double* u = vk_refl + (size_t)i * n;
        for (int r = 0; r < n; ++r) {
          double pu = 0.0;
          for (int c = i + 1; c < n; ++c) pu += pm[(size_t)r * n + c] * u[c];
          for (int c = i + 1; c < n; ++c) pm[(size_t)r * n + c] -= 2.0 * pu * u[c];
        }
      }
      /* V = P Q (solver.py:93) */
      const double* qk = q + k * nn;
      for (int r = 0; r < n; ++r)
        for (int c = 0; c < n; ++c) {
          double acc = 0.0;
          for (int j = 0; j < n; ++j) acc += pm[(size_t)r * n + j] * qk[(size_t)j * n + c];
          vk[(size_t)r * n + c] = acc;
        }
    }
    /* _sort_and_sign, solver.py:60-76: stable argsort of -w (desc) or w */
    for (int i = 0; i < n; ++i) perm[i] = i;
    if (cfg->sort != BEDO_SORT_NONE) {
      for (int i = 1; i < n; ++i) { /* stable insertion sort */
        int pi = perm[i];
        double key = cfg->sort == BEDO_SORT_DESC ? -vals[pi] : vals[pi];
        int j = i - 1;
        while (j >= 0) {
          double kj = cfg->sort == BEDO_SORT_DESC ? -vals[perm[j]] : vals[perm[j]];
          if (kj > key) { perm[j + 1] = perm[j]; --j; } else break;
        }
        perm[j + 1] = pi;
      }
    }
    for (int i = 0; i < n; ++i) job->evals[(size_t)gk * n + i] = vals[perm[i]];
    if (q && job->evecs) {
      double* out = job->evecs + (size_t)gk * nn;
      for (int j = 0; j < n; ++j) {
        int src = perm[j];
        int lead = 0;
        double best = -1.0;
        for (int r = 0; r < n; ++r) {
          double v = fabs(vk[(size_t)r * n + src]);
          if (v > best) { best = v; lead = r; }
        }
        double flip = vk[(size_t)lead * n + src] < 0 ? -1.0 : 1.0;
        for (int r = 0; r < n; ++r) out[(size_t)r * n + j] = vk[(size_t)r * n + src] * flip;
      }
    }
  }
  free(vals); free(perm); free(pm); free(vk);
  free(w); free(vec); free(d); free(e); free(scale); free(q); free(p); free(vstat);
}

typedef struct {
  group_job* jobs;
  int64_t njobs;
  int64_t next;
  pthread_mutex_t lock;
} job_queue;

static void* worker(void* arg) {
  job_queue* jq = (job_queue*)arg;
  for (;;) {
    pthread_mutex_lock(&jq->lock);
    int64_t j = jq->next++;
    pthread_mutex_unlock(&jq->lock);
    if (j >= jq->njobs) break;
    solve_group(&jq->jobs[j]);
  }
  return NULL;
}

/* Entry point.  a: (batch, n, n) float64 row-major.  evals: (batch, n).
 * evecs: (batch, n, n) or NULL.  Returns 0, or -1 on bad arguments.      */
int bedo_forward(const double* a, int64_t batch, int32_t n, const bedo_config* cfg,
                 double* evals, double* evecs, const bedo_outputs* outs) {
  if (!a || !evals || !cfg || !outs || n < 1 || batch < 0) return -1;
  if (batch == 0) return 0;
  int64_t group;
  if (cfg->gate == BEDO_GATE_MATRIX) group = cfg->chunk > 0 ? cfg->chunk : 256;
  else group = cfg->chunk > 0 ? cfg->chunk : batch;
  int64_t njobs = (batch + group - 1) / group;
  group_job* jobs = (group_job*)malloc(sizeof(group_job) * (size_t)njobs);
  for (int64_t j = 0; j < njobs; ++j) {
    jobs[j].a = a;
    jobs[j].n = n;
    jobs[j].k0 = j * group;
    jobs[j].b = (j + 1) * group <= batch ? group : batch - j * group;
    jobs[j].cfg = cfg;
    jobs[j].evals = evals;
    jobs[j].evecs = evecs;
    jobs[j].out = outs;
  }
  int threads = cfg->threads > 0 ? cfg->threads : 1;
  job_queue jq;
  jq.jobs = jobs; jq.njobs = njobs; jq.next = 0;
  pthread_mutex_init(&jq.lock, NULL);
  if (threads == 1 || njobs == 1) {
    worker(&jq);
  } else {
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, worker, &jq);
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
  }
  pthread_mutex_destroy(&jq.lock);
  free(jobs);
  return 0;
}

/* Stage-level entry points used by the known-answer tests. */
void bedo_wilkinson(double a, double b, double d, double* out4) {
  wilkinson(a, b, d, &out4[0], &out4[1], &out4[2], &out4[3]);
}

void bedo_tridiagonalize(double* w, int64_t batch, int32_t n, double* vectors) {
  double* p = (double*)calloc((size_t)n + 1, sizeof(double));
  for (int64_t k = 0; k < batch; ++k)
    tridiagonalize_one(w + (size_t)k * n * n, n, vectors + (size_t)k * (n > 2 ? n - 2 : 1) * n, p);
  free(p);
}
