/*
 * bed200.h -- C ABI of the B200-native batched symmetric eigendecomposition
 * (arXiv 2207.04228: Householder tridiagonalisation + double-Wilkinson-shift
 * Givens QR with per-matrix deflation, eigenvector accumulation, and the
 * Taylor-polynomial ED backward).
 *
 * Plain pointers and sizes only.  Device entry points take device pointers
 * and a CUDA stream (cudaStream_t passed as void*), are asynchronous and
 * stream-ordered and reentrant (one call per device stream).  For n <= 8
 * nothing is allocated.  For n >= 9 the forward needs a device workspace:
 * bed_forward_ws_f32 takes it from the caller (size from
 * bed_forward_workspace_bytes; a smaller one solves the batch in chunks),
 * bed_forward_f32 allocates it per call (at most 4 GiB, chunk by chunk) from
 * a private stream-ordered pool of the library on the current device --
 * the device's default pool is not touched.  The host entry point takes
 * host pointers and does the copies itself.
 *
 * Reference interfaces each entry point replaces (paths relative to the
 * reference package root /root/reference/pkg/src/batchedeig):
 *
 *   bed_forward_f32        batched_eig()            solver.py:79-112
 *                          = validate               core.py:286-309
 *                          + tridiagonalize_kernel  _kernels.py:36-92
 *                            (values-only: reduce_band_kernel _kernels.py:95-202)
 *                          + qr_loop_kernel         _kernels.py:321-398
 *                          + finalize_kernel        _kernels.py:401-417
 *                          + accumulate_reflectors / wy_accumulate
 *                                                   householder.py:216-271
 *                          + V = P @ Q              solver.py:93
 *                          + _sort_and_sign         solver.py:60-76
 *   bed_forward_ws_f32     the same, with a caller-owned workspace
 *   bed_forward_workspace_bytes  its size (the reference preallocates
 *                          its kernels' buffers in the caller the same way,
 *                          householder.py:190-192, qr.py:601-602)
 *   bed_forward_host_f32   the same call on host (numpy-side) buffers, the
 *                          way the reference API is called (solver.py:79)
 *   bed_forward_host_f64   the same on float64 host buffers with the reference's
 *                          float64 validate (core.py:286-309) on host threads
 *   bed_backward_f32       (absent in the reference: pkg/README.md:116-117)
 *                          ED backward with Taylor-K
 *   bed_forward_power_f32  batched_eig() + matrix_power() in one call, fused into the
 *                          forward's epilogue for n <= 24 (V never written)
 *   bed_matrix_power_f32   matrix_power()           solver.py:115-143
 *                          (the ED's spectral-
 *                          function consumer, V diag(f(lambda)) V^T)
 *   bed_scatter_f32        the scatter inside zca_whiten()  solver.py:161-166
 *                          (covariance producer)
 *   bed_scatter_forward_f32  scatter + batched_eig [+ matrix_power]  solver.py:79-166,
 *                          one kernel for n <= 8 (the covariance never written)
 *   bed_error_string       error text for the integer return codes; the
 *                          reference maps kernel status ints to exceptions
 *                          in qr.py:604-609 / oracle.py:76-79
 */
#ifndef BED200_H_
#define BED200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BED200_ABI_VERSION 2

/* Return codes of every entry point. */
#define BED_SUCCESS 0
#define BED_ERR_INVALID_ARGUMENT 1 /* null pointer, n out of [1, 64], batch < 0, bad enum */
#define BED_ERR_MISALIGNED 2       /* pointer not aligned to its 4-byte element size */
#define BED_ERR_CUDA 3             /* launch / runtime failure (see bed_last_cuda_error) */
#define BED_ERR_NO_DEVICE 4        /* no sm_100 device visible */

/* Per-matrix numerical status (written to `status`), mirroring the
 * reference exceptions NoConvergence / NonFinite / NonSymmetric
 * (core.py:46-93). */
#define BED_STATUS_OK 0
#define BED_STATUS_NO_CONVERGENCE 1 /* budget exhausted, a coupling >= deflation_tol remains */
#define BED_STATUS_NON_FINITE 2     /* NaN/Inf in the input matrix */
#define BED_STATUS_NON_SYMMETRIC 3  /* max|a_ij-a_ji| > symmetry_tol * max(1, ||A||_F) */
#define BED_STATUS_NON_POSITIVE 4   /* bed_matrix_power_f32: non-positive clamped eigenvalue
                                       with a negative or fractional power (NonPositiveSpectrum);
                                       bed_backward_f32: a pair outside the Taylor series'
                                       domain (see there) */

#define BED_SORT_NONE 0
#define BED_SORT_DESCENDING 1
#define BED_SORT_ASCENDING 2

/* SolverConfig (core.py:226-279) as the kernels see it. */
typedef struct bed_config {
  float deflation_tol;      /* absolute, on the power-of-two equilibrated band (qr.py:512-515);
                               values below the FP32 floor 2^-22 act as 2^-22 */
  float symmetry_tol;       /* relative asymmetry tolerance (core.py:254) */
  int32_t max_double_steps; /* <= 0 resolves to 2n (core.py:270-271) */
  int32_t sort;             /* BED_SORT_* */
  int32_t compute_vectors;  /* 0: eigenvalues only (solver.py:94-109) */
  int32_t reserved;         /* must be 0 */
} bed_config;

/* Forward: A (batch, n, n) row-major FP32, symmetrised on load.
 *   evals  (batch, n)            required
 *   evecs  (batch, n, n)         required iff compute_vectors; column j pairs with evals[:, j]
 *   status (batch) int32         nullable; BED_STATUS_*
 *   steps  (batch) int32         nullable; double-shift steps this matrix used
 *   flags  (1) int32             nullable; set to OR over matrices of (1 << status)
 * Eigenvalues are ordered per cfg->sort and every eigenvector column is sign
 * normalised so its largest-magnitude entry (first on ties) is >= 0.
 * All pointers are device pointers; `stream` is a cudaStream_t (NULL = legacy default). */
int bed_forward_f32(const float* A, int64_t batch, int32_t n, float* evals, float* evecs,
                    int32_t* status, int32_t* steps, int32_t* flags, const bed_config* cfg,
                    void* stream);

/* Bytes of device workspace bed_forward_ws_f32 needs to solve `batch`
 * matrices of order n in one pass; 0 for n <= 8 (or batch <= 0).  The
 * smallest workspace accepted is bed_forward_workspace_bytes(32, n, cfg):
 * between the two, the batch is solved in chunks of whole multiples of 32.
 * Values-only: 4 (2n + 1) bytes per matrix (the band, a status).  With
 * vectors: plus P (4 n^2 bytes), the unsorted eigenvalues (4 n) and the
 * rotation record the band QR streams to the eigenvector fold -- every sweep
 * the double-step budget allows (2 max_double_steps + 1), NMAX - 1 positions
 * of 8 bytes (NMAX = 16, 24, 32 or 64, the size tier of n). */
size_t bed_forward_workspace_bytes(int64_t batch, int32_t n, const bed_config* cfg);

/* bed_forward_f32 with a caller-owned device workspace (256-byte aligned,
 * ignored for n <= 8) and the optional per-matrix diagnostics of the
 * reference's SolveDiagnostics / NoConvergence (qr.py:101-118, :385-389):
 *   diag   (batch, 3) int32  nullable; [rotations applied (sum of active - 1
 *                            over the matrix's sweeps), reduction events
 *                            (trailing deflations), step_r_sum (reductions
 *                            so far, summed over its double steps)]
 *   resid  (batch) float     nullable; largest active coupling (equilibrated
 *                            band) left when the budget ran out, else 0
 * No allocation inside.  BED_ERR_INVALID_ARGUMENT if the workspace is
 * smaller than bed_forward_workspace_bytes(32, n, cfg). */
int bed_forward_ws_f32(const float* A, int64_t batch, int32_t n, float* evals, float* evecs,
                       int32_t* status, int32_t* steps, int32_t* flags, int32_t* diag, float* resid,
                       const bed_config* cfg, void* workspace, size_t workspace_bytes, void* stream);

/* Same computation on HOST buffers (pinned or pageable), on CUDA device
 * `device`.  Streams the batch through the GPU in chunks with copies
 * overlapped against compute; returns after the results are on the host. */
int bed_forward_host_f32(const float* A, int64_t batch, int32_t n, float* evals, float* evecs,
                         int32_t* status, int32_t* steps, const bed_config* cfg, int32_t device);

/* Backward with the Taylor-polynomial K of degree `taylor_degree` (paper: 9):
 *   gA = sym( V (F o (V^T gV) + diag(gL)) V^T ),  sym(M) = (M + M^T)/2,
 *   F_ij ~ 1/(l_j - l_i) via (1/l_big) sum_{k=0..degree} (l_small/l_big)^k.
 * The series is the paper's for positive spectra (covariance inputs).  A pair
 * outside its domain -- l_big <= 0, or l_small <= -l_big (|ratio| >= 1 and not
 * a tie) -- takes the exact 1/(l_j - l_i) instead, and the matrix's status is
 * BED_STATUS_NON_POSITIVE (bit 1 << 4 in flags).  Two zero eigenvalues give 0.
 * V (batch,n,n), evals (batch,n) as returned by bed_forward_f32; gV and gL
 * are nullable (zero cotangent); gA (batch,n,n) is written; status (batch)
 * and flags (1) are nullable.  Device pointers, stream-ordered. */
int bed_backward_f32(const float* V, const float* evals, const float* gV, const float* gL,
                     float* gA, int64_t batch, int32_t n, int32_t taylor_degree, int32_t* status,
                     int32_t* flags, void* stream);

/* Spectral power  out = sym( V diag(max(evals, floor)^p) V^T )  of a decomposed
 * batch (reference matrix_power, solver.py:115-143).  floor < 0 selects the
 * reference default 1e-12 * max(evals) per matrix.  With p negative or
 * fractional, a matrix whose clamped spectrum is not positive gets status
 * BED_STATUS_NON_POSITIVE (and bit 1 << 4 in flags) and a zero output.
 * V (batch,n,n), evals (batch,n) as returned by bed_forward_f32; out (batch,n,n);
 * status (batch) and flags (1) nullable.  Device pointers, stream-ordered. */
int bed_matrix_power_f32(const float* V, const float* evals, float* out, int32_t* status,
                         int32_t* flags, int64_t batch, int32_t n, float p, float floor,
                         void* stream);

/* The float64 host call a reference user makes (batched_eig on float64 numpy,
 * solver.py:79-112): A, evals, evecs are HOST float64 buffers (pageable is fine).
 * Host threads validate each matrix as the reference does (core.py:286-309:
 * finite, max|a_ij - a_ji| <= symmetry_tol * max(1, ||A||_F), then (A + A^T) / 2,
 * all in float64), cast it to FP32 into page-locked staging, and the chunks
 * stream through the device (one stream per staging slot) while the threads
 * convert the next chunk in and the previous one out.  A matrix rejected on the
 * host gets BED_STATUS_NON_FINITE / _NON_SYMMETRIC and the zero matrix's results.
 * status, steps, diag (batch x 3: rotations, reduction events, step_r_sum), resid
 * are host arrays, nullable.  threads <= 0: all hardware threads (<= 64).  Calls
 * for the same device serialise on its staging buffer (kept between calls). */
int bed_forward_host_f64(const double* A, int64_t batch, int32_t n, double* evals, double* evecs,
                         int32_t* status, int32_t* steps, int32_t* diag, float* resid,
                         const bed_config* cfg, int32_t device, int32_t threads);

/* Eigenvalues and the spectral power  out = V diag(max(evals, floor)^p) V^T  in one
 * call (reference batched_eig + matrix_power, solver.py:79-143),
 * without returning V.  n <= 24: the power is formed in the forward's epilogue (n <= 8:
 * from V in the registers of the thread that solved the matrix; 9 <= n <= 24: in the
 * eigenvector fold, from V in registers and shared memory), so V never reaches memory;
 * n >= 25: V goes to the workspace and the tiled power kernel reads it.  Workspace:
 * bed_forward_power_workspace_bytes.
 * cfg->compute_vectors is ignored (vectors are implied); floor < 0 = the reference
 * default 1e-12 * max(evals); status/flags as bed_forward_f32, plus
 * BED_STATUS_NON_POSITIVE as bed_matrix_power_f32.  out is symmetric. */
size_t bed_forward_power_workspace_bytes(int64_t batch, int32_t n, const bed_config* cfg);
int bed_forward_power_f32(const float* A, int64_t batch, int32_t n, float* evals, float* out,
                          int32_t* status, int32_t* flags, const bed_config* cfg, float p,
                          float floor, void* workspace, size_t workspace_bytes, void* stream);

/* Covariance producer: out = sym((X - mu)(X - mu)^T) + eps I
 * per matrix, X (batch, n, m) row-major FP32 (n channels <= 64, m >= 1 samples), mu the
 * per-channel sample mean -- the scatter of the reference zca_whiten (solver.py:161-166).
 * out (batch, n, n).  Device pointers, stream-ordered. */
int bed_scatter_f32(const float* X, int64_t batch, int32_t n, int32_t m, float eps, float* out,
                    void* stream);

/* Covariance -> eigendecomposition in one call (SURVEY.md 8(f) row 3 feeding row 1;
 * reference zca_whiten's scatter + batched_eig [+ matrix_power], solver.py:79-166):
 * A = sym((X - mu)(X - mu)^T) + eps I formed from X (batch, n, m) as bed_scatter_f32
 * does, then solved as bed_forward_f32 (power == 0: out = V when cfg->compute_vectors,
 * else unused) or bed_forward_power_f32 (power != 0: out = A^p with floor as there).
 * n <= 8: ONE kernel -- each thread forms its matrix from X in registers, so A never
 * reaches memory and no workspace is needed; n >= 9: A goes to the workspace, sized by
 * bed_scatter_forward_workspace_bytes.  status/flags as bed_forward_f32 /
 * bed_forward_power_f32; a non-finite sample in X gives BED_STATUS_NON_FINITE. */
size_t bed_scatter_forward_workspace_bytes(int64_t batch, int32_t n, int32_t m,
                                           const bed_config* cfg, int32_t power);
int bed_scatter_forward_f32(const float* X, int64_t batch, int32_t n, int32_t m, float eps,
                            float* evals, float* out, int32_t* status, int32_t* flags,
                            const bed_config* cfg, int32_t power, float p, float floor,
                            void* workspace, size_t workspace_bytes, void* stream);

const char* bed_error_string(int code);
const char* bed_last_cuda_error(void); /* thread-local text of the last BED_ERR_CUDA */
int bed_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* BED200_H_ */
