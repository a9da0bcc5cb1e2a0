/*
 * scg_phase.h -- C ABI of the B200-native SketchyCGAL hot path for the abstract phase retrieval
 * SDP ("Abstract phase retrieval").
 *
 * Problem (eqn:numerics-phase-retrieval-sdp):
 *     minimize tr X   s.t.  A X = b,  X psd,  tr X <= alpha,      A_i = a_i a_i^*,
 * with d = L n coded-diffraction measurements (L = 12 in the paper):
 *     a_{j n + l}^* = W_n(l, :) diag(psi_j)^*,  W_n(l, k) = exp(-2 pi i l k / n)   (reading R36),
 * so (A X)_{j,l} = (M_j X M_j^*)_{ll}, M_j = W_n diag(conj psi_j).  SketchyCGAL (Alg. 4,
 * P:1422-1470) with the trace-bounded linear minimization runs on the problem
 * scaled per eqn:problem-scaling (readings R37, R38):
 *     C~ = I / sqrt(n),  A~_i = kappa_j A_i  (kappa_j = 1 / (||psi_j||^2 ||A'||)),
 *     b~ = kappa b / alpha,  X = alpha X~.
 * Per iteration the library runs, on the GPU: one randomized Lanczos computation of the minimum
 * eigenvector of D_t = C~ + A~^*(y + beta_t (z - b~)) (Alg. 2 over C^n) whose
 * matrix-vector product is 2L FFTs of length n (a fused four-step FFT, n = n1 n2, written for
 * sm_100a: modulation, weights and the inner transposes happen inside the FFT kernels), the monitor
 * xi = v^* D_t v, the primal update z <- (1 - eta) z + eta A~(v v^*), the dual update
 * y <- y + gamma (z - b~), and the complex Nystrom sketch S <- (1 - eta) S + eta v (v^* Omega).
 *
 * Numerics: IEEE fp64 / complex128.  Unlike the MaxCut path (bitwise Canonical Arithmetic
 * Contract), the FFT's summation order is not the oracle's; parity is within the tolerances of
 * DESIGN.md section 11 (derived from the FFT's error bound).  Results are deterministic run to run
 * (fixed-order block reductions, no atomics on values).
 *
 * Conventions (as include/sketchycgal.h): every function returns scg_status (0 = OK, < 0 error;
 * the codes of sketchycgal.h).  Pointers are caller-owned HOST memory; inputs are copied before
 * the call returns; outputs go into caller-allocated buffers of the stated size.  Complex arrays
 * are interleaved (re, im) doubles.  The context owns its device memory and CUDA stream, is
 * single-writer, and is sticky-failed after a CUDA error (every later call: SCG_ESTATE).
 * One GPU ("replicas only" for this workload: DESIGN.md section 11).
 */
#ifndef SCG_PHASE_H
#define SCG_PHASE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct scg_pr_ctx scg_pr_ctx;

/* Per-iteration record (same fields as scg_iter_rec of sketchycgal.h), scaled units:
 * theta = Ritz value (Alg. 2), xi = v^* D_t v, c = v^* C~ v, p = <C~, X_t>,
 * znorm = ||z_{t+1} - b~||, gamma = dual step, tau = tr X_t, gap / bound = surrogate duality gap
 * and posterior bound with the trace-bounded term alpha~ min(xi, 0). */
typedef struct {
  int64_t t;
  int32_t q, k;
  double theta, xi, c, p, znorm, gamma, tau, gap, bound;
} scg_pr_rec;

/* Create a context on the current CUDA device.
 *   n      signal length; n = n1 n2 with 2 <= n1, n2 <= 4096 and every prime factor of n in
 *          {2, 3, 5} (n = 10^2 .. 10^6 of P:2028 qualify); else SCG_EUNSUPPORTED.
 *   L      number of modulations (d = L n), 1 <= L <= 32.
 *   psi    L x n complex, row j = waveform psi_j.  At most 256 distinct values over
 *          all entries (the coded-diffraction alphabet has 8), else SCG_EUNSUPPORTED; zero entries
 *          allowed but every psi_j must be nonzero (SCG_EINVAL).
 *   b      L x n measurements b[j n + l], original units.
 *   R      sketch rank 1 <= R <= 16 (the paper uses R = 5).
 *   alpha  trace bound (> 0; the paper sets alpha = 3 n); beta0 > 0 (default 1).
 *   seed   seeds Omega and the Lanczos start vectors (scg_rng.h streams 0 and 1, two normals per
 *          complex entry: re at index 2i, im at 2i + 1).
 *   flags  SCG_PR_PROFILE (1 << 8): per-kernel CUDA-event timing (scg_pr_kernel_stats);
 *          SCG_PR_TM2 (1 << 9): two transforms per FFT block instead of four (execution option);
 *          SCG_PR_GENERIC (1 << 10): runtime radix plans even where a compile-time plan exists
 *          (execution option; the results agree within the FFT's rounding);
 *          SCG_PR_NOPF_F1 / _B / _C (1 << 11 / 12 / 13): load the next tile after (instead of before)
 *          the current tile's transform in k_pr_f1 / k_pr_b / k_pr_c (execution options, same bits).
 * Errors: SCG_EINVAL, SCG_EUNSUPPORTED, SCG_ENOMEM, SCG_ECUDA. */
#define SCG_PR_PROFILE (1u << 8)
#define SCG_PR_TM2 (1u << 9)
#define SCG_PR_GENERIC (1u << 10)
#define SCG_PR_NOPF_F1 (1u << 11)
#define SCG_PR_NOPF_B (1u << 12)
#define SCG_PR_NOPF_C (1u << 13)
int scg_pr_init(int64_t n, int32_t L, const double *psi, const double *b, int32_t R, double alpha,
                double beta0, uint64_t seed, uint32_t flags, scg_pr_ctx **out);

/* Run T iterations (Alg. 4 lines 4-11), enqueued without host synchronization; returns after the
 * device finished.  q_t = min(n - 1, max(2, ceil(t^(1/4) ln n))); q_t > 256 is
 * SCG_EUNSUPPORTED (not reached before t ~ 10^5 at n = 10^6). */
int scg_pr_step(scg_pr_ctx *c, int64_t T);

/* Copy up to cap records of iterations 1..t (oldest first); *count = records written. */
int scg_pr_iter_log(scg_pr_ctx *c, scg_pr_rec *out, int64_t cap, int64_t *count);

/* State in natural order, scaled units:
 *   0 z (L n doubles)   1 y (L n)   2 v (n complex, last eigenvector)   3 S (n x R complex,
 *   column-major: S[k n + i])   4 Omega (n x R complex)   5 b~ (L n)   6 kappa (L doubles)
 *   7 scalars {t, tau, p, ||A'||, n1, n2, alpha, beta0} (8 doubles). */
int scg_pr_get_state(scg_pr_ctx *c, int32_t which, double *out);

/* NystromSketch.Reconstruct over C^n (Alg. 3): U (n x R complex, column-major,
 * orthonormal), Lam (R, descending) of the scaled X^ = U diag(Lam) U^*; no trace correction for the
 * trace-bounded set (reading R37).  SCG_ECHOL after 40 shift doublings. */
int scg_pr_reconstruct(scg_pr_ctx *c, double *U, double *Lam);

/* Signal estimate: chi = sqrt(alpha lambda_1) u_1 (n complex, original units) from
 * the last reconstruction (SCG_ESTATE before scg_pr_reconstruct). */
int scg_pr_signal(scg_pr_ctx *c, double *chi);

/* Test / bench hooks on the context's operator (device kernels, host buffers):
 *   apply_D: y = C~ x + A~^*(w) x for a given w (L n doubles, natural order) and x (n complex).
 *   measure: h = A~(x x^*), h[j n + l] = kappa_j |(M_j x)_l|^2 (L n doubles). */
int scg_pr_apply_D(scg_pr_ctx *c, const double *w, const double *x, double *y);
int scg_pr_measure(scg_pr_ctx *c, const double *x, double *h);

/* Per-kernel statistics (SCG_PR_PROFILE): name, launches, total ms, algorithmic bytes/launch. */
typedef struct {
  char name[32];
  int64_t launches;
  double total_ms;
  double bytes_per_launch;
} scg_pr_kstat;
int scg_pr_kernel_stats(scg_pr_ctx *c, scg_pr_kstat *out, int32_t cap, int32_t *count);
int scg_pr_reset_stats(scg_pr_ctx *c);

/* The CUDA stream the context launches on (cudaStream_t), for timing with events. */
void *scg_pr_stream(scg_pr_ctx *c);

int scg_pr_destroy(scg_pr_ctx *c);

#ifdef __cplusplus
}
#endif

#endif /* SCG_PHASE_H */
