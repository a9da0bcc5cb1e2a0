/*
 * sketchycgal.h -- C ABI of the B200-native SketchyCGAL MaxCut hot path.
 *
 * Method: SketchyCGAL (Yurtsever, Tropp, Fercoq, Udell, Cevher, arXiv 1912.02949),
 * Alg. 4 applied to the MaxCut SDP:
 *     maximize tr(L X)  s.t.  diag X = 1,  X psd,
 * posed as the model problem with C = -L, A = diag, b = 1,
 * alpha = n.  Per iteration t the library runs, on the GPU:
 *   - one randomized Lanczos min-eigenvector computation of
 *       D_t = C + A*(y + beta_t (z - b))          (Alg. 2)
 *     as two passes of fused SpMV + diagonal + three-term-recurrence kernels,
 *   - the primal update z <- (1-eta) z + eta alpha (v o v)   (Alg. 4 line 8)
 *   - the dual update    y <- y + gamma (z - b)               (Alg. 4 line 9)
 *   - the Nystrom sketch S <- (1-eta) S + eta alpha v (v^T Omega)  (Alg. 4 line 10,
 *     eqn:sketch-update PAPER.md:1162-1169).
 * The arithmetic follows the Canonical Arithmetic Contract of DESIGN.md section 3
 * (exact global sums, fixed row-sum order), so iterates are bitwise identical to
 * the CPU oracle's and independent of grid shape and GPU count.
 *
 * Conventions
 *   - All functions return scg_status (0 = OK, < 0 = error, see below).  No
 *     exception or C++ type crosses the ABI.  After a CUDA/NCCL error the context
 *     is sticky-failed and every later call returns SCG_ESTATE.
 *   - Ownership: every pointer argument is caller-owned HOST memory unless the
 *     comment says "device".  Inputs are copied before the call returns; outputs
 *     are written into caller-allocated buffers of the stated size.
 *   - The context owns all device memory and its CUDA stream.  A context is
 *     single-writer (not thread-safe); several contexts may coexist.
 *   - Multi-GPU: one process per GPU; every rank calls every function
 *     collectively with its own row range.  dist == NULL means one GPU owning
 *     all rows.
 *   - Results are reported in ORIGINAL units, even though the
 *     iteration runs on the scaled problem when SCG_SCALE
 *     is set.
 */
#ifndef SKETCHYCGAL_H
#define SKETCHYCGAL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct scg_ctx scg_ctx;

typedef enum {
  SCG_OK = 0,
  SCG_EINVAL = -1,   /* bad argument: n < 2, R < 1, R > n, alpha <= 0, beta0 <= 0,
                        malformed CSR (unsorted/out-of-range columns), bad shard bounds */
  SCG_ENOMEM = -2,   /* device or host allocation failed */
  SCG_ECUDA = -3,    /* CUDA runtime error (context becomes sticky-failed) */
  SCG_ENCCL = -4,    /* NCCL error (context becomes sticky-failed) */
  SCG_ECHOL = -5,    /* Nystrom reconstruction: Cholesky failed after 40 shift doublings */
  SCG_ESTATE = -6,   /* call on a failed context, or out of order (e.g. objective before reconstruct) */
  SCG_ERANGE = -7,   /* a summand of an exact sum was non-finite or >= 2^100 (DESIGN.md CAC-2) */
  SCG_EUNSUPPORTED = -8,
  SCG_ECOMM = -9     /* a host transport callback (scg_host_comm) failed */
} scg_status;

/* init flags */
enum {
  SCG_SCALE = 1u << 0,          /* problem scaling ||C||_F = ||A|| = alpha = 1; default on */
  SCG_TRACE_CORRECT = 1u << 1,  /* Lambda += (alpha - tr Lambda)/R after reconstruct (Alg. 4 line 13) */
  SCG_REGENERATE = 1u << 2,     /* storage-optimal two-pass Lanczos (regenerate v_2..v_k, Alg. 2 line 13 comment);
                                   default: keep the Lanczos vectors in HBM and combine them in one pass
                                   (Remark "Time-storage tradeoff") -- bitwise identical
                                   results, O(q n) device memory (falls back to two-pass if it does not fit) */
  SCG_TRACE_LE = 1u << 3,       /* trace-bounded set tr X <= alpha instead of tr X = alpha:
                                   the LMO is H = alpha v v^T if xi_t < 0, else 0; e.g. the
                                   DIMACS-style MaxCut setup alpha = 1.05 n.  Trace correction then
                                   uses the tracked trace tau instead of alpha (reading R29) */
  SCG_INEQ = 1u << 4,           /* general template with K = {u <= b}: diag X <= 1
                                   instead of diag X = 1; b is replaced by the slack w = min(z + y/beta, b) in D_t
                                   and in the dual update (reading R32); the gap / bound records are the
                                   general-template ones (reading R33) */
  SCG_PROFILE = 1u << 8,        /* record CUDA events around every 16th launch of each kernel class (bench /
                                   kernel stats) */
  /* execution options: none changes a single bit of the results (every variant is checked bitwise
     against the oracle by tests/test_gpu_parity.py); the defaults are the fastest measured on B200 */
  SCG_NO_PDL = 1u << 9,         /* launch without programmatic dependent launch (default: PDL on) */
  SCG_FUSED_PASS1 = 1u << 10,   /* one GPU: all q steps of Lanczos pass 1 in one persistent cooperative kernel */
  SCG_WS_SPMV = 1u << 11,       /* uniform weights: warp-specialized TMA SpMV (producer warp + mbarrier ring) */
  SCG_TMA_B = 1u << 12,         /* TMA-staged recurrence kernel (bulk copies into shared memory) */
  SCG_DEBUG_LOG = 1u << 13,     /* host init stage timings and layout facts on stderr */
  SCG_NO_ELL = 1u << 14,        /* keep the SELL-32 layout even when every row has <= 8 entries (ELL-W otherwise) */
  SCG_FUSED_RNG = 1u << 15,     /* one GPU: draw the next Lanczos start vector inside the dual-update kernel instead of
                                   on a lower-priority side stream overlapped with the Lanczos passes (sharded runs
                                   always draw inside the dual kernel) */
  SCG_NO_RESIDENT = 1u << 17,   /* one GPU, n <= 65536: keep the multi-kernel iteration instead of one launch of one
                                   thread-block cluster per iteration (k_resident) */
  SCG_SERIAL_RNG = 1u << 18,    /* one GPU: draw the next start vector with the full-grid kernel on the main stream
                                   (serial, no overlap with the Lanczos kernels) instead of the low-priority side
                                   stream; bitwise-neutral execution option */
  SCG_INLINE_PULL = 1u << 19    /* P > 1 (not with host-callback transports): pull each Lanczos step's omega / rho
                                   collective in the prologue of the kernel that consumes it instead of by a k_pull
                                   launch; bitwise-neutral execution option */
};

/* This rank's rows [row_begin, row_end) of the symmetric weighted Laplacian
 * L = sum_{ij in E} w_ij (e_i - e_j)(e_i - e_j)^T  (eqn:comb-laplacian).
 * Off-diagonal entries are L_ij = -w_ij (any sign: signed weights are accepted).
 * Columns must be strictly ascending within a row and global (0..n_global-1).  The pattern
 * must be symmetric (row-sharded runs derive the halo from it; an emulated-shard init
 * checks it and returns SCG_EINVAL, a multi-process rank cannot see the other rows). */
typedef struct {
  int64_t n_global;
  int64_t row_begin, row_end;
  const int64_t *row_ptr;   /* host, (row_end-row_begin)+1 offsets into col_idx / val */
  const int32_t *col_idx;   /* host, global column ids */
  const double *val;        /* host, L entries */
  int32_t has_diagonal;     /* 1: the diagonal entries L_rr are present (used as given);
                               0: absent, L_rr = -sum_j L_rj is formed */
} scg_csr;

/* Row-sharded execution.  The rows of
 * L and every row-indexed state vector (z, y, d, S, Omega, ...) are split into
 * `world` contiguous blocks [row_splits[p], row_splits[p+1]).  Each Lanczos matvec
 * needs the halo entries of the vector being multiplied: the producing kernel stores
 * them straight into the reader ranks' memory (NVLink peer stores), and the exact
 * global sums (CAC-2) combine through per-rank device mailboxes, so the iterates
 * are bitwise identical for every world size.  world <= 8.
 *
 *   emulate = 0: one process per rank (setup transport for the CUDA IPC handle exchange,
 *     the row-label exchange and the one-shot reconstruction reductions: NCCL, or the
 *     caller's scg_host_comm).  Every rank passes its own rows in scg_csr
 *     (row_begin = row_splits[rank], row_end = row_splits[rank+1]), the same row_splits
 *     (required when world > 1), and either host_comm or the same 128-byte NCCL unique
 *     id, created on rank 0 (sketchycgal_nccl_unique_id) and broadcast by the caller,
 *     e.g. through torch.distributed.
 *   emulate = 1: all `world` shards live in this one context on one device (peers are
 *     the other shards' buffers, no NCCL).  scg_csr holds ALL rows; row_splits may be
 *     NULL (balanced split, sketchycgal_row_splits).  Every per-row output of the
 *     context then covers all n rows.  This runs the sharded kernels on one GPU. */
/* Host-side transport for the setup and one-shot exchanges of a multi-process run (emulate = 0),
 * supplied by the caller (e.g. torch.distributed), instead of NCCL.  Every function is called
 * collectively by all ranks in the same order and returns 0 on success.
 *   allgather:     out (world * bytes, host) receives every rank's `in` (bytes, host) in rank order
 *   allreduce_sum: in-place sum of count doubles (host) over the ranks
 *   barrier:       returns once every rank has called it
 *   sync_collectives = 1: before each device-side collective (the mailbox pull of an exact sum or a
 *     halo barrier) the caller's stream is synchronized and the ranks meet in `barrier`, and the pull
 *     then only checks the peers' flags (an absent flag is an error, never a wait).  No kernel ever
 *     waits for another rank's kernel: ranks may share a GPU (tests), at the cost of one host round
 *     trip per collective.  0: the pulls wait on the device (one process per GPU). */
typedef struct {
  void *ctx;
  int32_t (*allgather)(void *ctx, const void *in, void *out, int64_t bytes);
  int32_t (*allreduce_sum)(void *ctx, double *buf, int64_t count);
  int32_t (*barrier)(void *ctx);
  int32_t sync_collectives;
} scg_host_comm;

typedef struct {
  int32_t rank, world;
  const void *nccl_unique_id;   /* host, 128 bytes (emulate = 0 without host_comm) */
  const int64_t *row_splits;    /* host, world + 1 ascending offsets, [0] = 0, [world] = n; may be NULL if emulate */
  int32_t emulate;
  const scg_host_comm *host_comm; /* emulate = 0: setup transport; NULL = NCCL (nccl_unique_id required) */
} scg_dist;

/* One record per iteration t (Alg. 4), original units where noted. */
typedef struct {
  int64_t t;          /* iteration index, 1-based */
  int32_t q;          /* Lanczos bound min(q_t, n-1), q_t = ceil(t^(1/4) ln n) */
  int32_t k;          /* Lanczos steps taken (< q on invariant-subspace break, Alg. 2 line 8) */
  double theta;       /* Ritz value: min eigenvalue of the Lanczos tridiagonal (Alg. 2 line 12), scaled units */
  double xi;          /* Rayleigh quotient v^T D_t v (eqn 5.1), scaled units */
  double c;           /* v^T C v, scaled units */
  double p;           /* objective tracker p_{t+1} = <C, X_{t+1}>, scaled units */
  double znorm;       /* ||z_{t+1} - b||, scaled units */
  double gamma;       /* dual step gamma_t (eqn:sketchy-cgal-dual-step) */
  double tau;         /* trace tracker tau */
  double gap;         /* surrogate duality gap g_t(X_t) with lambda_min(D_t) ~ xi_t (eqn:cgal-gap,
                         PAPER.md:1550-1555), scaled units, state before the update of iteration t;
                         box sets K: b replaced by the slack w_t (reading R33) */
  double bound;       /* posterior suboptimality bound of X_t, = the stopping numerator
                         p_t + <y_t, b> + beta_t/2 <z_t - b, z_t + b> - alpha xi_t
                         (PAPER.md:1557-1562, 4044-4048), scaled units */
} scg_iter_rec;

/* Per-kernel-class timing (SCG_PROFILE), for bench.py's roofline. */
typedef struct {
  char name[32];
  int64_t launches;
  double total_ms;          /* CUDA-event time on the context stream: every 16th launch of the class is
                               timed, the sum extrapolated to all launches */
  double bytes_per_launch;  /* algorithmic HBM bytes of one launch */
} scg_kstat;

/* Create a context: copy this rank's CSR to the device, form C = -L (scaled by
 * 1/||L||_F when SCG_SCALE), draw Omega (n x R standard normal, Alg. 3 line 2,
 * PAPER.md:1228) from the seeded stream, set z = y = 0, S = 0 (Alg. 4 lines 3-4).
 *   alpha: trace bound in ORIGINAL units (n for MaxCut); beta0: initial smoothing
 *   (1 by default); seed: stream seed for Omega and the Lanczos
 *   start vectors; device: CUDA device ordinal; cuda_stream: optional
 *   cudaStream_t to run on (NULL: the context creates its own).
 * Errors: SCG_EINVAL, SCG_ENOMEM, SCG_ECUDA, SCG_ENCCL.  *out is NULL on error. */
scg_status sketchycgal_maxcut_init(scg_ctx **out, const scg_csr *L, int32_t R, double alpha, double beta0,
                                   uint64_t seed, uint32_t flags, const scg_dist *dist, int32_t device,
                                   void *cuda_stream);

/* Advance T iterations (t continues across calls).  Asynchronous on the context
 * stream; returns after enqueueing and checking launch errors.  Device-side
 * range errors surface at the next synchronizing call as SCG_ERANGE. */
scg_status sketchycgal_step(scg_ctx *c, int64_t T);

/* Run up to T_max more iterations and stop at the first iteration t that meets the
 * stopping rule of PAPER.md:4044-4048, in ORIGINAL units (p, bound times ||L||_F n,
 * z times n when SCG_SCALE; b = 1):
 *   bound_t / (1 + |p_t|) <= eps   and   ||z_t - b|| / (1 + ||b||) <= eps,
 * with bound_t the posterior suboptimality bound of the record (lambda_min(D_t) ~ xi_t,
 * as the paper's own implementation does) and p_t, z_t the state before
 * iteration t's update.  The rule is checked on the iteration records every
 * check_every iterations, so up to check_every - 1 iterations past t may have run
 * (sketchycgal_iterations tells).  *t_stop = t, or -1 if T_max iterations ran without
 * meeting the rule.  Errors: SCG_EINVAL (T_max < 0, eps <= 0, check_every < 1). */
scg_status sketchycgal_run(scg_ctx *c, int64_t T_max, double eps, int64_t check_every, int64_t *t_stop);

/* Standard-form driver (Remark "Standard-form SDP"): a sequence of
 * trace-bounded SDPs tr X <= alpha_i (SCG_TRACE_LE forced) with
 * alpha_0 = alpha0 and alpha_{i+1} = 2 alpha_i, each solved from scratch for T iterations, until
 * the implicit objective tr(L X_T) of round i equals round i-1's: |o_i - o_{i-1}| <= rtol |o_i|
 * (the paper's "=" for approximate solutions, reading R31), or max_rounds rounds.
 *   out:       the context of the last round (caller destroys; reconstruct / round / ... apply)
 *   L, R, beta0, seed, flags, device, cuda_stream: as sketchycgal_maxcut_init (one GPU: no dist)
 *   alphas, objs: host arrays of max_rounds doubles: alpha_i and o_i of every round run
 *   rounds:    rounds run;  converged: 1 if the equality test stopped the sequence, else 0
 * Errors: SCG_EINVAL for alpha0 <= 0, T < 1, rtol < 0, max_rounds < 1 or NULL outputs; any
 * error of a round's init / step is returned with *out = NULL. */
scg_status sketchycgal_maxcut_alpha_doubling(scg_ctx **out, const scg_csr *L, int32_t R, double alpha0,
                                             double beta0, uint64_t seed, uint32_t flags, int32_t device,
                                             void *cuda_stream, int64_t T, double rtol, int32_t max_rounds,
                                             double *alphas, double *objs, int32_t *rounds, int32_t *converged);

/* Convex inclusion A X in K for the box K = {u : lo <= u_i <= hi} (general template,
 * PAPER.md:3909-3941; the l_inf ball |u - b| <= delta of P:3915-3918 is lo = 1 - delta,
 * hi = 1 + delta; lo = -INFINITY, hi = 1 is SCG_INEQ).  Original units (the MaxCut b is 1).
 * Call after init and before the first step (recomputes D_1's diagonal); SCG_EINVAL
 * otherwise, for NaN bounds, lo > hi or hi = -inf.  Reading R32: slack
 * w = min(max(z + y / beta, lo), hi); the gap / bound records use w in place of b (reading R33):
 * gap = p + <y,z> + beta <z-w,z> - alpha xi, bound = p + <y,w> + beta/2 <z-w,z+w> - alpha xi. */
scg_status sketchycgal_set_box(scg_ctx *c, double lo, double hi);

/* Convex inclusion A X in K for the l2 ball K = {u : ||u - b||_2 <= delta} (the norm constraint
 * ||A X - b|| <= delta of PAPER.md:3915-3918, general template P:3909-3941).  delta in original
 * units (the MaxCut b is 1; delta >= 0, finite).  Call after init and before the first step
 * (recomputes D_1's diagonal with the slack w_1); SCG_EINVAL otherwise.  Reading R34: the slack
 * w = proj_K(p), p = z + y / beta, is p when ||p - b|| <= delta, else b + s (p - b) with
 * s = delta / ||p - b||, the norm an exact sum over all ranks (each projection is one more
 * reduction per use: wbar_t before the dual step, w_{t+1} after it).  The gap / bound records use
 * w as in sketchycgal_set_box (reading R33).  Runs the multi-kernel path (no resident cluster
 * kernel) and draws the next Lanczos start vector inside the dual step. */
scg_status sketchycgal_set_ball(scg_ctx *c, double delta);

/* Convex inclusion A X in K for the l1 ball K = {u : ||u - b||_1 <= delta} (the norm constraint of
 * PAPER.md:3915-3918 with the l1 norm).  delta in original units, >= 0 and finite; call after init
 * and before the first step (SCG_EINVAL otherwise).  Reading R35: the slack w = proj_K(p) is p when
 * ||p - b||_1 <= delta, b when delta = 0, else the soft threshold w_r = b + sign(e_r) max(|e_r| -
 * theta, 0), e = p - b, theta = (S - delta) / c over the active set {|e_r| >= v*} (c entries, exact
 * sum S) whose least entry v* satisfies S(v) - c(v) v - delta < 0 -- found without a sort by a 63-step
 * bisection on the bit pattern of v, each step an exact-sum pass over all ranks.  Same execution
 * path and gap / bound records as sketchycgal_set_ball. */
scg_status sketchycgal_set_ball_l1(scg_ctx *c, double delta);

/* Fixed Lanczos bound: every later iteration runs Alg. 2 with q instead of the schedule
 * q_t = min(n - 1, max(2, ceil(t^(1/4) ln n))) (ApproxMinEvec takes q as an input, PAPER.md:1068-1086;
 * Fact 4.1, gives the q for a target accuracy).  q = 0 restores the schedule.
 * 1 <= q <= min(n, 255) (q = n spans the full Krylov space, SPEC-style exact checks).
 * Errors: SCG_EINVAL.  (sketchycgal_step returns SCG_EUNSUPPORTED instead of truncating when the
 * schedule's q_t exceeds the device bound 255: t > 47,000 iterations at n = 2^25.) */
scg_status sketchycgal_set_lanczos_q(scg_ctx *c, int32_t q);

/* Block until all queued work is done; reports deferred device errors. */
scg_status sketchycgal_synchronize(scg_ctx *c);

/* NystromSketch.Reconstruct (Alg. 3 lines 11-16; Alg. SM3
 * PAPER.md:3304-3317) followed by the optional trace correction (Alg. 4 line 13).
 *   U: host, n_local x R column-major (this rank's rows), orthonormal columns (may be NULL)
 *   Lambda: host, R, descending, ORIGINAL units (trace-corrected iff SCG_TRACE_CORRECT)
 *   err: host, R (may be NULL): err_r = tau - sum_{j<=r} Lambda_j, before correction.
 * The factor stays on the device for objective / feasibility / round. */
scg_status sketchycgal_reconstruct(scg_ctx *c, double *U, double *Lambda, double *err);

/* out[0] = tr(L X_t) of the implicit iterate from the tracked p;
 * out[1] = tr(L X^) of the reconstruction (needs reconstruct; NAN before).  Original units. */
scg_status sketchycgal_objective(scg_ctx *c, double out[2]);

/* out[0] = ||z - b|| / (1 + ||b||) of the implicit iterate;
 * out[1] = ||diag X^ - 1|| / ||1||;  out[2] = ||diag X^ - 1|| / (1 + ||1||).  Original units. */
scg_status sketchycgal_feasibility(scg_ctx *c, double out[3]);

/* Rounding: the best of the R sign cuts sgn(U[:,k]) (sgn(0)=+1,
 * ties -> lowest k), normalized so chi[0] = +1.  chi_local: host int8, n_local. */
scg_status sketchycgal_round(scg_ctx *c, int8_t *chi_local, double *cut_weight);

/* Copy iteration records t0..t0+count-1 (1-based t) into out. */
scg_status sketchycgal_iter_log(scg_ctx *c, int64_t t0, int64_t count, scg_iter_rec *out);

/* Test / diagnostics access to the state (this rank's rows).
 *   which: 0 z, 1 y, 2 S (n_local x R col-major), 3 Omega (same), 4 v (last eigenvector),
 *          5 d (diagonal of D for the NEXT iteration), 6 C diagonal (scaled). */
scg_status sketchycgal_get_state(scg_ctx *c, int32_t which, double *out);

/* Apply D_{t+1} = C + diag(d) (primitives 1+2, eqn:primitives PAPER.md:567-590) with
 * the same row-sum order as the Lanczos kernels: y = D x.  x: host, n_global; y: host, n_local. */
scg_status sketchycgal_apply_D(scg_ctx *c, const double *x, double *y);

/* Iterations done so far. */
int64_t sketchycgal_iterations(const scg_ctx *c);

/* Kernel launches issued since init / the last reset (counts only this library's kernels). */
int64_t sketchycgal_launch_count(const scg_ctx *c);

/* Kernel statistics (needs SCG_PROFILE): fills up to max entries, returns the count (<0 on error).
 * One entry per kernel class, plus "lanczos_pass1_in_flow" (one GPU, multi-kernel path): every 8th
 * iteration's whole Lanczos pass 1 (Alg. 2 lines 1-9) between ONE pair of events
 * with none between its launches; launches = passes timed, total_ms their summed time,
 * bytes_per_launch the mean algorithmic bytes of such a pass. */
int32_t sketchycgal_kernel_stats(scg_ctx *c, scg_kstat *out, int32_t max);
void sketchycgal_reset_stats(scg_ctx *c);

/* Balanced contiguous row split for `world` ranks: minimizes the largest per-rank
 * cost rows + nonzeros (row_ptr: host, n+1 offsets of the full CSR).  Host only (no
 * GPU needed).  splits: host, world + 1. */
scg_status sketchycgal_row_splits(const int64_t *row_ptr, int64_t n, int32_t world, int64_t *splits);

/* Halo plan of one shard (host only, no GPU needed): for each own row r in
 * [row_begin, row_end) of the symmetric L, mask[r - row_begin] = bitmask of the
 * OTHER ranks owning a column of row r -- by symmetry exactly the ranks that read
 * x_r in a matvec.  Returns the number of halo rows (mask != 0), < 0 on error.
 *   row_ptr/col_idx: this shard's rows as in scg_csr; splits: world + 1. */
int64_t sketchycgal_halo_plan(const int64_t *row_ptr, const int32_t *col_idx, int64_t row_begin, int64_t row_end,
                              const int64_t *splits, int32_t world, uint8_t *mask);

/* Write a 128-byte NCCL unique id (call on rank 0, broadcast to all ranks). */
scg_status sketchycgal_nccl_unique_id(void *out128);

/* Diagnostics: compare the kernels' shared-divisor division (a * RN(1/b) with two
 * fma corrections, used for the normalization v = w / rho of Alg. 2 line 9) with the
 * hardware IEEE division on n pseudo-random operand pairs; *mismatches = count. */
scg_status sketchycgal_selftest_division(int32_t device, int64_t n, uint64_t seed, int64_t *mismatches);

/* Exact-sum self-test (CAC-2): the n host values are copied to the device and
 * summed by a grid x block launch of the kernels' per-thread exact accumulators (fast fp64 bins,
 * spills, slow path, block and grid commits); *sum = xsum(values) rounded once, *range_error = 1 if
 * a value was non-finite or >= 2^100 in magnitude.  block a multiple of 32 in [32, 1024], grid >= 1.
 * Test access only (no context). */
scg_status sketchycgal_selftest_xsum(int32_t device, const double *values, int64_t n, int32_t grid, int32_t block,
                                     double *sum, int32_t *range_error);

const char *sketchycgal_last_error(const scg_ctx *c);
void sketchycgal_destroy(scg_ctx *c);

#ifdef __cplusplus
}
#endif
#endif /* SKETCHYCGAL_H */
