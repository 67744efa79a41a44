/*
 * duquad.h -- C ABI of the B200-native DuQuad hot path (arXiv 1504.05708).
 *
 * Solves   min_{u in U} F(u) = 1/2 u'Qu + q'u   s.t.  G u + g in K
 * (Eq. original_primal) with U = [lb, ub] a box and K a
 * product of per-row cones: ZERO ({0}, equality) or NONPOS (R_-, inequality),
 * by the inexact (augmented) dual gradient / dual fast gradient methods
 * DGM / DFGM (Algorithm DFOM) whose inner problem
 * (Eq. ul) is solved by Algorithm FOM
 * with a fixed number of inner iterations, warm-started.
 *
 * Every step of the path runs in this library's sm_100a kernels; the caller
 * only marshals arguments.  All floating point is IEEE binary64.
 *
 * Conventions for every entry point:
 *   - returns a duquad_status; no exception or abort crosses the ABI; a
 *     non-OK status stores a message retrievable with duquad_last_error();
 *   - "device pointer" = a pointer into global memory of the context's
 *     CUDA device; "host pointer" = ordinary (pageable or pinned) memory;
 *   - arrays are dense row-major unless stated otherwise;
 *   - the library never retains caller pointers after a call returns
 *     (except the trace buffers registered with duquad_set_trace).
 * One context per host thread; calls on one context are not reentrant.
 */
#ifndef DUQUAD_H
#define DUQUAD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DUQUAD_ABI_VERSION 4   /* 2: options gained eq_precompute, checkpoint, dual_average;
                                  3: nccl_self; 4: sell_path, duquad_theory_schedule's
                                  lambda_max_Q */

typedef enum {
    DUQUAD_OK = 0,
    DUQUAD_EINVAL = 1,      /* bad argument: dims, NaN in data, lb > ub, rho < 0, ...      */
    DUQUAD_ENOMEM = 2,      /* device or host allocation failed                           */
    DUQUAD_ECUDA = 3,       /* CUDA runtime error (message has the CUDA error string)     */
    DUQUAD_ENCCL = 4,       /* NCCL error in the sharded path                             */
    DUQUAD_ENONFINITE = 5,  /* an iterate became non-finite; results kept  */
    DUQUAD_ENODEV = 6,      /* no CUDA device, or not an sm_100 device                    */
    DUQUAD_ESTATE = 7,      /* call out of order (e.g. solve before constants are set)    */
    DUQUAD_EMAXITER = 8     /* eps_in mode: an inner solve hit inner_max first; the result
                               and the inner-step counts are still populated              */
} duquad_status;

typedef enum { DUQUAD_DGM = 0, DUQUAD_DFGM = 1 } duquad_alg;

typedef enum {
    DUQUAD_INNER_FGM = 0,       /* theta recurrence, restarted at every inner solve (default) */
    DUQUAD_INNER_GM = 1,        /* beta = 0                                                  */
    DUQUAD_INNER_FGM_SIGMA = 2  /* beta = (sqrt L - sqrt sigma)/(sqrt L + sqrt sigma)        */
} duquad_inner;

typedef enum { DUQUAD_DENSE = 0, DUQUAD_CSR = 1 } duquad_format;

enum { DUQUAD_CONE_ZERO = 0, DUQUAD_CONE_NONPOS = 1 };

typedef struct duquad_ctx duquad_ctx;

/*
 * Problem data.  Single QP (batch == 1):
 *   Q   n x n, symmetric positive (semi)definite; Q's symmetry is checked
 *       at setup on every path and rank count (EINVAL unless |Q_ij - Q_ji| <= 1e-12 (|Q_ij| +
 *       |Q_ji|)), because the byte-floor and small-QP kernels read Q through its symmetry (a
 *       row-sharded rank checks the caller's full Q; CSR: Q and its transpose must have the same
 *       pattern, i.e. both triangles stored, and the same values);
 *   G   p x n;  q n;  g p;  lb, ub n (entries may be -INFINITY / +INFINITY);
 *   cone p tags (DUQUAD_CONE_*), or NULL meaning every row is cone_all.
 * Batched (batch = B > 1, dense only; north_star (c)): Q and G are shared,
 *   q is B x n and g is B x p (row b belongs to QP b).
 * Dense: Q has leading dimension ldQ >= n, G has ldG >= n.
 * CSR (format == DUQUAD_CSR, batch == 1): int32 row pointers (rows+1),
 *   int32 column indices (sorted within a row), fp64 values, for Q (n rows)
 *   and G (p rows); the dense pointers are ignored.
 * on_device: 1 if every pointer is a device pointer, 0 if host.  With device inputs setup
 *   first synchronizes the device (inputs may be produced on any stream).
 * Ownership: duquad_setup copies/repacks everything into library-owned
 *   device memory; the caller may free its arrays when setup returns.
 */
typedef struct {
    int64_t n, p, batch;
    int32_t format;
    int32_t on_device;
    const double *Q;
    int64_t ldQ;
    const double *G;
    int64_t ldG;
    const int32_t *Q_rowptr, *Q_col;
    const double *Q_val;
    int64_t Q_nnz;
    const int32_t *G_rowptr, *G_col;
    const double *G_val;
    int64_t G_nnz;
    const double *q, *g, *lb, *ub;
    const uint8_t *cone;
    int32_t cone_all;
} duquad_problem;

/*
 * Solver options (fill with duquad_default_options, then override).
 *   dual_step_scale  dual step = dual_step_scale / L_d; 0.5 is the paper's
 *                    1/(2 L_d) (reading c1).
 *   project_dual     1: project NONPOS multipliers onto R_+ (K_d, PAPER.md:295-296,
 *                    reading c3); 0: K_d = R^p.  ZERO rows are never projected.
 *   inner_rule       duquad_inner; sigma used by FGM_SIGMA only (must be > 0).
 *   lambda_min_lb    lower bound on lambda_min(Q) used in L_d (Eq. Ld);
 *                    must be > 0 when rho == 0 (reading c13).
 *   l_mode           0: L_in = lambda_max(Q + rho G'G) (north_star);
 *                    1: L_in = lambda_max(Q) + rho ||G||^2.
 *   use_graphs       1: capture one outer iteration as a CUDA graph (default 1).
 *   world_size/rank  row sharding of [Q;G] and G' over world_size GPUs (one
 *                    process per GPU); nccl_id = 128-byte ncclUniqueId shared by
 *                    all ranks (see duquad_nccl_unique_id).  1 / 0 = single GPU.
 *   stream           cudaStream_t the context runs on; NULL = a library stream.
 *   device           CUDA device ordinal; -1 = the calling thread's current device.
 */
typedef struct {
    double dual_step_scale;
    int32_t project_dual;
    int32_t inner_rule;
    double sigma;
    double lambda_min_lb;
    int32_t l_mode;
    int32_t use_graphs;
    int32_t world_size;
    int32_t rank;
    const void *nccl_id;
    void *stream;
    int32_t device;
    int32_t time_passes;   /* 1: time a sample of pass A / pass B launches with CUDA events */
    int32_t small_path;    /* 1 (default): run the whole solve in ONE single-CTA kernel when
                              [Q;G], G' and the vectors fit in shared memory (single GPU,
                              dense, batch 1); 0: always use the streaming pass kernels    */
    int32_t rho0_path;     /* 1 (default): with rho == 0 (dense, batch 1) stream only Q per inner
                              step, c = q + G'mu formed once per outer iteration;
                              0: the generic two-pass inner step                           */
    int32_t emulate_ranks; /* testing: with world_size > 1, no NCCL communicator is created; the
                              world_size contexts (one per rank, same device and stream) are
                              driven together by duquad_solve_emulated, whose all-gathers are
                              device copies -- the sharded kernels and index math on 1 GPU  */
    int32_t fused_path;    /* 1 (default): for large dense QPs on one GPU (n >= 4096), the
                              byte-floor inner step: one streaming kernel reads the upper
                              triangle of the symmetric Q once and G once (CTA pairs exchange
                              row sums through distributed shared memory), 8(n(n+1)/2 + pn)
                              bytes instead of 8(n^2 + 2pn); 0: the two-pass inner step    */
    int32_t persist_path;  /* 1: dense single-GPU QPs whose matrices fit in 100 MB (L2) run every
                              inner step of a solve in ONE cooperative launch (two passes
                              separated by grid barriers; bitwise the multi-launch result).
                              0 (default): one launch per pass in a CUDA graph -- measured as
                              fast or faster on config 1 (the passes are L2-latency bound)  */
    int32_t eq_precompute; /* 1 (default): a dense single-GPU QP whose rows are all equalities
                              (K = {0}) with rho > 0 forms H = Q + rho G'G once at setup (cuBLAS
                              DGEMM, 2 n^2 p flops; n x n more device memory) and runs every inner
                              step on H alone, grad = H u + c with c = q + G'(mu + rho g) once per
                              outer iteration: 8 n(n+1)/2 bytes
                              per step on the byte-floor path instead of 8 (n(n+1)/2 + pn).
                              0: the generic inner step                                      */
    int32_t checkpoint;    /* 1: every solve snapshots its state after outer iteration K (before the
                              last-iterate solve) for duquad_get_state; the single-CTA and
                              persistent kernels defer to the streaming path.  0 (default)   */
    int32_t dual_average;  /* 1 (DGM only; EINVAL with DFGM or in eps_in mode): the final dual point
                              is lambda^K := [lam_hat + grad_bar d(lam_hat) / (2 L_d)]_{K_d} with the
                              average lam_hat = (1/(K+1)) sum_{j=0}^{K} lambda^j (PAPER.md:624-626,
                              the DGM rate of Theorem 1 holds for it); x_last = u_bar(lambda^K).
                              Costs one more inner solve (at lam_hat); the single-CTA and
                              persistent kernels defer to the streaming path.  0 (default): the
                              last dual iterate.                                             */
    int32_t nccl_self;     /* 1 (world_size 1, not batched): run the ROW-SHARDED code path (its
                              kernels, NCCL all-gathers / reduce-scatter / broadcasts /
                              all-reduce, their CUDA-graph capture) on a one-rank NCCL
                              communicator the library creates itself (nccl_id ignored): the
                              collective call sequence of a P-GPU run, exercised on one GPU.
                              Results agree with the oracle like any solve.  0 (default)      */
    int32_t sell_path;     /* 1 (default): a CSR matrix whose rows are short (mean <= 48 nonzeros)
                              runs lane-per-row kernels: SELL-32 (slices of 32 rows, the k-th
                              nonzeros of a slice in one coalesced 32-wide column; an extra
                              copy of the matrix) when that pads at most 15 %, else
                              thread-per-row CSR.  Both sum each row in CSR order.  0: the
                              sub-warp CSR kernels (a group of lanes per row, tree sums)      */
    int32_t pair_rows;     /* 1 (default): a batched QP whose constraint rows come in +/- pairs,
                              G = [G_t; -G_t] (two-sided bounds, e.g. config 3's |x_k| <= 5),
                              streams [Q; G_t] in pass A (the bottom rows' product is -(G_t y),
                              exactly) and forms G'w as G_t'(w_top - w_bottom) in pass B: half the
                              G work, the same step.  0: the unpaired matrices             */
    int32_t pdl;           /* 1 (default): the dense inner-step kernels are launched with
                              programmatic dependent launch -- a kernel's launch overlaps its
                              predecessor's tail; it reads and writes iterates only after its
                              dependency wait (same results).  CSR contexts launch plainly
                              (measured slower with it).  0: plain launches                  */
} duquad_options;

/* Per-solve report. */
typedef struct {
    int64_t outer_iters;        /* K_out executed                                         */
    int64_t inner_iters_total;  /* (K_out + 1) * K_in  (incl. the last-iterate solve)     */
    int64_t kernel_launches;    /* this library's kernels launched by the solve           */
    int64_t matrix_passes;      /* full passes over a stored matrix (matvec counter)      */
    double ms_device;           /* device time of the whole solve (CUDA events)           */
    double ms_pass_a;           /* mean duration of a sampled pass-A launch (time_passes) */
    double ms_pass_b;           /* mean duration of a sampled pass-B launch (time_passes) */
    int64_t n_timed_a, n_timed_b;
    double bytes_pass_a;        /* algorithmic bytes per pass-A launch (matrix + vectors) */
    double bytes_pass_b;        /* algorithmic bytes per pass-B launch                    */
    double flops_pass_a;        /* algorithmic flops per pass-A launch (2 per multiply-add) */
    double flops_pass_b;
    int32_t path;               /* duquad_path: which kernels ran the inner steps           */
    int32_t sparse_kernels;     /* CSR: pass A kind | pass B kind << 4, kind 0 = sub-warp CSR,
                                   1 = SELL-32, 2 = thread-per-row CSR (options.sell_path);
                                   + 8: pass A reads the banded Q rows as diagonals (DIA);
                                   + 64: only the band's upper half is stored and streamed
                                   (symmetric DIA; the lower entries re-read from it)         */
} duquad_result;

/* Kernel path of a solve (duquad_result.path).  "pass A" / "pass B" in the report map to:
 *   TWO_PASS   k_pass_a ([Q;G] y, w) / k_pass_b (G'w, projection, momentum)
 *   BYTE_FLOOR k_fused_stream (Q triangle + G once) / k_fused_epi (column sums, epilogue)
 *   RHO0       k_rho0_step (Q y + c) / -            RHO0_FLOOR k_fused_stream (Q only) / k_fused_epi
 *   BATCHED    DMMA pass 0 / pass 1                 CSR        k_pass_a_csr / k_pass_b_csr
 *   EQ_H       equality QP (all rows ZERO), rho > 0: k_rho0_step on H = Q + rho G'G (formed once,
 *              cuBLAS DGEMM) with c = q + G'(mu + rho g) per outer iteration
 *   EQ_H_FLOOR the same with k_fused_stream over the upper triangle of H
 *   SMALL      the whole solve in one single-CTA kernel (no per-pass timing)
 *   PERSIST    both passes of every inner step in one cooperative launch (no per-pass timing) */
typedef enum {
    DUQUAD_PATH_TWO_PASS = 0,
    DUQUAD_PATH_BYTE_FLOOR = 1,
    DUQUAD_PATH_RHO0 = 2,
    DUQUAD_PATH_RHO0_FLOOR = 3,
    DUQUAD_PATH_BATCHED = 4,
    DUQUAD_PATH_CSR = 5,
    DUQUAD_PATH_SMALL = 6,
    DUQUAD_PATH_PERSIST = 7,    /* k_persist: the two passes of every inner step in one cooperative
                                   launch (L2-resident dense QPs, e.g. config 1)              */
    DUQUAD_PATH_EQ_H = 8,
    DUQUAD_PATH_EQ_H_FLOOR = 9
} duquad_path;

int32_t duquad_abi_version(void);
/* sizeof of the ABI structs, for bindings to check their mirrors: which = 0 duquad_problem,
 * 1 duquad_options, 2 duquad_result, 3 duquad_schedule, 4 duquad_bounds, 5 duquad_monitor;
 * -1 for an unknown `which`.  Host only. */
int64_t duquad_struct_size(int32_t which);
const char *duquad_status_string(int32_t status);
void duquad_default_options(duquad_options *opts);

/*
 * Rows [*begin, *end) of a `rows`-row matrix owned by `rank` of `world`
 * (contiguous slices of ceil(rows/world) rows; the last may be short or
 * empty).  Host-only arithmetic, callable without a GPU.
 */
duquad_status duquad_shard_range(int64_t rows, int32_t world, int32_t rank,
                                 int64_t *begin, int64_t *end);

/* Writes a fresh 128-byte ncclUniqueId into out128 (call on rank 0 only). */
duquad_status duquad_nccl_unique_id(void *out128);

/*
 * Validates the problem (dims, finiteness, lb <= ub, rho >= 0) and builds a
 * context: packs [Q;G] row-major with a 256-byte aligned leading dimension,
 * stores G' separately (transposed on the device), uploads q, g, lb, ub,
 * cone tags; sharded mode keeps only this rank's rows and creates the NCCL
 * communicator.  *out is NULL on failure.
 */
duquad_status duquad_setup(duquad_ctx **out, const duquad_problem *prob, double rho,
                           const duquad_options *opts);

/*
 * Lipschitz constants on the device (north_star (a)); Lanczos with
 * `iters` steps for lambda_max(Q + rho G'G) (l_mode 0) or lambda_max(Q)
 * (l_mode 1) and for ||G||^2 = lambda_max(G'G).  Lanczos returns Ritz values,
 * which never exceed the true eigenvalues, so `safety` >= 0 inflates both
 * estimates (recommended 1e-6, SPEC.md:76's delta_safe; the Python binding's
 * default) and both constants come out as over-estimates:
 *   L_in = (1 + safety) * estimate,
 *   L_d  = nG2' / (lambda_min_lb + rho nG2'),  nG2' = (1 + safety) ||G||^2
 * (Eq. Ld; L_d is increasing in ||G||^2).  Stores them in the
 * context (as duquad_set_constants would) and returns them in the host scalars
 * (any may be NULL); *normG2 is the raw (uninflated) estimate.
 * DUQUAD_EINVAL: safety < 0, or rho == 0 with lambda_min_lb <= 0 and p > 0.
 */
duquad_status duquad_lipschitz(duquad_ctx *ctx, int32_t iters, double safety,
                               double *L_in, double *L_d, double *normG2);

/* Injects L_in > 0 and L_d >= 0 (parity tests pass identical constants to the oracle). */
duquad_status duquad_set_constants(duquad_ctx *ctx, double L_in, double L_d);

/*
 * Runs Algorithm DFOM with `alg`, `outer_iters` >= 1
 * outer iterations of `inner_iters` >= 1 inner FOM steps each, from
 * lambda^0 = mu^1 = 0 and u_bar^0 = [0]_U, then one more inner solve at
 * lambda^K for the last primal iterate (Eq. last_primal).
 * Results stay on the device (duquad_get_result).  `res` may be NULL.
 * Returns DUQUAD_ENONFINITE if an iterate became NaN/Inf.
 */
duquad_status duquad_solve(duquad_ctx *ctx, int32_t alg, int32_t outer_iters,
                           int32_t inner_iters, duquad_result *res);

/*
 * Warm start (sequential / receding-horizon solves): subsequent solves start
 * from u_bar^0 = [x0]_U instead of [0]_U (reading c7) and lambda^0 = mu^1 = lambda0 instead of 0
 * ("Given lambda^0 = mu^1 in K_d": lambda0 must lie in K_d, i.e. >= 0 on NONPOS rows when
 * project_dual).  x0 is n (batch: B x n, one row per QP), lambda0 is p (B x p), full vectors as
 * passed to duquad_setup; each context takes its QPs / row slices.  Host or device memory per
 * `on_device`.  NULL for either resets that one to the default.  Stays in effect until reset.
 */
/* With on_device = 1 the call first synchronizes the device (cudaDeviceSynchronize), so buffers
 * still being written on any stream (e.g. torch's current stream) are complete before the copy. */
duquad_status duquad_set_initial(duquad_ctx *ctx, const double *x0, const double *lambda0, int32_t on_device);

/*
 * DFOM with eps_in-driven inner stopping (Eq. duquad_in).
 * Every inner FGM solve runs until the gradient-map test
 *     L_in * ||y^k - x^k|| <= sqrt(2 * sigma_L * eps_in)
 * holds, x^k = [y^k - grad/L_in]_U the step's projected point, or `inner_max` steps ran.  For a
 * sigma_L-strongly convex L_rho(., mu) the test guarantees L_rho(x^k, mu) - d_rho(mu) <= eps_in
 * (the inexactness (duquad_in) of Theorem 1).  sigma_L > 0 is the caller's lower bound on
 * lambda_min(Q + rho G'G) (e.g. lambda_min(Q)), eps_in > 0 (e.g. from duquad_theory_schedule).
 * The norm is a fixed-order device reduction after each step; converged inner solves skip the
 * remaining steps of their (graph-captured) loop.  Any format; row-sharded groups all-reduce
 * the test's sum (one double per inner step), so every rank decides alike; a batch decides per
 * QP (stopped QPs are left untouched by the remaining steps, whose kernels exit once every QP
 * stopped) and reports counts QP-major, [QP][solve].
 * Returns DUQUAD_EMAXITER (result valid) when some inner solve was capped; per-outer step
 * counts via duquad_get_inner_counts.  res->inner_iters_total = steps actually run (summed over
 * the QPs of a batch).
 */
duquad_status duquad_solve_eps(duquad_ctx *ctx, int32_t alg, int32_t outer_iters, int32_t inner_max,
                               double eps_in, double sigma_L, duquad_result *res);

/*
 * Per-outer inner-step counts of the last duquad_solve_eps (K_out + 1 entries: the outer
 * iterations, then the last-iterate solve) and whether each met the eps_in test (1) or was
 * capped (0).  Either output may be NULL; copies min(max_entries, K_out + 1) entries.
 */
duquad_status duquad_get_inner_counts(duquad_ctx *ctx, int32_t *counts, int32_t *converged,
                                      int32_t max_entries);

/* Theory schedule of DuQuad for a target accuracy eps (host-only arithmetic, no GPU). */
typedef struct {
    double eps_in;      /* (choose_ein) PAPER.md:641-647: eps/4 (DGM), eps^1.5/(8 R_d sqrt(2 L_d)) (DFGM) */
    int64_t k_out;      /* (choose_ein): ceil(8 L_d R_d^2 / eps) (DGM), ceil(sqrt(8 L_d R_d^2 / eps)) (DFGM)  */
    int64_t k_in;       /* proof of Theorem in:th_last, rounded up:
                           sqrt(2 L D_U^2 / eps_in) (sigma_L = 0),
                           sqrt(L / sigma_L) log(L D_U^2 / eps_in) + 1 (sigma_L > 0)              */
    double rho_star;    /* 8 R_d^2 / eps (Theorem in:th_last)            */
    int64_t k_total;    /* Theorem in:th_last, PAPER.md:1162-1169 (floor):
                           24 ||G|| D_U R_d / eps (sigma_L = 0),
                           16 ||G|| R_d / sqrt(sigma_L eps) log(8 ||G|| D_U R_d / eps) (sigma_L > 0) */
    int32_t case_id;    /* 1 (Q > 0, rho = 0) iff lambda_min(Q) > tau_pd =
                           1e-7 max(1, lambda_max(Q)) (SPEC.md:186's threshold), else 2 (rho > 0) */
    int32_t reserved;
} duquad_schedule;

/*
 * Fills `out` from the algorithm (DUQUAD_DGM/DFGM), the target accuracy eps > 0, the dual
 * radius R_d = ||lambda*|| > 0 (an estimate), L_d > 0, the inner Lipschitz constant L_in > 0,
 * sigma_L >= 0, the box diameter D_U > 0, ||G|| >= 0, an estimate lambda_min_Q >= 0 of
 * lambda_min(Q) and lambda_max_Q >= 0 of lambda_max(Q) (0 if unknown: tau_pd = 1e-7).
 * Counts are clamped to [0, 2^62]; k_total's log argument to >= 1 (so ||G|| = 0 gives 0).
 * DUQUAD_EINVAL on a non-finite or out-of-range argument.  Pure host arithmetic.
 */
duquad_status duquad_theory_schedule(int32_t alg, double eps, double R_d, double L_d, double L_in,
                                     double sigma_L, double D_U, double normG, double lambda_min_Q,
                                     double lambda_max_Q, duquad_schedule *out);

/*
 * State export / resume (the DFOM state of PAPER.md:564-589 after outer iteration
 * j): x = u_bar^j (n, or B x n), mu = mu^j and lam_prev = lambda^{j-1} (p, or B x p, the two
 * points the next DFOM step reads), x_avg = the running primal average with
 * S = sum_{i<=j} omega_i, and j = outer_done.
 *   duquad_get_state: the snapshot the last solve took (options.checkpoint = 1), i.e. after its
 *     K-th outer iteration, before the last-iterate solve; DUQUAD_ESTATE if there is none.
 *   duquad_set_state: the next duquad_solve(alg, K, ...) continues with outer iterations
 *     j+1 .. j+K (theta, beta_out and the average weights continue; warm start ignored), so
 *     solve(K1) + get_state + set_state + solve(K2) equals solve(K1 + K2) bit for bit.
 * Buffers are host or device per on_device (layout as duquad_get_result: a row-sharded rank
 * exports and imports its own slices); fixed inner counts, no dual_average.  With on_device = 1,
 * set_state first synchronizes the device (inputs in flight on another stream are complete) and
 * get_state returns after its copies completed.  DUQUAD_EINVAL on bad arguments.
 */
duquad_status duquad_get_state(duquad_ctx *ctx, double *x, double *mu, double *lam_prev, double *x_avg,
                               int64_t *outer_done, double *S, int32_t on_device);
duquad_status duquad_set_state(duquad_ctx *ctx, const double *x, const double *mu, const double *lam_prev,
                               const double *x_avg, int64_t outer_done, double S, int32_t on_device);

/*
 * This context's rows: Q rows [r0, r0 + nloc) and constraint rows [s0, s0 + ploc) of the global
 * problem (the slices duquad_get_result returns for a row-sharded context; a batched context
 * reports the whole QP).  The constraint rows are equal slices except on the row-sharded
 * byte-floor path (dense, rho > 0, n >= 4096), where they are balanced against the ranks' Q
 * triangle slabs.  Any output pointer may be NULL.
 */
duquad_status duquad_local_ranges(const duquad_ctx *ctx, int64_t *r0, int64_t *nloc, int64_t *s0, int64_t *ploc);

/* Convergence-bound diagnostics of DuQuad (host-only arithmetic, no GPU), for k outer iterations. */
typedef struct {
    double dual_gap;    /* Theorem 1 (bound_gen_dfg): F* - d(lambda^k) <=
                           4 L_d R_d^2 / (k+1)^p + 2 (k+1)^(p-1) eps_in, p = 1 (DGM), 2 (DFGM)        */
    double drift;       /* (bound_seq_dgm) PAPER.md:736-738: ||lambda^k - lambda*|| <= R_d + sqrt(k eps_in / L_d) */
    double feas_last;   /* (aux_feas_bound) PAPER.md:805-810: dist_K(G x_last + g) <=
                           sqrt(2 L_d eps_in) + sqrt(2 L_d dual_gap)                                 */
    double feas_avg;    /* primal average over k iterates: DGM (feasibility_final) PAPER.md:918-939
                           4 L_d R_d / k + 2 sqrt(L_d eps_in / k); DFGM (infes_av) PAPER.md:1045-1056
                           8 L_d R_d / k^2 + 8 sqrt(L_d eps_in / k)                                  */
} duquad_bounds;

/*
 * Fills `out` for alg (DUQUAD_DGM/DFGM), k >= 1 outer iterations, L_d > 0, the dual radius
 * R_d = ||lambda* - lambda^0|| >= 0 and the inner accuracy eps_in >= 0 (reading c23 for
 * the iterate indexing).  DUQUAD_EINVAL on a non-finite or out-of-range argument.
 */
duquad_status duquad_theory_bounds(int32_t alg, int64_t k, double L_d, double R_d, double eps_in,
                                   duquad_bounds *out);

/*
 * Copies x_last = u_bar(lambda^K) (n, or B x n), x_avg (Eq. average_primal,
 * PAPER.md:700-706) and lambda^K (p, or B x p) into caller buffers (host or
 * device per `on_device`; any may be NULL).  Sharded: each rank copies its
 * local row slice (rows from duquad_shard_range).
 */
duquad_status duquad_get_result(duquad_ctx *ctx, double *x_last, double *x_avg, double *lambda,
                                int32_t on_device);

/*
 * Registers DEVICE buffers that the next solves fill with the per-outer
 * trace: lam_trace[(j-1)*p + i] = lambda^j_i and u_trace[(j-1)*n + i] = u_bar^j_i
 * for j = 1..min(K_out, max_outer) (local slices when sharded).  NULL
 * disables.  Tracing disables graph capture.  Not supported for batch > 1.
 */
duquad_status duquad_set_trace(duquad_ctx *ctx, double *lam_trace, double *u_trace,
                               int64_t max_outer);

/*
 * Stopping residuals (§8(a) a8) of x_last (which = 0) or x_avg (which = 1),
 * computed on the device with fixed-order reductions:
 *   F = 1/2 x'Qx + q'x,  dist = ||Gx + g - [Gx + g]_K||,
 *   lag = L_rho(x, lambda^K) by (auglag1) (an upper estimate of
 *         d_rho(lambda^K) = min_u L_rho(u, lambda^K) when x = u_bar(lambda^K)).
 * Single QP only.  Any output pointer may be NULL.
 */
duquad_status duquad_residuals(duquad_ctx *ctx, int32_t which, double *F, double *dist,
                               double *lag);

/* Report of duquad_solve_monitored. */
typedef struct {
    int64_t outer_done;    /* outer iterations of the returned iterates (a multiple of check_every,
                              or outer_max)                                                   */
    int64_t inner_total;   /* inner iterations executed, all segments (incl. their last-iterate
                              solves)                                                          */
    int64_t passes_total;  /* matrix passes executed, all segments                            */
    int32_t checks;        /* residual checks made                                            */
    int32_t converged;     /* 1: the stopping test held at outer_done                          */
    double F, dist;        /* F and dist_K of the checked iterate at outer_done                */
    double dual;           /* L_rho(x_last, lambda^j) = the inexact dual value d_bar(lambda^j)  */
} duquad_monitor;

/*
 * Stopping residuals every T outer iterations (§8(a) a8; the paper's stopping test, P:415-423,
 * P:1372-1378): runs DFOM in segments of check_every = T outer iterations.  After
 * each segment, duquad_residuals of x_last = u_bar(lambda^j) and of x_avg; the checked iterate
 * is which = 0 (x_last) or 1 (x_avg), and the solve stops at the first checked j with
 *     dist_K(Gx + g) <= eps  and  |F(x) - F_star| <= eps                     (F_star finite:
 *                                                     the paper's test with a known optimum), or
 *     dist_K(Gx + g) <= eps  and  |F(x) - d_bar(lambda^j)| <= eps (1 + |F(x)|)   (F_star = NaN:
 *         no reference value; d_bar(lambda^j) = L_rho(u_bar(lambda^j), lambda^j), the inexact dual
 *         value, so this is a primal-dual gap test -- reading c24),
 * else at j = outer_max.  Segments continue one another through the state checkpoint
 * (duquad_get_state / set_state semantics: theta, beta_out and the average weights continue), so
 * the returned iterates (duquad_get_result) are bitwise those of duquad_solve(alg, outer_done,
 * inner_iters); res (may be NULL) is the last segment's report.  Cost per check: the segment's
 * last-iterate inner solve and two residual passes, 10 doubles to the host.
 * history (NULL, or 8 * ceil(outer_max / check_every) doubles, caller-owned): one row per check,
 *     j, d_bar(lambda^j), F(x_last), F(x_avg), dist(x_last), dist(x_avg), inner iterations so far,
 *     matrix passes so far  -- the SPEC trace fields (k, dual_val, f_last, f_avg, infeas_last,
 *     infeas_avg, inner_iters, cum_matvecs).
 * Fixed inner counts; single QP (batch 1); not with options.dual_average (EINVAL).  Afterwards
 * duquad_get_state returns the state at outer_done; the next plain duquad_solve starts fresh.
 */
duquad_status duquad_solve_monitored(duquad_ctx *ctx, int32_t alg, int32_t outer_max, int32_t inner_iters,
                                     int32_t check_every, int32_t which, double eps, double F_star,
                                     duquad_monitor *mon, double *history, duquad_result *res);

/*
 * Testing entry point for the row-sharded path on ONE device: ctxs[r] (r = 0..P-1) must have
 * been set up with world_size = P, rank = r, emulate_ranks = 1 and the same stream and device.
 * Runs duquad_solve's schedule for all ranks in lock step, phase by phase; each all-gather of
 * the y / w replicas is done with device-to-device copies between the contexts (no waiting
 * kernels, no collective).  Constants must have been injected (duquad_set_constants) on every
 * context.  Results per rank as for duquad_solve (duquad_get_result gives local slices).
 */
duquad_status duquad_solve_emulated(duquad_ctx **ctxs, int32_t P, int32_t alg, int32_t outer_iters,
                                    int32_t inner_iters);

/*
 * duquad_solve_eps on an emulated row-sharded group (see above): the stop test's sum of
 * (y - x+)^2 is the sum over the ranks (added in rank order here; ncclAllReduce on a real group),
 * so every rank takes the same decision.  Counts per rank via duquad_get_inner_counts.
 */
duquad_status duquad_solve_eps_emulated(duquad_ctx **ctxs, int32_t P, int32_t alg, int32_t outer_iters,
                                        int32_t inner_max, double eps_in, double sigma_L);

void duquad_destroy(duquad_ctx *ctx);

/* Message for the last failing call on ctx (or of the last failed setup if ctx is NULL). */
const char *duquad_last_error(const duquad_ctx *ctx);

#ifdef __cplusplus
}
#endif

#endif /* DUQUAD_H */
