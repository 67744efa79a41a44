// Internal declarations shared by the host runtime (capi.cu) and the kernel
// translation units.  Not part of the public ABI (see include/duquad.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>
#include <vector>

#include "../../include/duquad.h"

namespace dq {

constexpr int kWarp = 32;

// Per-outer-iteration scalars read by the fused kernels through a device
// index (so that one captured CUDA graph serves every outer iteration).
struct OuterParam {
    double beta_out;   // beta_{j-1} used for mu^{j} = lambda^{j-1} + beta (lambda^{j-1} - lambda^{j-2})
    double avg_w;      // omega_j / S_j for the running primal average (0 = no update)
    int32_t dual_update;  // 1: the first inner pass A of this outer iteration does the DFOM step
    int32_t mu_hat;    // DGM dual averaging: mu := the updated dual average lam_hat
    double lhat_w;     // DGM dual averaging: lam_hat += lhat_w (lambda - lam_hat) at this DFOM step
};

enum PassMode : int { MODE_SOLVE = 0, MODE_LIN = 1 };

// Sparse kernel kinds (kernels_csr.cu, kernels_sell.cu)
enum SparseKind : int32_t { SPK_CSR = 0, SPK_SELL = 1, SPK_ROWT = 2 };

// SELL-32 view of a sparse matrix (kernels_sell.cu): slice s holds 32 rows; its k-th column of
// nonzeros is val/col[sptr[s] + 32 k + lane].  Rows form two segments, [0, nq) and [nq, rows),
// that never share a slice (pass A: Q rows, then G rows): slice s, lane l is row 32 s + l of the
// first segment (s < nsl_q), else row nq + 32 (s - nsl_q) + l (an empty lane past a segment's end).
struct SellMat {
    const double *val;
    const int32_t *col;
    const int64_t *sptr;   // nsl + 1 element offsets (32 x the slice width apart)
    int64_t nsl, nsl_q, nq, rows;
};

// Diagonal (DIA) view of the Q rows of pass A when Q is banded (config 4: 11 diagonals): value k of
// local row i sits in val[k * ldv + i] for the diagonal at column offset off[k] (ascending = CSR
// column order; 0 where the diagonal leaves the matrix).  No column indices, coalesced loads.
// Symmetric form (sym = 1; Q = Q'): only the diagonals off[k] >= 0 are stored, at
// val[k * ldv + halo + i] for i in [-halo, rows) (halo = the widest offset): row i's lower entry
// Q[gi, gi - o] is the stored upper entry of row i - o, Q[gi - o, gi]; the halo rows before the
// slice are filled from the local rows' own lower entries (so a row shard needs no remote data).
// Half the diagonal bytes of the band per step (config 4: 6 of 11 diagonals).
constexpr int kDiaMax = 16;
struct DiaMat {
    const double *val;
    int32_t nd;            // stored diagonals (0: Q rows are not in DIA form)
    int32_t off[kDiaMax];
    int64_t ldv;           // rows (+ halo) padded to a multiple of 32
    int64_t r0, n;         // global index of local row 0, columns
    int32_t sym;           // 1: symmetric half-band form (off[] >= 0 only)
    int32_t halo;          // sym: rows stored before local row 0 (= the widest offset)
};

// ---------------------------------------------------------------- pass A
// Streams rows [row_begin, row_end) of the local stacked matrix A = [Q_r; G_r]
// (row-major, leading dimension ld doubles, zero-padded) against y (full
// replica, ld doubles, zero-padded) staged in shared memory.
struct PassAArgs {
    const double *A;
    int64_t ld;
    int64_t nq;          // local Q rows (rows < nq are Q rows)
    int64_t row_begin, row_end;
    const double *y;
    double *qy;          // Q rows: qy[row] = (Q y)_row
    // G rows (k = row - nq):
    double *w;           // w[k]  (local slice of the full w replica)
    const double *g;
    double *mu;
    double *lam_prev;
    double *h;           // batched only (else null): h[k] = mu[k] + rho g[k], written by the DFOM step
    double *lam_hat;     // DGM dual averaging only (else null): running average of lambda^0..lambda^j
    int32_t w_plus_g;    // equality-QP H path, DFOM-step launch: w = mu + rho g (c = q + G'w)
    const uint8_t *cone;
    double rho;
    double step;         // dual_step_scale / L_d
    int32_t project_dual;
    int32_t first_inner; // this launch is the first inner step of an outer iteration
    const OuterParam *ops;
    const int32_t *d_j;
    double lin_coef;     // MODE_LIN: w[k] = lin_coef * (G y)_k
    // CSR storage of the stacked local [Q_r; G_r] (format == DUQUAD_CSR)
    int32_t fmt;
    int32_t gs;          // lanes per row (power of two, 2..32)
    const int32_t *rp;   // row pointers (rows + 1), rebased to 0
    const int32_t *ci;   // column indices
    const double *va;    // values
    const int32_t *skip; // eps_in mode: the inner solve has converged -> the launch does nothing
    int32_t sp_kind;     // SparseKind: sub-warp CSR, SELL-32 or thread-per-row CSR
    int32_t sp_u;        // lane kernels: nonzeros per load round
    SellMat sell;
    DiaMat dia;          // SELL pass A: the Q rows in DIA form (dia.nd > 0)
};

// ---------------------------------------------------------------- pass B
// Streams the local rows of G' (row-major, leading dim ldp, zero-padded)
// against the full w replica staged in shared memory.
struct PassBArgs {
    const double *GT;
    int64_t ldp;
    int64_t nrows;
    const double *w;
    const double *qy;
    const double *q, *lb, *ub;
    double *x;
    double *y;           // local slice of the full y replica
    double *xhat;
    double L_in;
    double beta_in;
    int32_t last_inner;
    int32_t use_qy;      // MODE_LIN: out = (use_qy ? qy : 0) + G'w
    const OuterParam *ops;
    const int32_t *d_j;
    int32_t *flag;       // set to 1 if an iterate is non-finite
    double *out;         // MODE_LIN output
    // CSR storage of the local rows of G'
    int32_t fmt;
    int32_t gs;
    const int32_t *rp;
    const int32_t *ci;
    const double *va;
    const int32_t *skip; // eps_in mode: the inner solve has converged -> the launch does nothing
    double *gm_sq;       // eps_in mode: gm_sq[j] = (y_j - x+_j)^2 (gradient-map test)
    int32_t box_uniform; // every lb_j == lb_u and ub_j == ub_u: the epilogue skips the lb / ub loads
    double lb_u, ub_u;
    int32_t sp_kind;     // SparseKind: sub-warp CSR, SELL-32 or thread-per-row CSR
    int32_t sp_u;        // lane kernels: nonzeros per load round
    SellMat sell;
};

// ---------------------------------------------------------------- batched (B QPs, shared Q, G)
// C[m][b] = sum_k Aop[m][k] Bop[b][k]; per-QP vectors are QP-major with strides sn / sp.
struct BatchedArgs {
    const double *Aop;
    int64_t lda, M;      // valid rows
    const double *Bop;
    int64_t ldb, N;      // valid QPs
    int64_t K;           // reduction length, padded to a multiple of 32 (zero padding)
    int64_t sn, sp;
    int64_t sw;          // stride of pass A's G-row output a.w (sp, or the paired rows' D buffer stride)
    int64_t pairP;       // > 0: G = [G_t; -G_t] with P = p/2 paired rows; pass A streams [Q; G_t] and
                         // writes d = w_top - w_bottom (a.w, stride sw), pass B multiplies G_t' d
    int64_t ncol8;       // QP octets (set by launch_batched)
    int32_t pdl;         // launch with programmatic dependent launch (epilogue.cuh pdl_wait)
    // eps_in mode (else null): per-QP stop-test sums, stop flags, number of stopped QPs
    double *gm_b;
    int32_t *done_b;
    const int32_t *ndone;
    PassAArgs a;         // pass 0 epilogue (pointers at QP 0)
    PassBArgs b;         // pass 1 epilogue
};

// ---------------------------------------------------------------- whole-solve small kernel (K4)
struct SmallArgs {
    const double *A, *GT;          // packed [Q;G] (n+p x ld) and G' (n x ldp) in HBM
    int64_t n, p, ld, ldp;
    const double *q, *lb, *ub, *g;
    const uint8_t *cone;
    int32_t K, Kin;
    const double *beta_in;         // device, Kin + 1 entries (1-based)
    PassAArgs a;                   // scalars (rho, step, project_dual, ops, nq)
    PassBArgs b;                   // scalars (L_in, ops, flag)
    double *trace_lam, *trace_u;
    int64_t trace_max;
    double *x_out, *xhat_out, *y_out, *lam_out, *mu_out;
    const double *x_init, *lam_init;   // warm start (NULL: [0]_U and 0)
};

// ---------------------------------------------------------------- byte-floor inner step
// Q-role piece: the (tile column, row) triangle sequence from (j0, r0) up to (j1, r1), exclusive.
struct FusedPiece {
    int32_t j0, r0, j1, r1;
};
constexpr int kFusedMaxTiles = 8;   // tile columns of 4096 (ld <= 32768)
struct FusedArgs {
    const double *Q;       // [Q] rows of the packed [Q;G] (ld doubles per row)
    const double *G;       // [G] rows
    const double *y;       // y replica (ld)
    double *ws_rowp;       // [nt][16][ld] Q row-dot partials per tile column and warp
    double *ws_col;        // [nq][2][4096] Q column sums per Q CTA and tile-column slot
    double *ws_g;          // [ng][ld]     G'w partials per G pair
    int32_t cslots;        // ws_col slots per Q CTA (tile columns a piece spans)
    const FusedPiece *pieces;   // [nq] (device)
    int64_t n, p, ld;
    int32_t nt;            // Q tile columns: [4096 J, min(4096 (J + 1), ld))
    int32_t cg;            // G-role cluster size (2)
    int32_t W;             // G column blocks [c W, (c + 1) W), c < cg (the last ends at ld)
    int32_t nchg;          // G: chunks of 4096 columns per block (template parameter)
    int32_t nb;            // grid (CTAs), a multiple of cg
    int32_t nq_ctas;       // Q-role CTAs (a multiple of cg); the rest are ng G-role clusters
    int32_t ng;
    int32_t qlo[kFusedMaxTiles], qhi[kFusedMaxTiles];   // Q CTAs with rows in tile column J
    int64_t qa, qb;        // this rank's Q rows [qa, qb) (global; Q row 0 is row qa); single GPU: [0, n)
    double *partial;       // row-sharded epilogue mode: write the rank's partial n-vector here, no epilogue
    size_t smem;
    int32_t pdl;           // launch the stream and epilogue kernels with programmatic dependent launch
    PassAArgs a;           // G-row epilogue (g, mu, lam_prev, cone, rho, step, ops, first_inner)
};

struct LaunchCfg {
    int grid;
    int threads;
    size_t smem;
    int pdl = 0;   // launch with programmatic dependent launch (epilogue.cuh pdl_wait)
};

// cudaLaunchKernelEx with the PDL attribute when `pdl` (plus an optional cluster width)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, int pdl,
                             int cluster, Args &&...args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (pdl) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (cluster > 0) {
        at[na].id = cudaLaunchAttributeClusterDimension;
        at[na].val.clusterDim.x = cluster;
        at[na].val.clusterDim.y = 1;
        at[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = na ? at : nullptr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// kernels_csr.cu
int csr_blocks_per_sm(int pass, int gs);
cudaError_t launch_pass_a_csr(const PassAArgs &a, int mode, const LaunchCfg &cfg, cudaStream_t s);
cudaError_t launch_pass_b_csr(const PassBArgs &b, int mode, const LaunchCfg &cfg, cudaStream_t s);
// dst[i] = src[i] - sub + add, i < count
cudaError_t launch_rebase(int32_t *dst, const int32_t *src, int64_t count, int32_t sub, int32_t add,
                          cudaStream_t s);
// flag |= CSR structure invalid (row pointers non-monotone / wrong ends, columns out of range,
// values non-finite)
cudaError_t launch_check_csr(const int32_t *rp, const int32_t *ci, const double *va, int64_t rows,
                             int64_t cols, int64_t nnz, int32_t *flag, cudaStream_t s);
// flag = 3 unless (rp, ci, va) and its transpose (trp, tci, tva) agree: same pattern, values to
// 1e-12 relative (the Q symmetry check of the CSR path)
cudaError_t launch_csr_sym_cmp(const int32_t *rp, const int32_t *ci, const double *va, const int32_t *trp,
                               const int32_t *tci, const double *tva, int64_t rows, int64_t nnz, int32_t *flag,
                               cudaStream_t s);
// Transpose of a CSR matrix (rows x cols) restricted to output rows [c0, c0 + nc):
// builds (rp_t, ci_t, va_t) with columns (original rows) sorted; allocates the outputs.
cudaError_t csr_transpose_rows(const int32_t *rp, const int32_t *ci, const double *va, int64_t rows,
                               int64_t cols, int64_t nnz, int64_t c0, int64_t nc, int32_t **rp_t,
                               int32_t **ci_t, double **va_t, int64_t *nnz_t, cudaStream_t s);
int csr_group_size(double avg_nnz_per_row);

// kernels_sell.cu: lane-per-row sparse kernels (SELL-32 storage built on the device from the
// rebased local CSR; thread-per-row CSR on the CSR arrays)
struct SellStore {
    double *val = nullptr;
    int32_t *col = nullptr;
    int64_t *sptr = nullptr;
    int64_t nsl = 0, nsl_q = 0, nq = 0, rows = 0, padded = 0;
};
struct SparsePlan {        // row statistics of a local CSR matrix (rows [0, nq) and [nq, rows))
    int64_t nsl = 0, nsl_q = 0;
    int64_t padded = 0;    // SELL-32 element count (32 x the longest row of every slice)
    int32_t max_len = 0;
};
cudaError_t sparse_plan(const int32_t *rp, int64_t rows, int64_t nq, SparsePlan *plan, cudaStream_t s);
cudaError_t sell_build(const int32_t *rp, const int32_t *ci, const double *va, int64_t rows, int64_t nq,
                       const SparsePlan &plan, SellStore *out, cudaStream_t s);
void sell_free(SellStore *st);
// DIA form of rows [0, rows) of a rebased CSR matrix (global row of local row i: r0 + i) when it has at
// most kDiaMax distinct column offsets within [-64, 64] and the diagonals hold at most `max_pad` x its
// nonzeros; *val = NULL (nothing allocated) otherwise.  allow_sym: store the symmetric half band
// (DiaMat.sym) when the offsets are symmetric and every in-slice pair Q[i, i-o] == Q[i-o, i] bitwise
// (else the full band is kept)
cudaError_t dia_build(const int32_t *rp, const int32_t *ci, const double *va, int64_t rows, int64_t r0, int64_t n,
                      int64_t nnz, double max_pad, bool allow_sym, DiaMat *out, double **val, cudaStream_t s);
SellMat sell_view(const SellStore &st);
int lane_unroll(int kind, int64_t max_width, double mean_len);
int lane_blocks_per_sm(int pass, int kind, int u);
cudaError_t launch_pass_a_lane(const PassAArgs &a, int mode, const LaunchCfg &cfg, cudaStream_t s);
cudaError_t launch_pass_b_lane(const PassBArgs &b, int mode, const LaunchCfg &cfg, cudaStream_t s);

// kernels_fused.cu
bool fused_supported(int64_t n, int64_t ld, size_t smem_optin);
int fused_block_width(int64_t ld, int cg);
int fused_nchg(int64_t ld, int cg);
int fused_max_clusters(int nchg, int cg, size_t smem);
int fused_tiles(int64_t ld);
size_t fused_smem_bytes();
cudaError_t launch_slice_epi(const PassBArgs &bl, const PassBArgs &bs, const double *sum, cudaStream_t s);
cudaError_t launch_vec_add(double *dst, const double *src, int64_t n, cudaStream_t s);
int fused_partition(int64_t n, int64_t ld, int nq, double row_cost, double diag_fac, double diag_slope,
                    std::vector<FusedPiece> &pieces, int32_t *qlo, int32_t *qhi, int64_t qa, int64_t qb);
cudaError_t configure_fused_kernels(int nchg, size_t smem);
cudaError_t launch_fused_stream(const FusedArgs &f, cudaStream_t s);
cudaError_t launch_fused_epi(const PassBArgs &bl, const PassBArgs &bs, const FusedArgs &f, cudaStream_t s);

// kernels_small.cu
size_t small_smem_bytes(int64_t n, int64_t p, int64_t ld, int64_t ldp, int K, int Kin);
cudaError_t configure_small_kernel(size_t smem);
cudaError_t launch_small_solve(const SmallArgs &sa, size_t smem, cudaStream_t s);

// kernels_batched.cu
cudaError_t configure_batched_kernels();
cudaError_t launch_batched(const BatchedArgs &a, int pass, int mode, cudaStream_t s);
cudaError_t launch_init_batched(double *x, double *y, double *xhat, const double *lb, const double *ub, int64_t n,
                                int64_t sn, double *mu, double *lam_prev, int64_t sp, int64_t B, int32_t *d_j,
                                int32_t *flag, cudaStream_t s);
cudaError_t launch_mirror_upper(double *H, int64_t n, int64_t ld, cudaStream_t s);
cudaError_t launch_batched_decide(double *gm_b, int32_t *done_b, int32_t *ndone, double thresh2, int32_t *counts,
                                  int64_t nc, const int32_t *d_j, int64_t B, cudaStream_t s);
cudaError_t launch_batched_finish(const double *x, double *y, double *xhat, int64_t n, int64_t sn, int64_t B,
                                  const OuterParam *ops, const int32_t *d_j, int32_t *done_b, int32_t *ndone,
                                  int32_t *conv, int64_t nc, cudaStream_t s);
// flag = 1 unless the rows of G (P + P rows, ld apart) satisfy G[k + P] == -G[k] (paired rows)
cudaError_t launch_check_pairs(const double *G, int64_t P, int64_t n, int64_t ld, int32_t *flag, cudaStream_t s);
cudaError_t launch_batched_h(double *h, const double *mu, const double *g, double rho, int64_t p, int64_t sp,
                             int64_t B, cudaStream_t s);

// kernels_dense.cu
cudaError_t launch_pass_a(const PassAArgs &a, int mode, const LaunchCfg &cfg, cudaStream_t s);
cudaError_t launch_pass_b(const PassBArgs &b, int mode, const LaunchCfg &cfg, cudaStream_t s);
int pass_threads();
// K3 (rho = 0): grad = Qy + c streamed over Q rows only; bl / bs: epilogue views for load (y = yin,
// q = c) and store (y = yout)
cudaError_t launch_rho0_step(const PassAArgs &a, const PassBArgs &bl, const PassBArgs &bs, const LaunchCfg &cfg,
                             cudaStream_t s);
cudaError_t configure_pass_kernels(size_t smem_a, size_t smem_b);
cudaError_t launch_init_state(double *x, double *y, double *xhat, const double *lb, const double *ub,
                              int64_t n, double *mu, double *lam_prev, int64_t p, int32_t *d_j,
                              int32_t *flag, cudaStream_t s);
cudaError_t launch_advance(int32_t *d_j, cudaStream_t s);
// persistent two-pass solve (one cooperative launch for (K + 1) x Kin inner steps; L2-resident QPs)
cudaError_t launch_persist(const PassAArgs &a, const PassBArgs &b, const double *beta_in, int K, int Kin,
                           uint32_t *bar, int grid, size_t smem, cudaStream_t s);
cudaError_t configure_persist(size_t smem);
// warm start: u_bar^0 = [x0]_U, lambda^0 = mu^1 = lam0 (either may be NULL), B QPs with strides sn / sp
cudaError_t launch_apply_initial(double *x, double *y, const double *lb, const double *ub, int64_t n, int64_t sn,
                                 const double *x0, double *mu, double *lam_prev, int64_t p, int64_t sp,
                                 const double *lam0, int64_t B, cudaStream_t s);
// eps_in mode (duquad_solve_eps): after an inner step, sum gm_sq (fixed order; partials + the last
// block) -> counts[*d_j - 1] += 1 and *done = 1 if L_in^2 sum <= 2 sigma eps_in (thresh2 = that / L_in^2)
cudaError_t launch_inner_check(const double *gm_sq, int64_t n, double *partials, uint32_t *counter, int32_t *done,
                               double thresh2, int32_t *counts, const int32_t *d_j, double *out_sum, cudaStream_t s);
cudaError_t launch_inner_decide(const double *sum, int32_t *done, double thresh2, int32_t *counts,
                                const int32_t *d_j, cudaStream_t s);
// after the inner loop: y_dst = x (u_bar^j), running average with ops[*d_j].avg_w, conv[*d_j - 1] = *done,
// *done = 0
cudaError_t launch_inner_finish(const double *x, double *y_dst, double *xhat, int64_t n, const OuterParam *ops,
                                const int32_t *d_j, int32_t *done, int32_t *conv, cudaStream_t s);
cudaError_t launch_transpose(const double *G, int64_t ldG, int64_t p, int64_t col0, int64_t ncols,
                             double *GT, int64_t ldp, cudaStream_t s);
cudaError_t launch_check(const double *v, int64_t rows, int64_t cols, int64_t ld, int32_t *flag,
                         cudaStream_t s);
// flag = 2 if the n x n block at A is not symmetric (|Q_ij - Q_ji| > 1e-12 (|Q_ij| + |Q_ji|))
cudaError_t launch_check_sym(const double *A, int64_t n, int64_t ld, int32_t *flag, cudaStream_t s);
cudaError_t launch_check_box(const double *lb, const double *ub, int64_t n, int32_t *flag,
                             cudaStream_t s);
// Deterministic reductions: `parts` partial sums per CTA, then a fixed-order final sum.
constexpr int kRedGrid = 148;
constexpr int kRedThreads = 256;
cudaError_t launch_dot_partial(const double *a, const double *b, int64_t n, double *partials,
                               cudaStream_t s);
cudaError_t launch_reduce_final(const double *partials, int nparts, int nvals, double *out,
                                cudaStream_t s);
// Lanczos helpers
cudaError_t launch_fill_hash(double *v, int64_t n, int64_t offset, cudaStream_t s);
cudaError_t launch_scale_by_rsqrt(double *v, int64_t n, const double *sumsq, double *beta_out,
                                  cudaStream_t s);
cudaError_t launch_lanczos_update(double *w, const double *v, const double *vprev, int64_t n,
                                  const double *alpha, const double *beta_prev, double *partials,
                                  cudaStream_t s);
cudaError_t launch_lanczos_next(double *v, double *vprev, const double *w, int64_t n,
                                const double *sumsq, double *beta, cudaStream_t s);
// Residual partials: per CTA 5 values:
//   [0] sum x*qy/2 + q*x over local n rows   [1] sum dist_K(r)^2, r = Gx+g (local p rows)
//   [2] sum dist_K(r + lam/rho)^2            [3] sum lam^2        [4] sum lam * r
cudaError_t launch_residual_partial(const double *x, const double *qy, const double *q, int64_t n,
                                    const double *Gx, const double *g, const double *lam,
                                    const uint8_t *cone, int64_t p, double rho, double *partials,
                                    cudaStream_t s);

}  // namespace dq
