// Host runtime + C ABI of the DuQuad hot path (include/duquad.h).
//
// Owns the device buffers, the per-solve parameter tables (theta / beta,
// PAPER.md:358-363, 587-589; averaging weights), the CUDA-graph
// capture of one outer DFOM iteration, the NCCL communicator of the sharded
// path, and the launch schedule:
//
//   for j = 1 .. K_out + 1:                 (j = K_out+1: last-iterate solve)
//     for k = 1 .. K_in:                    (Algorithm FOM)
//       pass A   [Q;G] y -> Qy, w   (k = 1 and j >= 2: fused DFOM step)
//       (all-gather w)
//       pass B   G'w -> x, y        (k = K_in: y <- x, running average)
//       (all-gather y)
//     advance j
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "duquad_internal.h"

using namespace dq;

struct duquad_ctx {
    int dev = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    duquad_options opt{};
    int64_t n = 0, p = 0, batch = 1;
    int32_t format = DUQUAD_DENSE;
    double rho = 0.0;
    // sharding
    int world = 1, rank = 0;
    bool sharded = false;    // world > 1, or nccl_self: the row-sharded code path and its collectives
    bool emulated = false;   // P ranks on one device, driven by duquad_solve_emulated
    ncclComm_t comm = nullptr;
    int64_t n_slice = 0, p_slice = 0, r0 = 0, s0 = 0, nloc = 0, ploc = 0;
    std::vector<int64_t> gs0, gcnt;   // G rows [gs0[r], gs0[r] + gcnt[r]) of every rank (contiguous, ascending)
    bool floor_shard = false;         // row-sharded byte floor (G rows balanced against the Q triangle slabs)
    // layout
    int64_t ld = 0, ldp = 0, ylen = 0, wlen = 0;
    // device buffers (dense)
    double *A = nullptr, *GT = nullptr;
    double *y_full = nullptr, *w_full = nullptr;
    double *qy = nullptr, *x = nullptr, *xhat = nullptr, *q = nullptr, *lb = nullptr, *ub = nullptr;
    double *g = nullptr, *mu = nullptr, *lam_prev = nullptr;
    uint8_t *cone = nullptr;
    double *lz_vprev = nullptr, *lz_w = nullptr;
    // CSR storage (format == DUQUAD_CSR): stacked local [Q_r; G_r] and local rows of G'
    int32_t *a_rp = nullptr, *a_ci = nullptr, *b_rp = nullptr, *b_ci = nullptr;
    double *a_va = nullptr, *b_va = nullptr;
    int64_t nnz_a = 0, nnz_b = 0;
    int gs_a = 4, gs_b = 4;
    SellStore sell_a, sell_b;   // SELL-32 copies of the two (options.sell_path; empty unless kind SPK_SELL)
    int kind_a = SPK_CSR, kind_b = SPK_CSR, u_a = 8, u_b = 8;   // SparseKind and load-round width per pass
    DiaMat dia{};               // pass A's Q rows in DIA form (banded Q; SELL pass A only)
    double *dia_val = nullptr;
    int box_uniform = 0;        // this context's lb / ub are constant vectors (lb_u, ub_u)
    double lb_u = 0.0, ub_u = 0.0;
    // batched storage (batch > 1): QP-major per-QP vectors, strides ld (n-vectors) / ldp (p-vectors)
    int64_t Btot = 1, Bloc = 1, b0 = 0;
    double *Yb = nullptr, *Xb = nullptr, *XHb = nullptr, *QYb = nullptr, *qb = nullptr;
    double *Wb = nullptr, *gb = nullptr, *mub = nullptr, *lpb = nullptr;
    double *hb = nullptr;   // batched: h = mu + rho g per (QP, G row), refreshed by every DFOM step
    int64_t pairP = 0;       // batched, G = [G_t; -G_t] (options.pair_rows): P = p / 2 paired rows
    double *Db = nullptr;    // paired rows: d = w_top - w_bottom per (QP, pair), stride ldd
    int64_t ldd = 0;
    // rho = 0 specialisation (K3): second y replica (ping-pong) and c = q + G'mu
    bool rho0 = false;
    bool davg = false;
    bool eqh = false;
    double *fpart = nullptr, *rs_out = nullptr;   // row-sharded byte floor: partial n-vector, its reduced slice
    // state export / resume (NEXT-2): the state after outer iteration j (before the last-iterate solve)
    double *ck_x = nullptr, *ck_mu = nullptr, *ck_lp = nullptr, *ck_xh = nullptr;
    bool ck_valid = false;     // a checkpoint from the last solve (options.checkpoint) or set_state
    bool resume = false;       // the next solve continues from the checkpoint (duquad_set_state)
    bool resumed = false;      // this solve is a continuation
    int64_t ck_j = 0, j0 = 0;  // outer iterations done at the checkpoint; offset of this solve
    double ck_S = 0.0, S_end = 0.0;
    int32_t h_j = 0;          // equality QP on H = Q + rho G'G (options.eq_precompute, NEXT-3)
    double *Hq = nullptr;      // H, n x ld row-major (exactly symmetric)   // this solve: DGM dual-averaging final point (options.dual_average)
    double *lam_hat = nullptr, *lhb = nullptr;   // running dual average (single QP / batched)
    double *y_full2 = nullptr, *cvec = nullptr;
    LaunchCfg cfg_k3{};
    // byte-floor inner step (symmetric Q read once as a triangle, G read once)
    bool fused = false;
    FusedArgs fz{};
    double *ws = nullptr;          // ws_rowp | ws_col | ws_g
    FusedPiece *fpieces = nullptr;
    // warm start (duquad_set_initial): local slices, batched layout for batch > 1
    double *init_x = nullptr, *init_lam = nullptr;
    // eps_in-driven inner stopping (duquad_solve_eps): device flag / counters, active during a solve
    bool eps_mode = false;
    double eps_thresh2 = 0.0;
    double *gm_sq = nullptr, *gm_part = nullptr;
    double *gm_tot = nullptr;    // row-sharded eps_in mode: this rank's sum, then the all-reduced one
    double *gm_b = nullptr;      // batched eps_in mode: per-QP sums, stop flags, number stopped
    int32_t *done_b = nullptr, *ndone = nullptr;
    int64_t eps_nc = 0;          // eps_in mode: solves per QP (K + 1)
    bool pend_decide = false;    // a stop decision waits for the all-reduce (issued with the y gather)
    uint32_t *gm_counter = nullptr;
    int32_t *d_done = nullptr, *d_counts = nullptr;   // d_counts: [K+1] steps, then [K+1] converged flags
    int64_t counts_cap = 0;
    std::vector<int32_t> last_counts, last_conv;
    // persistent two-pass solve (L2-resident dense QPs): one cooperative launch per solve
    bool persist = false;
    size_t persist_smem = 0;
    uint32_t *pbar = nullptr;
    // whole-solve single-CTA kernel (small dense QPs)
    bool small = false;
    size_t small_smem = 0;
    double *d_beta = nullptr;
    int64_t beta_cap = 0;
    double *scal = nullptr;       // device scalars
    double *partials = nullptr;   // kRedGrid * 5
    OuterParam *d_ops = nullptr;
    int64_t ops_cap = 0;
    int32_t *d_j = nullptr, *d_flag = nullptr;
    // constants
    double L_in = 0.0, L_d = 0.0;
    bool have_consts = false;
    // launch configuration
    LaunchCfg cfg_a{}, cfg_b{};
    // trace
    double *trace_lam = nullptr, *trace_u = nullptr;
    int64_t trace_max = 0;
    bool solved = false;
    std::string err;
};

namespace {

thread_local std::string g_err;

duquad_status fail(duquad_ctx *ctx, duquad_status st, const std::string &msg) {
    if (ctx)
        ctx->err = msg;
    else
        g_err = msg;
    return st;
}

#define CK(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(ctx, DUQUAD_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define NK(call)                                                                              \
    do {                                                                                      \
        ncclResult_t r_ = (call);                                                             \
        if (r_ != ncclSuccess)                                                                \
            return fail(ctx, DUQUAD_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
    } while (0)

inline int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

template <typename T>
cudaError_t dalloc(T **p, int64_t count) {
    size_t bytes = (size_t)std::max<int64_t>(count, 2) * sizeof(T);
    cudaError_t e = cudaMalloc((void **)p, bytes);
    if (e == cudaSuccess) e = cudaMemset(*p, 0, bytes);
    return e;
}

void free_all(duquad_ctx *c) {
    double *ds[] = {c->A,   c->GT,  c->y_full, c->w_full, c->qy,       c->x,        c->xhat,     c->q,
                    c->lb,  c->ub,  c->g,      c->mu,     c->lam_prev, c->lz_vprev, c->lz_w,     c->scal,
                    c->partials, c->Yb, c->Xb, c->XHb,   c->QYb,      c->qb,       c->Wb,       c->gb,
                    c->mub, c->lpb, c->hb, c->Db, c->d_beta, c->y_full2, c->cvec, c->ws, c->lam_hat, c->lhb, c->Hq, c->ck_x, c->ck_mu, c->ck_lp, c->ck_xh, c->fpart, c->rs_out};
    for (double *d : ds)
        if (d) cudaFree(d);
    if (c->cone) cudaFree(c->cone);
    int32_t *is[] = {c->a_rp, c->a_ci, c->b_rp, c->b_ci};
    for (int32_t *d : is)
        if (d) cudaFree(d);
    if (c->a_va) cudaFree(c->a_va);
    if (c->b_va) cudaFree(c->b_va);
    sell_free(&c->sell_a);
    sell_free(&c->sell_b);
    if (c->dia_val) cudaFree(c->dia_val);
    if (c->d_ops) cudaFree(c->d_ops);
    if (c->d_j) cudaFree(c->d_j);
    if (c->d_flag) cudaFree(c->d_flag);
    if (c->fpieces) cudaFree(c->fpieces);
    if (c->pbar) cudaFree(c->pbar);
    if (c->init_x) cudaFree(c->init_x);
    if (c->init_lam) cudaFree(c->init_lam);
    if (c->gm_sq) cudaFree(c->gm_sq);
    if (c->gm_part) cudaFree(c->gm_part);
    if (c->gm_tot) cudaFree(c->gm_tot);
    if (c->gm_b) cudaFree(c->gm_b);
    if (c->done_b) cudaFree(c->done_b);
    if (c->ndone) cudaFree(c->ndone);
    if (c->gm_counter) cudaFree(c->gm_counter);
    if (c->d_done) cudaFree(c->d_done);
    if (c->d_counts) cudaFree(c->d_counts);
    if (c->comm) ncclCommDestroy(c->comm);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
}

// device scalar slots
enum { SC_ALPHA = 0, SC_BETA = 1024, SC_TMP = 2048, SC_TMP2 = 2049, SC_NSCAL = 2056 };
constexpr int kMaxLanczos = 1000;

struct DevGuard {
    int prev = -1;
    explicit DevGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DevGuard() {
        int cur;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// ----------------------------------------------------------- collectives
duquad_status allgather_vec(duquad_ctx *ctx, double *full) {
    if (!ctx->sharded || ctx->emulated) return DUQUAD_OK;
    NK(ncclAllGather(full + ctx->rank * ctx->n_slice, full, (size_t)ctx->n_slice, ncclDouble, ctx->comm,
                     ctx->stream));
    return DUQUAD_OK;
}

duquad_status allgather_y(duquad_ctx *ctx) { return allgather_vec(ctx, ctx->y_full); }

// w replica: every rank's G-row slice in global order.  Equal slices: one all-gather; the balanced
// partition of the row-sharded byte floor: one broadcast per rank inside a group.
duquad_status allgather_w(duquad_ctx *ctx) {
    if (!ctx->sharded || ctx->emulated) return DUQUAD_OK;
    if (!ctx->floor_shard) {
        NK(ncclAllGather(ctx->w_full + ctx->rank * ctx->p_slice, ctx->w_full, (size_t)ctx->p_slice,
                         ncclDouble, ctx->comm, ctx->stream));
        return DUQUAD_OK;
    }
    NK(ncclGroupStart());
    for (int r = 0; r < ctx->world; ++r)
        if (ctx->gcnt[r] > 0)
            NK(ncclBroadcast(ctx->w_full + ctx->gs0[r], ctx->w_full + ctx->gs0[r], (size_t)ctx->gcnt[r], ncclDouble,
                             r, ctx->comm, ctx->stream));
    NK(ncclGroupEnd());
    return DUQUAD_OK;
}

duquad_status allreduce_sum(duquad_ctx *ctx, double *buf, int count) {
    if (!ctx->sharded) return DUQUAD_OK;
    if (ctx->emulated) return fail(ctx, DUQUAD_ESTATE, "not available on emulated ranks (inject constants)");
    NK(ncclAllReduce(buf, buf, (size_t)count, ncclDouble, ncclSum, ctx->comm, ctx->stream));
    return DUQUAD_OK;
}

// ----------------------------------------------------------- pass args
PassAArgs make_a(duquad_ctx *c) {
    PassAArgs a{};
    a.A = c->A;
    a.ld = c->ld;
    a.nq = c->nloc;
    a.row_begin = 0;
    a.row_end = c->nloc + c->ploc;
    a.y = c->y_full;
    a.qy = c->qy;
    a.w = c->w_full + c->s0;
    a.g = c->g;
    a.mu = c->mu;
    a.lam_prev = c->lam_prev;
    a.cone = c->cone;
    a.rho = c->rho;
    a.step = c->have_consts && c->L_d > 0 ? c->opt.dual_step_scale / c->L_d : 0.0;
    a.project_dual = c->opt.project_dual;
    a.ops = c->d_ops;
    a.d_j = c->d_j;
    a.lin_coef = 1.0;
    a.fmt = c->format;
    a.gs = c->gs_a;
    a.rp = c->a_rp;
    a.ci = c->a_ci;
    a.va = c->a_va;
    a.skip = c->eps_mode ? c->d_done : nullptr;
    a.lam_hat = c->davg ? c->lam_hat : nullptr;
    a.sp_kind = c->kind_a;
    a.sp_u = c->u_a;
    a.sell = sell_view(c->sell_a);
    a.dia = c->dia;
    return a;
}

PassBArgs make_b(duquad_ctx *c) {
    PassBArgs b{};
    b.GT = c->GT;
    b.ldp = c->ldp;
    b.nrows = c->nloc;
    b.w = c->w_full;
    b.qy = c->qy;
    b.q = c->q;
    b.lb = c->lb;
    b.ub = c->ub;
    b.x = c->x;
    b.y = c->y_full + c->rank * c->n_slice;
    b.xhat = c->xhat;
    b.L_in = c->L_in;
    b.ops = c->d_ops;
    b.d_j = c->d_j;
    b.flag = c->d_flag;
    b.use_qy = 1;
    b.fmt = c->format;
    b.gs = c->gs_b;
    b.rp = c->b_rp;
    b.ci = c->b_ci;
    b.va = c->b_va;
    b.skip = c->eps_mode ? c->d_done : nullptr;
    b.gm_sq = c->eps_mode ? c->gm_sq : nullptr;
    b.box_uniform = c->box_uniform;
    b.lb_u = c->lb_u;
    b.ub_u = c->ub_u;
    b.sp_kind = c->kind_b;
    b.sp_u = c->u_b;
    b.sell = sell_view(c->sell_b);
    return b;
}

BatchedArgs make_batched(duquad_ctx *c, int pass);

// ---------------------------------------------------------------- outer iteration, by phases
// An outer DFOM iteration is a fixed sequence of phases, each a kernel (plus trace copies)
// followed by an optional all-gather of one replica buffer.  run_outer() interleaves them with
// NCCL all-gathers; duquad_solve_emulated() runs the phases of P contexts in lock step and
// replaces the all-gather by device copies.
enum GatherBuf { G_NONE = -1, G_Y = 0, G_Y2 = 1, G_W = 2, G_RS = 3 };   // G_RS: reduce-scatter of fpart

double *gather_ptr(duquad_ctx *c, int b) { return b == G_W ? c->w_full : (b == G_Y2 ? c->y_full2 : c->y_full); }
int64_t gather_slice(duquad_ctx *c, int b) { return b == G_W ? c->p_slice : c->n_slice; }

duquad_status gather_impl(duquad_ctx *ctx, int b);
// the gather of the phase, then (row-sharded eps_in mode) the all-reduce of the stop test's sum and
// the decision, identical on every rank
duquad_status gather(duquad_ctx *ctx, int b) {
    duquad_status st = gather_impl(ctx, b);
    if (st != DUQUAD_OK || !ctx->pend_decide || ctx->emulated) return st;
    ctx->pend_decide = false;
    NK(ncclAllReduce(ctx->gm_tot, ctx->gm_tot, 1, ncclDouble, ncclSum, ctx->comm, ctx->stream));
    CK(launch_inner_decide(ctx->gm_tot, ctx->d_done, ctx->eps_thresh2, ctx->d_counts, ctx->d_j, ctx->stream));
    return DUQUAD_OK;
}

duquad_status gather_impl(duquad_ctx *ctx, int b) {
    if (b < 0 || !ctx->sharded || ctx->emulated) return DUQUAD_OK;   // emulated: group driver copies
    if (b == G_W) return allgather_w(ctx);
    if (b == G_RS) {
        NK(ncclReduceScatter(ctx->fpart, ctx->rs_out, (size_t)ctx->n_slice, ncclDouble, ncclSum, ctx->comm,
                             ctx->stream));
        return DUQUAD_OK;
    }
    double *full = gather_ptr(ctx, b);
    const int64_t sl = gather_slice(ctx, b);
    NK(ncclAllGather(full + ctx->rank * sl, full, (size_t)sl, ncclDouble, ctx->comm, ctx->stream));
    return DUQUAD_OK;
}

int num_phases(const duquad_ctx *c, int Kin) { return (c->rho0 ? Kin + 3 : 2 * Kin + 1) + (c->eps_mode ? 1 : 0); }

// eps_in mode: gradient-map test after inner step k (a no-op once the solve has converged)
duquad_status inner_check(duquad_ctx *ctx) {
    if (!ctx->eps_mode) return DUQUAD_OK;
    if (ctx->Btot > 1) {   // per-QP decisions on the sums the pass-B epilogue accumulated
        CK(launch_batched_decide(ctx->gm_b, ctx->done_b, ctx->ndone, ctx->eps_thresh2, ctx->d_counts, ctx->eps_nc,
                                 ctx->d_j, ctx->Bloc, ctx->stream));
        return DUQUAD_OK;
    }
    CK(launch_inner_check(ctx->gm_sq, ctx->nloc, ctx->gm_part, ctx->gm_counter, ctx->d_done, ctx->eps_thresh2,
                          ctx->d_counts, ctx->d_j, ctx->sharded ? ctx->gm_tot : nullptr, ctx->stream));
    ctx->pend_decide = ctx->sharded;
    return DUQUAD_OK;
}

duquad_status trace_lam_copy(duquad_ctx *ctx, int j) {
    if (j >= 2 && ctx->trace_lam && j - 2 < ctx->trace_max)
        CK(cudaMemcpyAsync(ctx->trace_lam + (j - 2) * ctx->ploc, ctx->lam_prev, ctx->ploc * sizeof(double),
                           cudaMemcpyDeviceToDevice, ctx->stream));
    return DUQUAD_OK;
}

duquad_status end_outer(duquad_ctx *ctx, int j) {
    if (j >= 1 && ctx->trace_u && j - 1 < ctx->trace_max)
        CK(cudaMemcpyAsync(ctx->trace_u + (j - 1) * ctx->nloc, ctx->x, ctx->nloc * sizeof(double),
                           cudaMemcpyDeviceToDevice, ctx->stream));
    CK(launch_advance(ctx->d_j, ctx->stream));
    return DUQUAD_OK;
}

// Phase ph of outer iteration j (reads its per-outer scalars through d_j); *gb = buffer to
// all-gather afterwards.
//   generic:  ph = 2(k-1): pass A (k = 1: fused DFOM step), gather w;  ph = 2k-1: pass B, gather y
//   rho = 0 (row a1', K3):  ph 0: pass A over the G rows at y = u_bar^{j-1} (DFOM step, w = mu^j),
//             gather w;  ph 1: c = q + G'w and y^1 = u_bar^{j-1} into replica A, gather it;
//             ph 1+k: K3 step k (Q only), y ping-pong between replicas A and B
//   last phase: trace u_bar^j, advance j
duquad_status outer_phase(duquad_ctx *ctx, const std::vector<double> &beta_in, int Kin, int j, int ph,
                          std::vector<cudaEvent_t> *ev, int *gb) {
    *gb = G_NONE;
    const int64_t off = ctx->rank * ctx->n_slice;
    duquad_status st;
    if (ph == num_phases(ctx, Kin) - 1) return end_outer(ctx, j);
    if (ctx->eps_mode && ph == num_phases(ctx, Kin) - 2) {   // u_bar^j = x: y, average, flag reset
        if (ctx->Btot > 1) {
            CK(launch_batched_finish(ctx->Xb, ctx->Yb, ctx->XHb, ctx->n, ctx->ld, ctx->Bloc, ctx->d_ops, ctx->d_j,
                                     ctx->done_b, ctx->ndone, ctx->d_counts + ctx->counts_cap, ctx->eps_nc,
                                     ctx->stream));
            return DUQUAD_OK;
        }
        const bool y2 = ctx->rho0 && Kin % 2;
        double *ydst = (y2 ? ctx->y_full2 : ctx->y_full) + ctx->rank * ctx->n_slice;   // this rank's slice
        CK(launch_inner_finish(ctx->x, ydst, ctx->xhat, ctx->nloc, ctx->d_ops, ctx->d_j, ctx->d_done,
                               ctx->d_counts + ctx->counts_cap, ctx->stream));
        *gb = ctx->sharded ? (y2 ? G_Y2 : G_Y) : G_NONE;   // row-sharded: the new y slices to every rank
        return DUQUAD_OK;
    }
    if (ctx->rho0) {
        double *Y[2] = {ctx->y_full, ctx->y_full2};
        if (ph == 0) {
            PassAArgs a = make_a(ctx);
            a.row_begin = ctx->nloc;          // G rows only
            a.first_inner = 1;
            a.w_plus_g = ctx->eqh;            // H path: w = mu + rho g, so c = q + G'(mu + rho g)
            a.y = Y[Kin % 2];                 // the replica the previous inner solve finished in
            CK(launch_pass_a(a, MODE_SOLVE, ctx->cfg_a, ctx->stream));
            if ((st = trace_lam_copy(ctx, j)) != DUQUAD_OK) return st;
            *gb = G_W;
        } else if (ph == 1) {
            PassBArgs c = make_b(ctx);
            c.qy = ctx->q;                    // c = q + G'w
            c.use_qy = 1;
            c.out = ctx->cvec;
            CK(launch_pass_b(c, MODE_LIN, ctx->cfg_b, ctx->stream));
            CK(cudaMemcpyAsync(Y[0] + off, ctx->x, ctx->nloc * sizeof(double), cudaMemcpyDeviceToDevice,
                               ctx->stream));
            *gb = G_Y;
        } else {
            const int k = ph - 1;
            PassAArgs a3 = make_a(ctx);
            if (ctx->eqh) a3.A = ctx->Hq;     // H = Q + rho G'G
            a3.y = Y[(k - 1) % 2];
            PassBArgs bl = make_b(ctx);
            bl.q = ctx->cvec;
            bl.y = Y[(k - 1) % 2] + off;
            bl.beta_in = beta_in[k];
            bl.last_inner = (k == Kin) && !ctx->eps_mode;
            PassBArgs bs = bl;
            bs.y = Y[k % 2] + off;
            if (ev) CK(cudaEventRecord((*ev)[4 * (k - 1) + 0], ctx->stream));
            if (ctx->fused) {   // symmetric-Q stream (upper triangle once) + epilogue with c
                FusedArgs fz = ctx->fz;
                fz.y = Y[(k - 1) % 2];
                fz.a = make_a(ctx);
                CK(launch_fused_stream(fz, ctx->stream));
                if (ev) CK(cudaEventRecord((*ev)[4 * (k - 1) + 1], ctx->stream));
                if (ev) CK(cudaEventRecord((*ev)[4 * (k - 1) + 2], ctx->stream));
                CK(launch_fused_epi(bl, bs, fz, ctx->stream));
                if (ev) CK(cudaEventRecord((*ev)[4 * (k - 1) + 3], ctx->stream));
            } else {
                CK(launch_rho0_step(a3, bl, bs, ctx->cfg_k3, ctx->stream));
                if (ev) {
                    CK(cudaEventRecord((*ev)[4 * (k - 1) + 1], ctx->stream));
                    CK(cudaEventRecord((*ev)[4 * (k - 1) + 2], ctx->stream));
                    CK(cudaEventRecord((*ev)[4 * (k - 1) + 3], ctx->stream));
                }
            }
            if ((st = inner_check(ctx)) != DUQUAD_OK) return st;
            *gb = (k % 2) ? G_Y2 : G_Y;
        }
        return DUQUAD_OK;
    }
    const int k = ph / 2 + 1;
    const bool bt = ctx->Btot > 1;
    if (ctx->fused) {   // byte-floor step: one stream over the Q triangle and G, then the epilogue
        if (ph % 2 == 0) {
            FusedArgs fz = ctx->fz;
            fz.a = make_a(ctx);
            fz.a.first_inner = (k == 1);
            if (ev) CK(cudaEventRecord((*ev)[4 * (k - 1) + 0], ctx->stream));
            CK(launch_fused_stream(fz, ctx->stream));
            if (ev) CK(cudaEventRecord((*ev)[4 * (k - 1) + 1], ctx->stream));
            if (k == 1 && (st = trace_lam_copy(ctx, j)) != DUQUAD_OK) return st;
            if (ctx->sharded) {   // this rank's partial n-vector, then the reduce-scatter over the slices
                fz.partial = ctx->fpart;
                CK(launch_fused_epi(make_b(ctx), make_b(ctx), fz, ctx->stream));
                *gb = G_RS;
            }
        } else {
            PassBArgs b = make_b(ctx);
            b.beta_in = beta_in[k];
            b.last_inner = (k == Kin) && !ctx->eps_mode;
            if (ev) CK(cudaEventRecord((*ev)[4 * (k - 1) + 2], ctx->stream));
            if (ctx->sharded) {
                CK(launch_slice_epi(b, b, ctx->rs_out, ctx->stream));
                *gb = G_Y;
            } else {
                CK(launch_fused_epi(b, b, ctx->fz, ctx->stream));
            }
            if (ev) CK(cudaEventRecord((*ev)[4 * (k - 1) + 3], ctx->stream));
            if ((st = inner_check(ctx)) != DUQUAD_OK) return st;
        }
        return DUQUAD_OK;
    }
    if (ph % 2 == 0) {
        if (ev) CK(cudaEventRecord((*ev)[4 * (k - 1) + 0], ctx->stream));
        if (bt) {
            BatchedArgs BA = make_batched(ctx, 0);
            BA.a.first_inner = (k == 1);
            CK(launch_batched(BA, 0, MODE_SOLVE, ctx->stream));
        } else {
            PassAArgs a = make_a(ctx);
            a.first_inner = (k == 1);
            CK(launch_pass_a(a, MODE_SOLVE, ctx->cfg_a, ctx->stream));
        }
        if (ev) CK(cudaEventRecord((*ev)[4 * (k - 1) + 1], ctx->stream));
        if (k == 1 && (st = trace_lam_copy(ctx, j)) != DUQUAD_OK) return st;
        *gb = G_W;
    } else {
        if (ev) CK(cudaEventRecord((*ev)[4 * (k - 1) + 2], ctx->stream));
        if (bt) {
            BatchedArgs BB = make_batched(ctx, 1);
            BB.b.beta_in = beta_in[k];
            BB.b.last_inner = (k == Kin) && !ctx->eps_mode;
            CK(launch_batched(BB, 1, MODE_SOLVE, ctx->stream));
        } else {
            PassBArgs b = make_b(ctx);
            b.beta_in = beta_in[k];
            b.last_inner = (k == Kin) && !ctx->eps_mode;
            CK(launch_pass_b(b, MODE_SOLVE, ctx->cfg_b, ctx->stream));
        }
        if (ev) CK(cudaEventRecord((*ev)[4 * (k - 1) + 3], ctx->stream));
        if ((st = inner_check(ctx)) != DUQUAD_OK) return st;
        *gb = G_Y;
    }
    return DUQUAD_OK;
}

duquad_status run_outer(duquad_ctx *ctx, const std::vector<double> &beta_in, int Kin, int j,
                        std::vector<cudaEvent_t> *ev) {
    duquad_status st;
    for (int ph = 0; ph < num_phases(ctx, Kin); ++ph) {
        int gb;
        if ((st = outer_phase(ctx, beta_in, Kin, j, ph, ev, &gb)) != DUQUAD_OK) return st;
        if ((st = gather(ctx, gb)) != DUQUAD_OK) return st;
    }
    return DUQUAD_OK;
}

// Batched passes (row a9): the single-QP argument blocks re-pointed at QP 0 of the
// QP-major batched vectors; the kernels offset them per QP.
BatchedArgs make_batched(duquad_ctx *c, int pass) {
    BatchedArgs ba{};
    ba.a = make_a(c);
    ba.b = make_b(c);
    ba.sn = c->ld;
    ba.sp = std::max<int64_t>(c->ldp, 2);
    ba.N = c->Bloc;
    ba.pairP = c->pairP;
    ba.pdl = c->cfg_a.pdl;
    ba.sw = c->pairP ? c->ldd : ba.sp;
    ba.a.qy = c->QYb;
    ba.a.w = c->pairP ? c->Db : c->Wb;
    ba.a.g = c->gb;
    ba.a.mu = c->mub;
    ba.a.lam_prev = c->lpb;
    ba.a.h = c->hb;
    ba.a.lam_hat = c->davg ? c->lhb : nullptr;
    if (c->eps_mode) {
        ba.gm_b = c->gm_b;
        ba.done_b = c->done_b;
        ba.ndone = c->ndone;
    }
    ba.b.qy = c->QYb;
    ba.b.q = c->qb;
    ba.b.x = c->Xb;
    ba.b.y = c->Yb;
    ba.b.xhat = c->XHb;
    if (pass == 0) {   // [Q;G] (n+p x n) . Y  (paired rows: [Q;G_t], the first n + P rows of [Q;G])
        ba.Aop = c->A;
        ba.lda = c->ld;
        ba.M = c->n + (c->pairP ? c->pairP : c->p);
        ba.Bop = c->Yb;
        ba.ldb = c->ld;
        ba.K = c->ld;
    } else {           // G' (n x p) . W  (paired rows: G_t' . D over the first ldd columns of G'; D's
                       // zero padding cancels the bottom rows' columns P .. ldd - 1)
        ba.Aop = c->GT;
        ba.lda = c->ldp;
        ba.M = c->n;
        ba.Bop = c->pairP ? c->Db : c->Wb;
        ba.ldb = c->pairP ? c->ldd : ba.sp;
        ba.K = c->pairP ? c->ldd : c->ldp;
    }
    return ba;
}

// Linear operator for Lanczos: out = op(v), v given in the y_full replica.
//   0: (Q + rho G'G) v     1: G'G v     2: Q v
duquad_status apply_op(duquad_ctx *ctx, int op, double *out) {
    PassAArgs a = make_a(ctx);
    PassBArgs b = make_b(ctx);
    duquad_status st;
    if (op == 2) {
        a.row_end = ctx->nloc;
        a.qy = out;
        CK(launch_pass_a(a, MODE_LIN, ctx->cfg_a, ctx->stream));
        return DUQUAD_OK;
    }
    if (op == 1) a.row_begin = ctx->nloc;
    a.lin_coef = op == 0 ? ctx->rho : 1.0;
    CK(launch_pass_a(a, MODE_LIN, ctx->cfg_a, ctx->stream));
    if ((st = allgather_w(ctx)) != DUQUAD_OK) return st;
    b.use_qy = op == 0 ? 1 : 0;
    b.out = out;
    CK(launch_pass_b(b, MODE_LIN, ctx->cfg_b, ctx->stream));
    return DUQUAD_OK;
}

// largest eigenvalue of the symmetric tridiagonal (alpha[0..m-1], beta[0..m-2]) by Sturm bisection
double tridiag_max_eig(const std::vector<double> &al, const std::vector<double> &be, int m) {
    double lo = 1e300, hi = -1e300;
    for (int i = 0; i < m; ++i) {
        const double r = (i > 0 ? std::fabs(be[i - 1]) : 0.0) + (i < m - 1 ? std::fabs(be[i]) : 0.0);
        lo = std::min(lo, al[i] - r);
        hi = std::max(hi, al[i] + r);
    }
    auto count_below = [&](double x) {   // number of eigenvalues < x
        int cnt = 0;
        double d = 1.0;
        for (int i = 0; i < m; ++i) {
            const double b2 = i > 0 ? be[i - 1] * be[i - 1] : 0.0;
            d = (al[i] - x) - (i > 0 ? b2 / d : 0.0);
            if (d == 0.0) d = -1e-300;
            if (d < 0) ++cnt;
        }
        return cnt;
    };
    for (int it = 0; it < 200 && hi - lo > 1e-15 * std::max(std::fabs(lo), std::fabs(hi)); ++it) {
        const double mid = 0.5 * (lo + hi);
        if (count_below(mid) >= m)
            hi = mid;
        else
            lo = mid;
    }
    return hi;
}

duquad_status lanczos_max(duquad_ctx *ctx, int op, int iters, double *out) {
    if (iters < 1) iters = 1;
    if (iters > kMaxLanczos) iters = kMaxLanczos;
    double *v = ctx->y_full + ctx->rank * ctx->n_slice;   // local slice of the replica
    double *sc = ctx->scal;
    duquad_status st;
    const int64_t nl = ctx->nloc;
    CK(cudaMemsetAsync(ctx->y_full, 0, ctx->ylen * sizeof(double), ctx->stream));
    CK(cudaMemsetAsync(ctx->lz_vprev, 0, std::max<int64_t>(nl, 1) * sizeof(double), ctx->stream));
    CK(cudaMemsetAsync(sc, 0, SC_NSCAL * sizeof(double), ctx->stream));
    CK(launch_fill_hash(v, nl, ctx->r0, ctx->stream));
    CK(launch_dot_partial(v, v, nl, ctx->partials, ctx->stream));
    CK(launch_reduce_final(ctx->partials, kRedGrid, 1, sc + SC_TMP, ctx->stream));
    if ((st = allreduce_sum(ctx, sc + SC_TMP, 1)) != DUQUAD_OK) return st;
    CK(launch_scale_by_rsqrt(v, nl, sc + SC_TMP, nullptr, ctx->stream));
    int m = 0;
    for (int it = 0; it < iters; ++it) {
        if ((st = allgather_y(ctx)) != DUQUAD_OK) return st;
        if ((st = apply_op(ctx, op, ctx->lz_w)) != DUQUAD_OK) return st;
        CK(launch_dot_partial(v, ctx->lz_w, nl, ctx->partials, ctx->stream));
        CK(launch_reduce_final(ctx->partials, kRedGrid, 1, sc + SC_ALPHA + it, ctx->stream));
        if ((st = allreduce_sum(ctx, sc + SC_ALPHA + it, 1)) != DUQUAD_OK) return st;
        // beta_0 = 0 lives in sc[SC_BETA + kMaxLanczos] (zeroed)
        const double *beta_prev = it == 0 ? sc + SC_TMP2 : sc + SC_BETA + it - 1;
        CK(launch_lanczos_update(ctx->lz_w, v, ctx->lz_vprev, nl, sc + SC_ALPHA + it, beta_prev,
                                 ctx->partials, ctx->stream));
        CK(launch_reduce_final(ctx->partials, kRedGrid, 1, sc + SC_TMP, ctx->stream));
        if ((st = allreduce_sum(ctx, sc + SC_TMP, 1)) != DUQUAD_OK) return st;
        CK(launch_lanczos_next(v, ctx->lz_vprev, ctx->lz_w, nl, sc + SC_TMP, sc + SC_BETA + it,
                               ctx->stream));
        m = it + 1;
    }
    std::vector<double> al(m), be(m);
    CK(cudaMemcpyAsync(al.data(), sc + SC_ALPHA, m * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(be.data(), sc + SC_BETA, m * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    // stop at an invariant subspace (beta ~ 0)
    int mm = m;
    double amax = 0.0;
    for (int i = 0; i < m; ++i) amax = std::max(amax, std::fabs(al[i]));
    for (int i = 0; i < m - 1; ++i)
        if (!(std::fabs(be[i]) > 1e-14 * std::max(amax, 1e-300))) {
            mm = i + 1;
            break;
        }
    *out = tridiag_max_eig(al, be, mm);
    return DUQUAD_OK;
}

// Host-side finiteness scan of a rows x cols block (leading dim ld); large blocks are split over
// up to 16 host threads (config 2's 3.2 GB of Q and G took ~0.4 s single-threaded).
bool finite_host(const double *v, int64_t rows, int64_t cols, int64_t ld) {
    auto scan = [&](int64_t r0, int64_t r1) {
        for (int64_t r = r0; r < r1; ++r)
            for (int64_t c = 0; c < cols; ++c)
                if (!std::isfinite(v[r * ld + c])) return false;
        return true;
    };
    const int64_t work = rows * cols;
    const int nt = (int)std::min<int64_t>({16, std::max<int64_t>(1, work >> 22), std::max<int64_t>(rows, 1),
                                            (int64_t)std::max(1u, std::thread::hardware_concurrency())});
    if (nt <= 1) return scan(0, rows);
    std::vector<char> ok((size_t)nt, 1);
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
        th.emplace_back([&, t] { ok[(size_t)t] = scan(rows * t / nt, rows * (t + 1) / nt); });
    for (auto &x : th) x.join();
    for (char c : ok)
        if (!c) return false;
    return true;
}

duquad_status upload_vec(duquad_ctx *ctx, double *dst, const double *src, int64_t count) {
    if (count <= 0) return DUQUAD_OK;
    CK(cudaMemcpyAsync(dst, src, count * sizeof(double), cudaMemcpyDefault, ctx->stream));
    return DUQUAD_OK;
}

// CSR setup: device copies of Q and G (validated), the stacked local [Q_r; G_r]
// and the local rows of G' (device transpose, deterministic order).
// Programmatic dependent launch for the inner-step kernels (options.pdl; DUQUAD_PDL=0 / =2 force it
// off / on for measurements): a kernel's launch and prologue overlap its predecessor's tail
// (epilogue.cuh pdl_wait).  Measured (profiles/r02_pdl_ab.jsonl): config 1 (dense two-pass, L2-
// resident, launch-bound) 11.7 -> 10.1 us per step; the sparse lane kernels 75.6 -> 78.0 us (their
// waiting CTAs take the slots of the grid-stride waves), so CSR contexts launch plainly.
void apply_pdl(duquad_ctx *ctx) {
    const char *ev = getenv("DUQUAD_PDL");
    int on = ctx->opt.pdl && ctx->format != DUQUAD_CSR ? 1 : 0;
    if (ev) on = atoi(ev) == 2 ? 1 : atoi(ev) == 0 ? 0 : on;
    ctx->cfg_a.pdl = ctx->cfg_b.pdl = ctx->cfg_k3.pdl = on;
    ctx->fz.pdl = on;
}

// Lane-per-row kernels serve matrices whose mean row length is at most kLaneMaxMean; among them
// SELL-32 is used when its padded layout holds at most kSellMaxPad x the nonzeros
constexpr double kLaneMaxMean = 48.0, kSellMaxPad = 1.15;

duquad_status setup_csr(duquad_ctx *ctx, const duquad_problem *prob) {
    cudaStream_t s = ctx->stream;
    const int64_t n = ctx->n, p = ctx->p;
    const int64_t qnnz = prob->Q_nnz, gnnz = p > 0 ? prob->G_nnz : 0;
    std::vector<void *> tmp;
    struct Freer {
        std::vector<void *> &v;
        ~Freer() {
            for (void *q : v) cudaFree(q);
        }
    } freer{tmp};
    auto dev_copy = [&](const void *src, size_t bytes, const void **dst) -> cudaError_t {
        if (prob->on_device) {
            *dst = src;
            return cudaSuccess;
        }
        void *d = nullptr;
        cudaError_t e = cudaMalloc(&d, std::max<size_t>(bytes, 8));
        if (e) return e;
        tmp.push_back(d);
        *dst = d;
        return bytes ? cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, s) : cudaSuccess;
    };
    const int32_t *Qrp, *Qci, *Grp = nullptr, *Gci = nullptr;
    const double *Qva, *Gva = nullptr;
    CK(dev_copy(prob->Q_rowptr, (n + 1) * 4, (const void **)&Qrp));
    CK(dev_copy(prob->Q_col, qnnz * 4, (const void **)&Qci));
    CK(dev_copy(prob->Q_val, qnnz * 8, (const void **)&Qva));
    if (p > 0) {
        CK(dev_copy(prob->G_rowptr, (p + 1) * 4, (const void **)&Grp));
        CK(dev_copy(prob->G_col, gnnz * 4, (const void **)&Gci));
        CK(dev_copy(prob->G_val, gnnz * 8, (const void **)&Gva));
    }
    CK(cudaMemsetAsync(ctx->d_flag, 0, sizeof(int32_t), s));
    CK(launch_check_csr(Qrp, Qci, Qva, n, n, qnnz, ctx->d_flag, s));
    if (p > 0) CK(launch_check_csr(Grp, Gci, Gva, p, n, gnnz, ctx->d_flag, s));
    int32_t flag = 0;
    CK(cudaMemcpyAsync(&flag, ctx->d_flag, sizeof(flag), cudaMemcpyDeviceToHost, s));
    int32_t qb[2] = {0, 0}, gb[2] = {0, 0};
    CK(cudaMemcpyAsync(&qb[0], Qrp + ctx->r0, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&qb[1], Qrp + ctx->r0 + ctx->nloc, 4, cudaMemcpyDeviceToHost, s));
    if (p > 0) {
        CK(cudaMemcpyAsync(&gb[0], Grp + ctx->s0, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&gb[1], Grp + ctx->s0 + ctx->ploc, 4, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    if (flag) return fail(ctx, DUQUAD_EINVAL, "invalid CSR data (row pointers, column range or non-finite value)");
    {   // Q symmetric: Q' (device transpose of the full Q) has Q's pattern and values
        int32_t *trp = nullptr, *tci = nullptr;
        double *tva = nullptr;
        int64_t tnnz = 0;
        cudaError_t e = csr_transpose_rows(Qrp, Qci, Qva, n, n, qnnz, 0, n, &trp, &tci, &tva, &tnnz, s);
        if (e == cudaSuccess) e = launch_csr_sym_cmp(Qrp, Qci, Qva, trp, tci, tva, n, qnnz, ctx->d_flag, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&flag, ctx->d_flag, sizeof(flag), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        cudaFree(trp);
        cudaFree(tci);
        cudaFree(tva);
        CK(e);
        if (flag || tnnz != qnnz)
            return fail(ctx, DUQUAD_EINVAL,
                        "Q must be symmetric (PAPER.md:199): the CSR pattern and values of Q and Q' must agree "
                        "(|Q_ij - Q_ji| <= 1e-12 (|Q_ij| + |Q_ji|); store both triangles)");
    }
    const int64_t nq = qb[1] - qb[0], ng = gb[1] - gb[0];
    ctx->nnz_a = nq + ng;
    CK(dalloc(&ctx->a_rp, ctx->nloc + ctx->ploc + 1));
    CK(dalloc(&ctx->a_ci, ctx->nnz_a));
    CK(dalloc(&ctx->a_va, ctx->nnz_a));
    CK(launch_rebase(ctx->a_rp, Qrp + ctx->r0, ctx->nloc + 1, qb[0], 0, s));
    if (ctx->ploc > 0) CK(launch_rebase(ctx->a_rp + ctx->nloc, Grp + ctx->s0, ctx->ploc + 1, gb[0], (int32_t)nq, s));
    if (nq) {
        CK(cudaMemcpyAsync(ctx->a_ci, Qci + qb[0], nq * 4, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(ctx->a_va, Qva + qb[0], nq * 8, cudaMemcpyDeviceToDevice, s));
    }
    if (ng) {
        CK(cudaMemcpyAsync(ctx->a_ci + nq, Gci + gb[0], ng * 4, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(ctx->a_va + nq, Gva + gb[0], ng * 8, cudaMemcpyDeviceToDevice, s));
    }
    if (p > 0) {
        CK(csr_transpose_rows(Grp, Gci, Gva, p, n, gnnz, ctx->r0, ctx->nloc, &ctx->b_rp, &ctx->b_ci, &ctx->b_va,
                              &ctx->nnz_b, s));
    } else {
        CK(dalloc(&ctx->b_rp, ctx->nloc + 1));
        CK(dalloc(&ctx->b_ci, 1));
        CK(dalloc(&ctx->b_va, 1));
    }
    // group sizes from the GLOBAL mean nnz per row (identical on every rank)
    ctx->gs_a = csr_group_size((double)(qnnz + gnnz) / (double)(n + p));
    ctx->gs_b = csr_group_size((double)gnnz / (double)n);
    CK(cudaStreamSynchronize(s));
    // Lane-per-row kernels for short rows (kernels_sell.cu).  Lane kernels vs the sub-warp kernels
    // sum a row in different orders, so that choice uses GLOBAL statistics (every rank alike); the
    // lane layout (SELL-32 when it pads little, else thread-per-row CSR) is per rank: both sum
    // each row in CSR order, so the results do not depend on it.
    auto lane_choice = [&](const int32_t *rp, const int32_t *ci, const double *va, int64_t rows, int64_t nq,
                           int64_t nnz_loc, double mean, SellStore *st, int *kind, int *u) -> duquad_status {
        *kind = SPK_CSR;
        if (!ctx->opt.sell_path || mean > kLaneMaxMean) return DUQUAD_OK;
        SparsePlan pl;
        CK(sparse_plan(rp, rows, nq, &pl, s));
        if ((double)pl.padded <= kSellMaxPad * (double)nnz_loc + 1024.0 && pl.max_len <= 64) {
            CK(sell_build(rp, ci, va, rows, nq, pl, st, s));
            *kind = SPK_SELL;
            *u = lane_unroll(SPK_SELL, pl.max_len, mean);
        } else {
            *kind = SPK_ROWT;
            *u = lane_unroll(SPK_ROWT, pl.max_len, mean);
        }
        return DUQUAD_OK;
    };
    duquad_status st;
    if ((st = lane_choice(ctx->a_rp, ctx->a_ci, ctx->a_va, ctx->nloc + ctx->ploc, ctx->nloc, ctx->nnz_a,
                          (double)(qnnz + gnnz) / (double)(n + p), &ctx->sell_a, &ctx->kind_a, &ctx->u_a)) != DUQUAD_OK)
        return st;
    if (p > 0 && (st = lane_choice(ctx->b_rp, ctx->b_ci, ctx->b_va, ctx->nloc, ctx->nloc, ctx->nnz_b,
                                   (double)gnnz / (double)n, &ctx->sell_b, &ctx->kind_b, &ctx->u_b)) != DUQUAD_OK)
        return st;
    // measurement overrides (scripts/sparse_sweep.py): kind / load-round width per pass
    auto env_int = [](const char *k, int d) { const char *v = getenv(k); return v ? atoi(v) : d; };
    // banded Q (config 4: 11 diagonals): pass A reads the Q rows as diagonals -- no column indices,
    // every load coalesced (8 instead of 12 bytes per nonzero); for a symmetric band only its upper
    // half is stored and streamed (6 of config 4's 11 diagonals), the lower half re-read from it
    if (ctx->kind_a == SPK_SELL && ctx->nloc > 0 && env_int("DUQUAD_DIA", 1))
        CK(dia_build(ctx->a_rp, ctx->a_ci, ctx->a_va, ctx->nloc, ctx->r0, n, nq, 1.15, env_int("DUQUAD_DIA_SYM", 1) != 0,
                     &ctx->dia, &ctx->dia_val, s));
    if (ctx->kind_a == SPK_ROWT || (ctx->kind_a == SPK_SELL && env_int("DUQUAD_SPK_A", 1) == SPK_ROWT)) {
        ctx->kind_a = SPK_ROWT;
        ctx->u_a = env_int("DUQUAD_LANE_UA", ctx->u_a == 4 ? 4 : 8) <= 4 ? 4 : 8;
    } else if (ctx->kind_a == SPK_SELL) {
        // with the Q rows in DIA form only the G slices use U: rounds of 8 (one per config-4 G row)
        // measured 0.3-0.6 us faster per step than 4 (r02_c4_ua_mix.txt)
        ctx->u_a = env_int("DUQUAD_LANE_UA", ctx->dia.nd > 0 ? 8 : ctx->u_a);
    }
    if (ctx->kind_b == SPK_ROWT) ctx->u_b = env_int("DUQUAD_LANE_UB", ctx->u_b) <= 4 ? 4 : 8;
    return DUQUAD_OK;
}

}  // namespace

// ======================================================================= ABI
extern "C" {

int32_t duquad_abi_version(void) { return DUQUAD_ABI_VERSION; }

int64_t duquad_struct_size(int32_t which) {
    switch (which) {
        case 0: return (int64_t)sizeof(duquad_problem);
        case 1: return (int64_t)sizeof(duquad_options);
        case 2: return (int64_t)sizeof(duquad_result);
        case 3: return (int64_t)sizeof(duquad_schedule);
        case 4: return (int64_t)sizeof(duquad_bounds);
        case 5: return (int64_t)sizeof(duquad_monitor);
        default: return -1;
    }
}

const char *duquad_status_string(int32_t s) {
    switch (s) {
        case DUQUAD_OK: return "ok";
        case DUQUAD_EINVAL: return "invalid argument";
        case DUQUAD_ENOMEM: return "out of memory";
        case DUQUAD_ECUDA: return "CUDA error";
        case DUQUAD_ENCCL: return "NCCL error";
        case DUQUAD_ENONFINITE: return "non-finite iterate";
        case DUQUAD_ENODEV: return "no suitable CUDA device";
        case DUQUAD_ESTATE: return "call out of order";
        case DUQUAD_EMAXITER: return "inner iteration cap reached (result valid)";
        default: return "unknown status";
    }
}

void duquad_default_options(duquad_options *o) {
    if (!o) return;
    std::memset(o, 0, sizeof(*o));
    o->dual_step_scale = 0.5;
    o->project_dual = 1;
    o->inner_rule = DUQUAD_INNER_FGM;
    o->sigma = 0.0;
    o->lambda_min_lb = 0.0;
    o->l_mode = 0;
    o->use_graphs = 1;
    o->world_size = 1;
    o->rank = 0;
    o->nccl_id = nullptr;
    o->stream = nullptr;
    o->device = -1;
    o->time_passes = 0;
    o->small_path = 1;
    o->rho0_path = 1;
    o->emulate_ranks = 0;
    o->fused_path = 1;
    o->persist_path = 0;
    o->dual_average = 0;
    o->eq_precompute = 1;
    o->checkpoint = 0;
    o->nccl_self = 0;
    o->sell_path = 1;
    o->pair_rows = 1;
    o->pdl = 1;
}

duquad_status duquad_shard_range(int64_t rows, int32_t world, int32_t rank, int64_t *begin,
                                 int64_t *end) {
    if (rows < 0 || world < 1 || rank < 0 || rank >= world || !begin || !end)
        return fail(nullptr, DUQUAD_EINVAL, "duquad_shard_range: bad arguments");
    const int64_t slice = (rows + world - 1) / world;
    *begin = std::min<int64_t>(rows, (int64_t)rank * slice);
    *end = std::min<int64_t>(rows, *begin + slice);
    return DUQUAD_OK;
}

duquad_status duquad_nccl_unique_id(void *out128) {
    duquad_ctx *ctx = nullptr;
    if (!out128) return fail(nullptr, DUQUAD_EINVAL, "null output");
    ncclUniqueId id;
    NK(ncclGetUniqueId(&id));
    std::memcpy(out128, &id, sizeof(id));
    return DUQUAD_OK;
}

const char *duquad_last_error(const duquad_ctx *ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

void duquad_destroy(duquad_ctx *ctx) {
    if (!ctx) return;
    {
        DevGuard guard(ctx->dev);
        if (ctx->stream) cudaStreamSynchronize(ctx->stream);
        free_all(ctx);
    }
    delete ctx;
}

duquad_status duquad_setup(duquad_ctx **out, const duquad_problem *prob, double rho,
                           const duquad_options *opts_in) {
    if (!out) return fail(nullptr, DUQUAD_EINVAL, "out is NULL");
    *out = nullptr;
    if (!prob) return fail(nullptr, DUQUAD_EINVAL, "prob is NULL");
    duquad_options opt;
    duquad_default_options(&opt);
    if (opts_in) opt = *opts_in;
    const int64_t n = prob->n, p = prob->p;
    if (n < 1 || p < 0) return fail(nullptr, DUQUAD_EINVAL, "need n >= 1 and p >= 0");
    if (!(rho >= 0.0) || !std::isfinite(rho)) return fail(nullptr, DUQUAD_EINVAL, "rho must be finite and >= 0");
    if (prob->batch < 1) return fail(nullptr, DUQUAD_EINVAL, "batch must be >= 1");
    const bool batched = prob->batch > 1;
    if (batched && prob->format != DUQUAD_DENSE) return fail(nullptr, DUQUAD_EINVAL, "batch > 1 needs dense Q, G");
    if (batched && (n > 27000 || p > 27000)) return fail(nullptr, DUQUAD_EINVAL, "batched path: n, p too large");
    const bool csr = prob->format == DUQUAD_CSR;
    if (prob->format != DUQUAD_DENSE && !csr) return fail(nullptr, DUQUAD_EINVAL, "bad format");
    if (!prob->q || !prob->lb || !prob->ub || (p > 0 && !prob->g))
        return fail(nullptr, DUQUAD_EINVAL, "missing problem vector");
    if (!csr && (!prob->Q || (p > 0 && !prob->G))) return fail(nullptr, DUQUAD_EINVAL, "missing problem matrix");
    if (csr && (!prob->Q_rowptr || !prob->Q_col || !prob->Q_val ||
                (p > 0 && (!prob->G_rowptr || !prob->G_col || !prob->G_val)) || prob->Q_nnz < 0 ||
                prob->G_nnz < 0 || prob->Q_nnz > INT32_MAX || prob->G_nnz > INT32_MAX))
        return fail(nullptr, DUQUAD_EINVAL, "missing or oversized CSR array (int32 indices)");
    if (!csr && (prob->ldQ < n || (p > 0 && prob->ldG < n)))
        return fail(nullptr, DUQUAD_EINVAL, "leading dimension < n");
    if (!prob->cone && prob->cone_all != DUQUAD_CONE_ZERO && prob->cone_all != DUQUAD_CONE_NONPOS)
        return fail(nullptr, DUQUAD_EINVAL, "bad cone_all");
    if (!(opt.dual_step_scale > 0.0)) return fail(nullptr, DUQUAD_EINVAL, "dual_step_scale must be > 0");
    if (opt.inner_rule < 0 || opt.inner_rule > 2) return fail(nullptr, DUQUAD_EINVAL, "bad inner_rule");
    if (opt.inner_rule == DUQUAD_INNER_FGM_SIGMA && !(opt.sigma > 0.0))
        return fail(nullptr, DUQUAD_EINVAL, "FGM_SIGMA needs sigma > 0");
    if (opt.world_size < 1 || opt.rank < 0 || opt.rank >= opt.world_size)
        return fail(nullptr, DUQUAD_EINVAL, "bad world_size / rank");
    if (opt.world_size > 1 && !batched && !opt.nccl_id && !opt.emulate_ranks)
        return fail(nullptr, DUQUAD_EINVAL, "row-sharded setup needs nccl_id");
    // host data: validate here (device data is validated by a kernel); a single rank's dense Q and G
    // are checked on the device after their upload instead (3.2 GB at config 2: a host scan costs
    // tens of ms of every end-to-end solve, the device check ~1 ms)
    int ndev0 = 0;
    if (cudaGetDeviceCount(&ndev0) != cudaSuccess) ndev0 = 0;
    const bool qg_dev_check = !prob->on_device && !csr && opt.world_size == 1 && ndev0 > 0;
    if (!prob->on_device) {
        if ((!csr && !qg_dev_check &&
             (!finite_host(prob->Q, n, n, prob->ldQ) || (p > 0 && !finite_host(prob->G, p, n, prob->ldG)))) ||
            !finite_host(prob->q, prob->batch, n, n) || (p > 0 && !finite_host(prob->g, prob->batch, p, p)))
            return fail(nullptr, DUQUAD_EINVAL, "non-finite problem data");
        for (int64_t i = 0; i < n; ++i)
            if (std::isnan(prob->lb[i]) || std::isnan(prob->ub[i]) || prob->lb[i] > prob->ub[i] ||
                prob->lb[i] == INFINITY || prob->ub[i] == -INFINITY)
                return fail(nullptr, DUQUAD_EINVAL, "box needs lb <= ub (lb < +inf, ub > -inf)");
        if (prob->cone)
            for (int64_t i = 0; i < p; ++i)
                if (prob->cone[i] > 1) return fail(nullptr, DUQUAD_EINVAL, "bad cone tag");
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(nullptr, DUQUAD_ENODEV, "no CUDA device");
    duquad_ctx *ctx = new duquad_ctx();
    ctx->opt = opt;
    ctx->n = n;
    ctx->p = p;
    ctx->rho = rho;
    ctx->format = prob->format;
    if (opt.device >= 0)
        ctx->dev = opt.device;
    else
        cudaGetDevice(&ctx->dev);
    DevGuard guard(ctx->dev);
    auto bail = [&](duquad_status st) {
        g_err = ctx->err;
        duquad_destroy(ctx);
        return st;
    };
#define CKS(call)                                                                        \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess) {                                                         \
            ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);               \
            return bail(e_ == cudaErrorMemoryAllocation ? DUQUAD_ENOMEM : DUQUAD_ECUDA); \
        }                                                                                \
    } while (0)
    cudaDeviceProp prop;
    CKS(cudaGetDeviceProperties(&prop, ctx->dev));
    if (prop.major != 10) {
        ctx->err = std::string("device is not sm_100 (got sm_") + std::to_string(prop.major) +
                   std::to_string(prop.minor) + ")";
        return bail(DUQUAD_ENODEV);
    }
    ctx->num_sms = prop.multiProcessorCount;
    if (opt.stream) {
        ctx->stream = (cudaStream_t)opt.stream;
    } else {
        CKS(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        ctx->own_stream = true;
    }
    // ---- sharding: rows of one QP over the ranks (NCCL), or, batched, whole QPs (no collective)
    ctx->world = batched ? 1 : opt.world_size;
    ctx->rank = batched ? 0 : opt.rank;
    ctx->sharded = ctx->world > 1 || (opt.nccl_self && !batched);
    ctx->Btot = prob->batch;
    {
        const int64_t bs = (prob->batch + opt.world_size - 1) / opt.world_size;
        ctx->b0 = std::min<int64_t>(prob->batch, (int64_t)opt.rank * bs);
        ctx->Bloc = std::min<int64_t>(prob->batch, ctx->b0 + bs) - ctx->b0;
    }
    ctx->n_slice = (n + ctx->world - 1) / ctx->world;
    ctx->p_slice = (p + ctx->world - 1) / ctx->world;
    ctx->r0 = std::min<int64_t>(n, ctx->rank * ctx->n_slice);
    ctx->nloc = std::min<int64_t>(n, ctx->r0 + ctx->n_slice) - ctx->r0;
    // G rows: equal slices, except for the row-sharded byte floor, where rank r's triangle slab of Q
    // (rows r0..r0+nloc, columns >= row) shrinks with r: there the G rows are split so that every
    // rank streams the same number of matrix elements (slab + G rows x n), contiguous and ascending
    ctx->floor_shard = ctx->sharded && !csr && !batched && rho > 0.0 && p > 0 && opt.fused_path &&
                       fused_supported(n, round_up(n, 32), prop.sharedMemPerBlockOptin);
    ctx->gs0.assign(ctx->world, 0);
    ctx->gcnt.assign(ctx->world, 0);
    if (ctx->floor_shard) {
        std::vector<double> want(ctx->world);
        double tot = (double)p * (double)n;
        std::vector<double> slab(ctx->world);
        for (int r = 0; r < ctx->world; ++r) {
            const double qa = (double)std::min<int64_t>(n, r * ctx->n_slice);
            const double qb = (double)std::min<int64_t>(n, (r + 1) * ctx->n_slice);
            slab[r] = (qb - qa) * (double)n - 0.5 * (qb * qb - qa * qa) + 0.5 * (qb - qa);
            tot += slab[r];
        }
        double sw = 0.0;
        for (int r = 0; r < ctx->world; ++r) sw += (want[r] = std::max(0.0, (tot / ctx->world - slab[r]) / n));
        int64_t given = 0;
        std::vector<std::pair<double, int>> frac;
        for (int r = 0; r < ctx->world; ++r) {
            const double x = sw > 0.0 ? want[r] * (double)p / sw : (double)p / ctx->world;
            ctx->gcnt[r] = (int64_t)std::floor(x);
            given += ctx->gcnt[r];
            frac.push_back({-(x - std::floor(x)), r});
        }
        std::sort(frac.begin(), frac.end());
        for (int64_t i = 0; given < p; ++i, ++given) ++ctx->gcnt[frac[(size_t)(i % ctx->world)].second];
        for (int r = 1; r < ctx->world; ++r) ctx->gs0[r] = ctx->gs0[r - 1] + ctx->gcnt[r - 1];
    } else {
        for (int r = 0; r < ctx->world; ++r) {
            ctx->gs0[r] = std::min<int64_t>(p, r * ctx->p_slice);
            ctx->gcnt[r] = std::min<int64_t>(p, ctx->gs0[r] + ctx->p_slice) - ctx->gs0[r];
        }
    }
    ctx->s0 = ctx->gs0[ctx->rank];
    ctx->ploc = ctx->gcnt[ctx->rank];
    ctx->emulated = ctx->world > 1 && opt.emulate_ranks;
    if (ctx->sharded && !ctx->emulated) {
        ncclUniqueId id;
        ncclResult_t r = ncclSuccess;
        if (ctx->world == 1)   // nccl_self: a one-rank communicator of our own
            r = ncclGetUniqueId(&id);
        else
            std::memcpy(&id, opt.nccl_id, sizeof(id));
        if (r == ncclSuccess) r = ncclCommInitRank(&ctx->comm, ctx->world, id, ctx->rank);
        if (r != ncclSuccess) {
            ctx->err = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
            return bail(DUQUAD_ENCCL);
        }
    }
    // ---- layout: 256-byte aligned rows, vectors zero-padded
    ctx->ld = round_up(n, 32);
    ctx->ldp = round_up(std::max<int64_t>(p, 1), 32);
    if (p == 0) ctx->ldp = 0;
    ctx->ylen = round_up(std::max(ctx->ld, ctx->world * ctx->n_slice), 32);
    ctx->wlen = round_up(std::max(ctx->ldp, ctx->world * ctx->p_slice), 32);
    const int64_t rows = ctx->nloc + ctx->ploc;
    if (!csr) {
        CKS(dalloc(&ctx->A, rows * ctx->ld));
        CKS(dalloc(&ctx->GT, ctx->nloc * std::max<int64_t>(ctx->ldp, 1)));
    }
    CKS(dalloc(&ctx->y_full, ctx->ylen));
    CKS(dalloc(&ctx->w_full, ctx->wlen));
    CKS(dalloc(&ctx->qy, ctx->nloc));
    CKS(dalloc(&ctx->x, ctx->nloc));
    CKS(dalloc(&ctx->xhat, ctx->nloc));
    CKS(dalloc(&ctx->q, ctx->nloc));
    CKS(dalloc(&ctx->lb, ctx->nloc));
    CKS(dalloc(&ctx->ub, ctx->nloc));
    CKS(dalloc(&ctx->lz_vprev, ctx->nloc));
    CKS(dalloc(&ctx->lz_w, ctx->nloc));
    CKS(dalloc(&ctx->g, ctx->ploc));
    CKS(dalloc(&ctx->mu, ctx->ploc));
    CKS(dalloc(&ctx->lam_prev, ctx->ploc));
    CKS(dalloc(&ctx->cone, (ctx->ploc + 7) / 8 * 8));   // whole 32-bit words (the byte floor reads cone words)
    CKS(dalloc(&ctx->scal, SC_NSCAL));
    CKS(dalloc(&ctx->partials, kRedGrid * 8));
    CKS(dalloc(&ctx->d_j, 4));
    CKS(dalloc(&ctx->d_flag, 4));
    cudaStream_t s = ctx->stream;
    // Device inputs may still be in flight on another stream of the caller (e.g. torch's):
    // wait for the whole device before reading them (setup is not on the hot path).
    if (prob->on_device) CKS(cudaDeviceSynchronize());
    // ---- pack [Q_r; G_r] and G'_r
    if (csr) {
        duquad_status st = setup_csr(ctx, prob);
        if (st != DUQUAD_OK) return bail(st);
    } else {
    CKS(cudaMemcpy2DAsync(ctx->A, ctx->ld * sizeof(double), prob->Q + ctx->r0 * prob->ldQ,
                          prob->ldQ * sizeof(double), n * sizeof(double), ctx->nloc, cudaMemcpyDefault, s));
    if (p > 0) {
        if (ctx->ploc > 0)
            CKS(cudaMemcpy2DAsync(ctx->A + ctx->nloc * ctx->ld, ctx->ld * sizeof(double),
                                  prob->G + ctx->s0 * prob->ldG, prob->ldG * sizeof(double),
                                  n * sizeof(double), ctx->ploc, cudaMemcpyDefault, s));
        // G' rows r0..r0+nloc = columns r0.. of G; stage G on the device when it is on the host
        // (a rank holding every G row transposes its own device copy: no second upload)
        const double *Gd = prob->G;
        double *Gtmp = nullptr;
        const bool g_local = !prob->on_device && ctx->s0 == 0 && ctx->ploc == p;
        if (g_local) Gd = ctx->A + ctx->nloc * ctx->ld;
        if (!prob->on_device && !g_local) {
            CKS(cudaMalloc(&Gtmp, (size_t)p * n * sizeof(double)));
            CKS(cudaMemcpy2DAsync(Gtmp, n * sizeof(double), prob->G, prob->ldG * sizeof(double),
                                  n * sizeof(double), p, cudaMemcpyHostToDevice, s));
            Gd = Gtmp;
        }
        cudaError_t e = launch_transpose(Gd, prob->on_device ? prob->ldG : g_local ? ctx->ld : n, p, ctx->r0,
                                         ctx->nloc, ctx->GT, ctx->ldp, s);
        if (Gtmp) {
            cudaStreamSynchronize(s);
            cudaFree(Gtmp);
        }
        CKS(e);
    }
    }  // dense
    if (upload_vec(ctx, ctx->q, prob->q + ctx->r0, ctx->nloc) ||
        upload_vec(ctx, ctx->lb, prob->lb + ctx->r0, ctx->nloc) ||
        upload_vec(ctx, ctx->ub, prob->ub + ctx->r0, ctx->nloc) ||
        (p > 0 && upload_vec(ctx, ctx->g, prob->g + ctx->s0, ctx->ploc)))
        return bail(DUQUAD_ECUDA);
    if (ctx->nloc > 0) {   // a box with scalar bounds (every lb_j, ub_j equal): the epilogues skip their loads
        std::vector<double> hl(ctx->nloc), hu(ctx->nloc);
        CKS(cudaMemcpyAsync(hl.data(), ctx->lb, ctx->nloc * sizeof(double), cudaMemcpyDeviceToHost, s));
        CKS(cudaMemcpyAsync(hu.data(), ctx->ub, ctx->nloc * sizeof(double), cudaMemcpyDeviceToHost, s));
        CKS(cudaStreamSynchronize(s));
        bool uni = true;
        for (int64_t i = 1; i < ctx->nloc && uni; ++i)
            uni = std::memcmp(&hl[i], &hl[0], sizeof(double)) == 0 && std::memcmp(&hu[i], &hu[0], sizeof(double)) == 0;
        ctx->box_uniform = uni ? 1 : 0;
        ctx->lb_u = hl[0];
        ctx->ub_u = hu[0];
    }
    if (p > 0 && ctx->ploc > 0) {
        if (prob->cone)
            CKS(cudaMemcpyAsync(ctx->cone, prob->cone + ctx->s0, ctx->ploc, cudaMemcpyDefault, s));
        else
            CKS(cudaMemsetAsync(ctx->cone, prob->cone_all, ctx->ploc, s));
    }
    if (batched) {   // QP-major per-QP vectors of this rank's QPs [b0, b0 + Bloc)
        const int64_t B = ctx->Bloc, lp = std::max<int64_t>(ctx->ldp, 2);
        CKS(dalloc(&ctx->Yb, B * ctx->ld));
        CKS(dalloc(&ctx->Xb, B * ctx->ld));
        CKS(dalloc(&ctx->XHb, B * ctx->ld));
        CKS(dalloc(&ctx->QYb, B * ctx->ld));
        CKS(dalloc(&ctx->qb, B * ctx->ld));
        CKS(dalloc(&ctx->Wb, B * lp));
        CKS(dalloc(&ctx->gb, B * lp));
        CKS(dalloc(&ctx->mub, B * lp));
        CKS(dalloc(&ctx->lpb, B * lp));
        CKS(dalloc(&ctx->hb, B * lp));
        if (B > 0) {
            CKS(cudaMemcpy2DAsync(ctx->qb, ctx->ld * sizeof(double), prob->q + ctx->b0 * n, n * sizeof(double),
                                  n * sizeof(double), B, cudaMemcpyDefault, s));
            if (p > 0)
                CKS(cudaMemcpy2DAsync(ctx->gb, ctx->ldp * sizeof(double), prob->g + ctx->b0 * p, p * sizeof(double),
                                      p * sizeof(double), B, cudaMemcpyDefault, s));
        }
        CKS(configure_batched_kernels());
        // constraint rows in +/- pairs, G = [G_t; -G_t] (two-sided bounds, e.g. config 3's |x_k| <= 5):
        // pass A streams [Q; G_t] and pass B G_t' (w_top - w_bottom) -- the same products (the bottom
        // rows' G u is -(G_t u) exactly), half the G work
        if (opt.pair_rows && p > 0 && p % 2 == 0) {
            const int64_t P = p / 2;
            CKS(cudaMemsetAsync(ctx->d_flag, 0, sizeof(int32_t), s));
            CKS(launch_check_pairs(ctx->A + n * ctx->ld, P, n, ctx->ld, ctx->d_flag, s));
            int32_t flag = 1;
            CKS(cudaMemcpyAsync(&flag, ctx->d_flag, sizeof(flag), cudaMemcpyDeviceToHost, s));
            CKS(cudaStreamSynchronize(s));
            CKS(cudaMemsetAsync(ctx->d_flag, 0, sizeof(int32_t), s));
            if (!flag) {
                ctx->pairP = P;
                ctx->ldd = round_up(P, 32);
                CKS(dalloc(&ctx->Db, B * ctx->ldd));   // zero padding: pass B's K runs to ldd
            }
        }
    }
    if (qg_dev_check) {   // the uploaded [Q;G] of a single rank (host input)
        CKS(cudaMemsetAsync(ctx->d_flag, 0, sizeof(int32_t), s));
        CKS(launch_check(ctx->A, rows, n, ctx->ld, ctx->d_flag, s));
        int32_t flag = 0;
        CKS(cudaMemcpyAsync(&flag, ctx->d_flag, sizeof(flag), cudaMemcpyDeviceToHost, s));
        CKS(cudaStreamSynchronize(s));
        if (flag) {
            ctx->err = "non-finite problem data";
            return bail(DUQUAD_EINVAL);
        }
    }
    if (prob->on_device) {
        CKS(cudaMemsetAsync(ctx->d_flag, 0, sizeof(int32_t), s));
        if (batched) {
            CKS(launch_check(ctx->qb, ctx->Bloc, n, ctx->ld, ctx->d_flag, s));
            if (p > 0) CKS(launch_check(ctx->gb, ctx->Bloc, p, ctx->ldp, ctx->d_flag, s));
        }
        if (!csr) CKS(launch_check(ctx->A, rows, n, ctx->ld, ctx->d_flag, s));
        CKS(launch_check(ctx->q, 1, ctx->nloc, ctx->nloc, ctx->d_flag, s));
        if (ctx->ploc > 0) CKS(launch_check(ctx->g, 1, ctx->ploc, ctx->ploc, ctx->d_flag, s));
        CKS(launch_check_box(ctx->lb, ctx->ub, ctx->nloc, ctx->d_flag, s));
        int32_t flag = 0;
        CKS(cudaMemcpyAsync(&flag, ctx->d_flag, sizeof(flag), cudaMemcpyDeviceToHost, s));
        CKS(cudaStreamSynchronize(s));
        if (flag) {
            ctx->err = "non-finite problem data or lb > ub";
            return bail(DUQUAD_EINVAL);
        }
    }
    if (!csr && n > 0) {   // the byte-floor and small kernels read Q by symmetry
        // A row-sharded rank holds only its rows: check the caller's full Q instead, so that an
        // asymmetric Q is rejected alike on every rank count and every kernel path
        const double *Qs = ctx->A;
        int64_t ldq = ctx->ld;
        double *Qtmp = nullptr;
        if (ctx->nloc != n) {
            if (prob->on_device) {
                Qs = prob->Q;
                ldq = prob->ldQ;
            } else {
                CKS(cudaMalloc(&Qtmp, (size_t)n * n * sizeof(double)));
                CKS(cudaMemcpy2DAsync(Qtmp, n * sizeof(double), prob->Q, prob->ldQ * sizeof(double),
                                      n * sizeof(double), n, cudaMemcpyHostToDevice, s));
                Qs = Qtmp;
                ldq = n;
            }
        }
        CKS(cudaMemsetAsync(ctx->d_flag, 0, sizeof(int32_t), s));
        CKS(launch_check_sym(Qs, n, ldq, ctx->d_flag, s));
        int32_t flag = 0;
        CKS(cudaMemcpyAsync(&flag, ctx->d_flag, sizeof(flag), cudaMemcpyDeviceToHost, s));
        CKS(cudaStreamSynchronize(s));
        if (Qtmp) cudaFree(Qtmp);
        CKS(cudaMemsetAsync(ctx->d_flag, 0, sizeof(int32_t), s));
        if (flag) {
            ctx->err = "Q must be symmetric (PAPER.md:199): |Q_ij - Q_ji| > 1e-12 (|Q_ij| + |Q_ji|)";
            return bail(DUQUAD_EINVAL);
        }
    }
    if (csr) {   // grid-stride sub-warp SpMV / SELL-32 warp-per-slice, full occupancy
        ctx->cfg_a = {ctx->num_sms * (ctx->kind_a != SPK_CSR ? lane_blocks_per_sm(0, ctx->kind_a, ctx->u_a)
                                                             : csr_blocks_per_sm(0, ctx->gs_a)),
                      256, 0};   // whole waves
        ctx->cfg_b = {ctx->num_sms * (ctx->kind_b != SPK_CSR ? lane_blocks_per_sm(1, ctx->kind_b, ctx->u_b)
                                                             : csr_blocks_per_sm(1, ctx->gs_b)),
                      256, 0};
        CKS(cudaStreamSynchronize(s));
        apply_pdl(ctx);
        *out = ctx;
        return DUQUAD_OK;
    }
    // ---- launch configuration: persistent grid, one CTA per SM, vector staged in smem
    const size_t smem_a = (size_t)ctx->ld * sizeof(double);
    const size_t smem_b = (size_t)std::max<int64_t>(ctx->ldp, 2) * sizeof(double);
    if (smem_a > (size_t)prop.sharedMemPerBlockOptin || smem_b > (size_t)prop.sharedMemPerBlockOptin) {
        ctx->err = "dense path needs the vector in shared memory: n and p must be <= " +
                   std::to_string(prop.sharedMemPerBlockOptin / 8);
        return bail(DUQUAD_EINVAL);
    }
    CKS(configure_pass_kernels(smem_a, smem_b));
    const int wpc = pass_threads() / 32;
    ctx->cfg_a = {(int)std::max<int64_t>(1, std::min<int64_t>(ctx->num_sms, (rows + wpc - 1) / wpc)),
                  pass_threads(), smem_a};
    ctx->cfg_b = {(int)std::max<int64_t>(1, std::min<int64_t>(ctx->num_sms, (ctx->nloc + wpc - 1) / wpc)),
                  pass_threads(), smem_b};
    if (!batched && rho == 0.0 && opt.rho0_path) {   // K3: Q-only inner steps
        CKS(dalloc(&ctx->y_full2, ctx->ylen));
        CKS(dalloc(&ctx->cvec, ctx->nloc));
        ctx->cfg_k3 = {ctx->cfg_b.grid, pass_threads(), smem_a};
        ctx->rho0 = true;
    }
    if (!batched && !csr && !ctx->sharded && rho > 0.0 && p > 0 && opt.eq_precompute) {
        // NEXT-3: with every row an equality (K = {0}) the inner gradient is
        // (Q + rho G'G) u + q + G'(mu + rho g): form H once, then the K3 machinery streams H alone.
        bool all_zero = true;
        if (!prob->cone) {
            all_zero = prob->cone_all == DUQUAD_CONE_ZERO;
        } else {
            std::vector<uint8_t> hc((size_t)p);
            CKS(cudaMemcpy(hc.data(), prob->cone, (size_t)p, cudaMemcpyDefault));
            for (uint8_t c : hc) all_zero = all_zero && c == DUQUAD_CONE_ZERO;
        }
        if (all_zero) {
            CKS(dalloc(&ctx->Hq, n * ctx->ld));
            CKS(cudaMemcpyAsync(ctx->Hq, ctx->A, n * ctx->ld * sizeof(double), cudaMemcpyDeviceToDevice, s));
            // column-major view of the G rows: Gc (ld x p), column k = G row k; H += rho Gc Gc'
            cublasHandle_t hb = nullptr;
            if (cublasCreate(&hb) != CUBLAS_STATUS_SUCCESS) {
                ctx->err = "cublasCreate failed";
                return bail(DUQUAD_ECUDA);
            }
            const double alpha = rho, beta = 1.0;
            cublasSetStream(hb, s);
            const cublasStatus_t cs = cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_T, (int)n, (int)n, (int)p, &alpha,
                                                  ctx->A + n * ctx->ld, (int)ctx->ld, ctx->A + n * ctx->ld,
                                                  (int)ctx->ld, &beta, ctx->Hq, (int)ctx->ld);
            cublasDestroy(hb);
            if (cs != CUBLAS_STATUS_SUCCESS) {
                ctx->err = "cublasDgemm (H = Q + rho G'G) failed";
                return bail(DUQUAD_ECUDA);
            }
            CKS(launch_mirror_upper(ctx->Hq, n, ctx->ld, s));   // exactly symmetric: H_ji := H_ij, i < j
            if (!ctx->rho0) {
                CKS(dalloc(&ctx->y_full2, ctx->ylen));
                CKS(dalloc(&ctx->cvec, ctx->nloc));
                ctx->cfg_k3 = {ctx->cfg_b.grid, pass_threads(), smem_a};
            }
            ctx->rho0 = true;
            ctx->eqh = true;
        }
    }
    // byte-floor inner step: single GPU, or row-sharded with rho > 0 (each rank streams the upper
    // triangle of its rows and its G rows; the ranks' partial n-vectors are reduce-scattered)
    const bool shard_floor = ctx->sharded && !csr && rho > 0.0 && !ctx->rho0;
    if (!batched && (!ctx->sharded || shard_floor) && opt.fused_path &&
        fused_supported(n, ctx->ld, prop.sharedMemPerBlockOptin)) {
        const int cg = (!ctx->rho0 && p > 0) ? 2 : 1;   // G role: CTA pairs (148 SMs usable)
        const int nchg = cg > 1 ? fused_nchg(ctx->ld, cg) : 0;
        CKS(configure_fused_kernels(nchg, fused_smem_bytes()));
        const int maxc = fused_max_clusters(nchg, cg, fused_smem_bytes());
        const int nb = std::min(ctx->num_sms / cg, maxc > 0 ? maxc : ctx->num_sms / cg) * cg;
        int nq = nb;                        // rho = 0 (K3) or p = 0: Q role only
        if (cg > 1) {
            // Q : G split by bytes, G weighted by its measured per-byte cost (config 2: nq = 66 of 148)
            double gw = 1.24;
            if (const char *ov = std::getenv("DUQUAD_FUSED_GW")) gw = std::atof(ov);
            const double qa = (double)ctx->r0, qb = (double)(ctx->r0 + ctx->nloc);   // this rank's Q rows
            const double bq = (qb - qa) * (double)n - 0.5 * (qb * qb - qa * qa) + 0.5 * (qb - qa),
                         bg = gw * (double)ctx->ploc * (double)n;
            nq = cg * (int)std::llround((double)nb / cg * bq / (bq + bg));
            nq = std::max(cg, std::min(nb - cg, nq));
        }
        if (const char *ov = std::getenv("DUQUAD_FUSED_NQ")) {   // tuning experiments
            const int v = std::atoi(ov) / cg * cg;
            if (v >= cg && v <= nb && (v < nb || cg == 1)) nq = v;
        }
        double row_cost = 32768.0;          // bytes-equivalent cost of one Q row step (latency-bound: ~a full step)
        if (const char *ov = std::getenv("DUQUAD_FUSED_ROWCOST")) row_cost = std::atof(ov);
        double diag_fac = 1.145, diag_slope = 0.0746;   // diagonal-tile row step: fit to per-CTA times
        if (const char *ov = std::getenv("DUQUAD_FUSED_DIAG")) diag_fac = std::atof(ov);
        if (const char *ov = std::getenv("DUQUAD_FUSED_DSLOPE")) diag_slope = std::atof(ov);
        FusedArgs &fz = ctx->fz;
        fz.n = n;
        fz.p = p;
        fz.ld = ctx->ld;
        fz.nt = fused_tiles(ctx->ld);
        fz.cg = std::max(cg, 2);
        fz.W = fused_block_width(ctx->ld, fz.cg);
        fz.nchg = nchg;
        fz.nb = nb;
        fz.nq_ctas = nq;
        fz.ng = (nb - nq) / fz.cg;
        fz.smem = fused_smem_bytes();
        std::vector<FusedPiece> pcs;
        fz.qa = ctx->r0;
        fz.qb = ctx->r0 + ctx->nloc;
        fz.partial = nullptr;
        fz.cslots = fused_partition(n, ctx->ld, nq, row_cost, diag_fac, diag_slope, pcs, fz.qlo, fz.qhi, fz.qa, fz.qb);
        const int64_t wrow = (int64_t)fz.nt * 16 * ctx->ld, wcol = (int64_t)nq * fz.cslots * 4096,
                      wg = (int64_t)fz.ng * ctx->ld;
        CKS(dalloc(&ctx->ws, wrow + wcol + wg));
        CKS(dalloc(&ctx->fpieces, (int64_t)nq));
        CKS(cudaMemcpy(ctx->fpieces, pcs.data(), nq * sizeof(FusedPiece), cudaMemcpyHostToDevice));
        fz.Q = ctx->eqh ? ctx->Hq : ctx->A;
        fz.G = ctx->A + ctx->nloc * ctx->ld;
        fz.p = ctx->ploc;
        if (ctx->sharded) {
            CKS(dalloc(&ctx->fpart, ctx->world * ctx->n_slice));
            CKS(dalloc(&ctx->rs_out, ctx->n_slice));
        }
        fz.y = ctx->y_full;
        fz.ws_rowp = ctx->ws;
        fz.ws_col = ctx->ws + wrow;
        fz.ws_g = ctx->ws + wrow + wcol;
        fz.pieces = ctx->fpieces;
        ctx->fused = true;
        if (std::getenv("DUQUAD_DEBUG"))
            fprintf(stderr, "duquad fused: nb %d (max clusters %d) nq %d cg %d ng %d W %d nchg %d nt %d cslots %d\n", nb,
                    maxc, nq, fz.cg, fz.ng, fz.W, fz.nchg, fz.nt, fz.cslots);
    }
    {   // persistent two-pass solve for dense single-GPU QPs whose matrices stay in L2
        const double mbytes = 8.0 * ((double)(n + p) * ctx->ld + (double)n * ctx->ldp);
        int coop = 0;
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, ctx->dev);
        const char *ov = std::getenv("DUQUAD_PERSIST");
        if (!batched && !ctx->sharded && opt.persist_path && !ctx->fused && !ctx->rho0 && coop && mbytes <= 100e6 &&
            !(ov && std::atoi(ov) == 0)) {
            ctx->persist_smem = std::max(smem_a, smem_b);
            CKS(configure_persist(ctx->persist_smem));
            CKS(dalloc(&ctx->pbar, 2));
            ctx->persist = true;
        }
    }
    if (!batched && !ctx->sharded && opt.small_path) {
        // the tables (beta, per-outer scalars) add per-solve bytes: the final check is in duquad_solve
        ctx->small_smem = (size_t)prop.sharedMemPerBlockOptin - 1024;   // minus the static shared memory
        if (small_smem_bytes(n, p, ctx->ld, ctx->ldp, 0, 0) <= ctx->small_smem) {
            CKS(configure_small_kernel(ctx->small_smem));
            ctx->small = true;
        }
    }
    CKS(cudaStreamSynchronize(s));
    apply_pdl(ctx);
    *out = ctx;
    return DUQUAD_OK;
#undef CKS
}

duquad_status duquad_set_constants(duquad_ctx *ctx, double L_in, double L_d) {
    if (!ctx) return fail(nullptr, DUQUAD_EINVAL, "ctx is NULL");
    if (!(L_in > 0.0) || !std::isfinite(L_in) || !(L_d >= 0.0) || !std::isfinite(L_d))
        return fail(ctx, DUQUAD_EINVAL, "need L_in > 0 and L_d >= 0, finite");
    if (ctx->p > 0 && !(L_d > 0.0)) return fail(ctx, DUQUAD_EINVAL, "need L_d > 0 when p > 0");
    ctx->L_in = L_in;
    ctx->L_d = L_d;
    ctx->have_consts = true;
    return DUQUAD_OK;
}

duquad_status duquad_lipschitz(duquad_ctx *ctx, int32_t iters, double safety, double *L_in_out,
                               double *L_d_out, double *normG2_out) {
    if (!ctx) return fail(nullptr, DUQUAD_EINVAL, "ctx is NULL");
    if (!(safety >= 0.0)) return fail(ctx, DUQUAD_EINVAL, "safety must be >= 0");
    DevGuard guard(ctx->dev);
    duquad_status st;
    double normG2 = 0.0, lmax = 0.0;
    if (ctx->p > 0 && (st = lanczos_max(ctx, 1, iters, &normG2)) != DUQUAD_OK) return st;
    if (ctx->opt.l_mode == 0 && ctx->p > 0) {
        if ((st = lanczos_max(ctx, 0, iters, &lmax)) != DUQUAD_OK) return st;
    } else {
        if ((st = lanczos_max(ctx, 2, iters, &lmax)) != DUQUAD_OK) return st;
        lmax += ctx->rho * normG2;
    }
    // The Lanczos values are Ritz values, never above the true eigenvalues: both constants must
    // over-estimate, so the safety factor inflates lambda_max and ||G||^2 alike.  L_d =
    // nG2 / (lambda_min_lb + rho nG2) is increasing in nG2, so it is formed from the inflated
    // ||G||^2 (for l_mode 1, L_in's rho ||G||^2 term is inflated by the outer (1 + safety)).
    const double L_in = (1.0 + safety) * lmax;
    const double normG2_up = (1.0 + safety) * normG2;
    const double denom = ctx->opt.lambda_min_lb + ctx->rho * normG2_up;
    double L_d = 0.0;
    if (ctx->p > 0) {
        if (!(denom > 0.0))
            return fail(ctx, DUQUAD_EINVAL,
                        "L_d undefined: rho == 0 needs lambda_min_lb > 0 (Eq. Ld, PAPER.md:277)");
        L_d = normG2_up / denom;
    }
    if ((st = duquad_set_constants(ctx, L_in, ctx->p > 0 ? L_d : 0.0)) != DUQUAD_OK) return st;
    if (L_in_out) *L_in_out = L_in;
    if (L_d_out) *L_d_out = L_d;
    if (normG2_out) *normG2_out = normG2;
    return DUQUAD_OK;
}

duquad_status duquad_set_trace(duquad_ctx *ctx, double *lam_trace, double *u_trace, int64_t max_outer) {
    if (!ctx) return fail(nullptr, DUQUAD_EINVAL, "ctx is NULL");
    if (ctx->Btot > 1 && (lam_trace || u_trace)) return fail(ctx, DUQUAD_EINVAL, "trace: single QP only");
    DevGuard guard(ctx->dev);
    if (ctx->own_stream) CK(cudaDeviceSynchronize());   // caller's buffers may be in flight
    ctx->trace_lam = lam_trace;
    ctx->trace_u = u_trace;
    ctx->trace_max = (lam_trace || u_trace) ? max_outer : 0;
    return DUQUAD_OK;
}

// Per-solve host tables (fp64, PAPER.md:358-363 / 587-589 / 700-706), their upload, and the
// initial state u_bar^0 = [0]_U, mu^1 = lambda^0 = 0 (before the first all-gather of y).
static duquad_status solve_prepare(duquad_ctx *ctx, int alg, int K, int Kin, std::vector<double> &beta_in) {
    cudaStream_t s = ctx->stream;
    ctx->davg = ctx->opt.dual_average != 0;
    if (ctx->davg && alg != DUQUAD_DGM)
        return fail(ctx, DUQUAD_EINVAL, "dual_average is the DGM final-point rule (PAPER.md:624-626): use alg = DGM");
    if (ctx->davg && ctx->eps_mode)
        return fail(ctx, DUQUAD_EINVAL, "dual_average: fixed inner counts only");
    ctx->resumed = ctx->resume;
    ctx->resume = false;
    if ((ctx->resumed || ctx->opt.checkpoint) && (ctx->davg || ctx->eps_mode))
        return fail(ctx, DUQUAD_EINVAL, "checkpoint / resume: fixed counts, no dual_average");
    ctx->j0 = ctx->resumed ? ctx->ck_j : 0;
    const int J0 = (int)ctx->j0;
    // ---- host tables (fp64, PAPER.md:358-363 / 587-589 / 700-706)
    std::vector<double> theta(J0 + K + 3, 0.0);
    theta[1] = 1.0;
    for (int k = 1; k < J0 + K + 2; ++k) theta[k + 1] = (1.0 + std::sqrt(1.0 + 4.0 * theta[k] * theta[k])) / 2.0;
    beta_in.assign(Kin + 1, 0.0);
    if (ctx->opt.inner_rule == DUQUAD_INNER_FGM) {
        std::vector<double> th(Kin + 2, 0.0);
        th[1] = 1.0;
        for (int k = 1; k < Kin + 1; ++k) th[k + 1] = (1.0 + std::sqrt(1.0 + 4.0 * th[k] * th[k])) / 2.0;
        for (int k = 1; k <= Kin; ++k) beta_in[k] = (th[k] - 1.0) / th[k + 1];
    } else if (ctx->opt.inner_rule == DUQUAD_INNER_FGM_SIGMA) {
        const double b = (std::sqrt(ctx->L_in) - std::sqrt(ctx->opt.sigma)) /
                         (std::sqrt(ctx->L_in) + std::sqrt(ctx->opt.sigma));
        for (int k = 1; k <= Kin; ++k) beta_in[k] = b;
    }
    // outer iterations j = J0+1 .. J0+K (J0 > 0: a continuation of an earlier solve, duquad_set_state)
    std::vector<OuterParam> ops(J0 + K + 2);
    double S = ctx->resumed ? ctx->ck_S : 0.0;
    for (int j = J0 + 1; j <= J0 + K; ++j) {
        const double omega = alg == DUQUAD_DFGM ? theta[j] : 1.0;
        S += omega;
        ops[j].avg_w = omega / S;
        ops[j].dual_update = j >= 2;
        ops[j].beta_out = (j >= 2 && alg == DUQUAD_DFGM) ? (theta[j - 1] - 1.0) / theta[j] : 0.0;
    }
    ctx->S_end = S;
    ops[J0 + K + 1] = OuterParam{0.0, 0.0, 1, 0, 0.0};   // last-iterate solve at lambda^K (mu := lambda^K)
    if (ctx->davg) {
        // DGM dual averaging: the DFOM step of outer j >= 2 computes lambda^{j-1} and
        // folds it into lam_hat with weight 1/j (lam_hat starts at lambda^0); outer K+1 folds in
        // lambda^K and sets mu := lam_hat (inner solve at the average); outer K+2 takes the DFOM step
        // from mu = lam_hat (beta = 0): the final lambda, and its inner solve gives x_last.
        for (int j = 2; j <= K; ++j) ops[j].lhat_w = 1.0 / j;
        ops[K + 1] = OuterParam{0.0, 0.0, 1, 1, 1.0 / (K + 1)};
        ops.push_back(OuterParam{0.0, 0.0, 1, 0, 0.0});
    }
    const int nops = (int)ops.size();
    if (ctx->ops_cap < nops) {
        if (ctx->d_ops) cudaFree(ctx->d_ops);
        ctx->d_ops = nullptr;
        CK(cudaMalloc(&ctx->d_ops, nops * sizeof(OuterParam)));
        ctx->ops_cap = nops;
    }
    CK(cudaMemcpyAsync(ctx->d_ops, ops.data(), nops * sizeof(OuterParam), cudaMemcpyHostToDevice, s));
    // ---- initial state
    if (ctx->Btot > 1)
        CK(launch_init_batched(ctx->Xb, ctx->Yb, ctx->XHb, ctx->lb, ctx->ub, ctx->n, ctx->ld, ctx->mub, ctx->lpb,
                               std::max<int64_t>(ctx->ldp, 2), ctx->Bloc, ctx->d_j, ctx->d_flag, s));
    else
        CK(launch_init_state(ctx->x, ctx->y_full + ctx->rank * ctx->n_slice, ctx->xhat, ctx->lb, ctx->ub,
                             ctx->nloc, ctx->mu, ctx->lam_prev, ctx->ploc, ctx->d_j, ctx->d_flag, s));
    if (ctx->init_x || ctx->init_lam) {   // warm start
        if (ctx->Btot > 1)
            CK(launch_apply_initial(ctx->Xb, ctx->Yb, ctx->lb, ctx->ub, ctx->n, ctx->ld, ctx->init_x, ctx->mub,
                                    ctx->lpb, ctx->p, std::max<int64_t>(ctx->ldp, 2), ctx->init_lam, ctx->Bloc, s));
        else
            CK(launch_apply_initial(ctx->x, ctx->y_full + ctx->rank * ctx->n_slice, ctx->lb, ctx->ub, ctx->nloc, 0,
                                    ctx->init_x, ctx->mu, ctx->lam_prev, ctx->ploc, 0, ctx->init_lam, 1, s));
    }
    if (ctx->resumed) {   // continue from the checkpoint: u_bar^{j0}, mu^{j0}, lambda^{j0-1}, x_hat, j = j0 + 1
        const bool bt = ctx->Btot > 1;
        const int64_t nx = bt ? ctx->Bloc * ctx->ld : ctx->nloc, nl = bt ? ctx->Bloc * std::max<int64_t>(ctx->ldp, 2)
                                                                         : ctx->ploc;
        double *X = bt ? ctx->Xb : ctx->x, *Y = bt ? ctx->Yb : ctx->y_full + ctx->rank * ctx->n_slice;
        double *XH = bt ? ctx->XHb : ctx->xhat, *MU = bt ? ctx->mub : ctx->mu, *LP = bt ? ctx->lpb : ctx->lam_prev;
        const cudaMemcpyKind d2d = cudaMemcpyDeviceToDevice;
        if (nx > 0) {
            CK(cudaMemcpyAsync(X, ctx->ck_x, nx * sizeof(double), d2d, s));
            CK(cudaMemcpyAsync(Y, ctx->ck_x, nx * sizeof(double), d2d, s));
            // the rho = 0 / EQ_H paths' DFOM step reads y from the replica the previous inner solve
            // finished in, Y[K_in % 2]: both replicas start at u_bar^{j0}
            if (!bt && ctx->y_full2)
                CK(cudaMemcpyAsync(ctx->y_full2 + ctx->rank * ctx->n_slice, ctx->ck_x, nx * sizeof(double), d2d, s));
            CK(cudaMemcpyAsync(XH, ctx->ck_xh, nx * sizeof(double), d2d, s));
        }
        if (nl > 0) {
            CK(cudaMemcpyAsync(MU, ctx->ck_mu, nl * sizeof(double), d2d, s));
            CK(cudaMemcpyAsync(LP, ctx->ck_lp, nl * sizeof(double), d2d, s));
        }
        ctx->h_j = (int32_t)(J0 + 1);
        CK(cudaMemcpyAsync(ctx->d_j, &ctx->h_j, sizeof(int32_t), cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));   // h_j is pageable host memory
    }
    if (ctx->Btot > 1)   // h = mu + rho g for the first outer iteration (no DFOM step there)
        CK(launch_batched_h(ctx->hb, ctx->mub, ctx->gb, ctx->rho, ctx->p, std::max<int64_t>(ctx->ldp, 2), ctx->Bloc,
                            s));
    if (ctx->davg) {   // lam_hat := lambda^0
        const int64_t cnt = ctx->Btot > 1 ? ctx->Bloc * std::max<int64_t>(ctx->ldp, 2) : ctx->ploc;
        double *&lh = ctx->Btot > 1 ? ctx->lhb : ctx->lam_hat;
        if (!lh) CK(dalloc(&lh, cnt));
        if (cnt > 0)
            CK(cudaMemcpyAsync(lh, ctx->Btot > 1 ? ctx->lpb : ctx->lam_prev, cnt * sizeof(double),
                               cudaMemcpyDeviceToDevice, s));
    }
    return DUQUAD_OK;
}

duquad_status duquad_set_initial(duquad_ctx *ctx, const double *x0, const double *lambda0, int32_t on_device) {
    if (!ctx) return fail(nullptr, DUQUAD_EINVAL, "ctx is NULL");
    DevGuard guard(ctx->dev);
    // device inputs may still be in flight on the caller's stream (as in duquad_setup): the copies
    // below run on the library's own stream, so wait for all prior work on the device first
    if (on_device) CK(cudaDeviceSynchronize());
    const bool bt = ctx->Btot > 1;
    const int64_t sn = bt ? ctx->ld : ctx->nloc, sp = bt ? std::max<int64_t>(ctx->ldp, 2) : ctx->ploc;
    const int64_t B = bt ? ctx->Bloc : 1;
    // the caller's full vectors: x0 is (batch x) n, lambda0 (batch x) p, row per QP; this context
    // takes its QPs (batched) or its row slices (row-sharded)
    const int64_t xoff = bt ? ctx->b0 * ctx->n : ctx->rank * ctx->n_slice;
    const int64_t loff = bt ? ctx->b0 * ctx->p : ctx->s0;
    const int64_t nx = bt ? ctx->n : ctx->nloc, nl = bt ? ctx->p : ctx->ploc;
    const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (x0) {
        if (!on_device && !finite_host(x0 + xoff, B, nx, bt ? ctx->n : nx))
            return fail(ctx, DUQUAD_EINVAL, "non-finite x0");
        if (!ctx->init_x) CK(dalloc(&ctx->init_x, B * sn));
        if (nx > 0)
            CK(cudaMemcpy2DAsync(ctx->init_x, sn * sizeof(double), x0 + xoff, (bt ? ctx->n : nx) * sizeof(double),
                                 nx * sizeof(double), B, kind, ctx->stream));
    } else if (ctx->init_x) {
        cudaFree(ctx->init_x);
        ctx->init_x = nullptr;
    }
    if (lambda0) {
        if (!on_device && !finite_host(lambda0 + loff, B, nl, bt ? ctx->p : nl))
            return fail(ctx, DUQUAD_EINVAL, "non-finite lambda0");
        if (!ctx->init_lam) CK(dalloc(&ctx->init_lam, B * std::max<int64_t>(sp, 1)));
        if (nl > 0)
            CK(cudaMemcpy2DAsync(ctx->init_lam, std::max<int64_t>(sp, 1) * sizeof(double), lambda0 + loff,
                                 (bt ? ctx->p : nl) * sizeof(double), nl * sizeof(double), B, kind, ctx->stream));
    } else if (ctx->init_lam) {
        cudaFree(ctx->init_lam);
        ctx->init_lam = nullptr;
    }
    CK(cudaStreamSynchronize(ctx->stream));
    return DUQUAD_OK;
}

static duquad_status solve_body(duquad_ctx *ctx, int32_t alg, int32_t outer, int32_t inner, duquad_result *res);

duquad_status duquad_solve(duquad_ctx *ctx, int32_t alg, int32_t outer, int32_t inner, duquad_result *res) {
    if (!ctx) return fail(nullptr, DUQUAD_EINVAL, "ctx is NULL");
    ctx->eps_mode = false;
    return solve_body(ctx, alg, outer, inner, res);
}

// eps_in mode around a solve: buffers, counters and the threshold, then (after) the per-solve
// counts and the EMAXITER status
static duquad_status eps_begin(duquad_ctx *ctx, int32_t outer, double eps_in, double sigma_L) {
    const int64_t B = ctx->Btot > 1 ? ctx->Bloc : 1;
    const int64_t nc = ((int64_t)outer + 1) * B;   // per QP (batched: QP-major [QP][solve])
    ctx->eps_nc = (int64_t)outer + 1;
    if (ctx->Btot > 1) {
        if (ctx->gm_b) cudaFree(ctx->gm_b);
        if (ctx->done_b) cudaFree(ctx->done_b);
        if (!ctx->ndone) CK(dalloc(&ctx->ndone, 2));
        ctx->gm_b = nullptr;
        ctx->done_b = nullptr;
        CK(dalloc(&ctx->gm_b, B));
        CK(dalloc(&ctx->done_b, B));
        CK(cudaMemsetAsync(ctx->ndone, 0, sizeof(int32_t), ctx->stream));
    }
    if (!ctx->gm_sq) {
        CK(dalloc(&ctx->gm_sq, std::max<int64_t>(ctx->nloc, 1)));
        CK(dalloc(&ctx->gm_part, (int64_t)kRedGrid));
        CK(dalloc(&ctx->gm_counter, 2));
        CK(dalloc(&ctx->d_done, 2));
        CK(dalloc(&ctx->gm_tot, 2));
    }
    if (ctx->counts_cap < nc) {
        if (ctx->d_counts) cudaFree(ctx->d_counts);
        ctx->d_counts = nullptr;
        CK(dalloc(&ctx->d_counts, 2 * nc));
        ctx->counts_cap = nc;
    }
    CK(cudaMemsetAsync(ctx->d_counts, 0, 2 * ctx->counts_cap * sizeof(int32_t), ctx->stream));
    CK(cudaMemsetAsync(ctx->d_done, 0, sizeof(int32_t), ctx->stream));
    CK(cudaMemsetAsync(ctx->gm_counter, 0, sizeof(uint32_t), ctx->stream));
    // stop when L_in ||y - x+|| <= sqrt(2 sigma_L eps_in), i.e. sum (y - x+)^2 <= 2 sigma_L eps_in / L_in^2
    ctx->eps_thresh2 = 2.0 * sigma_L * eps_in / (ctx->L_in * ctx->L_in);
    ctx->eps_mode = true;
    ctx->pend_decide = false;
    return DUQUAD_OK;
}

static duquad_status eps_end(duquad_ctx *ctx, int32_t outer, duquad_status st, duquad_result *res) {
    const int64_t nc = ((int64_t)outer + 1) * (ctx->Btot > 1 ? ctx->Bloc : 1);
    ctx->eps_mode = false;
    if (st != DUQUAD_OK && st != DUQUAD_ENONFINITE) return st;
    std::vector<int32_t> buf(2 * ctx->counts_cap);
    CK(cudaMemcpy(buf.data(), ctx->d_counts, buf.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
    ctx->last_counts.assign(buf.begin(), buf.begin() + nc);
    ctx->last_conv.assign(buf.begin() + ctx->counts_cap, buf.begin() + ctx->counts_cap + nc);
    int64_t total = 0;
    bool capped = false;
    for (int64_t j = 0; j < nc; ++j) {
        total += ctx->last_counts[j];
        capped |= ctx->last_conv[j] == 0;
    }
    if (res) {
        res->inner_iters_total = total;   // batched: summed over the QPs
        // the matvec accounting of the fixed-count solve: two passes per inner step,
        // except on the Q-only paths (rho = 0, EQ_H), whose inner step is one pass plus two passes
        // (G u_bar, G' mu) per inner solve, i.e. per outer iteration and the last-iterate solve
        res->matrix_passes = ctx->rho0 && ctx->Btot == 1 ? total + 2 * (int64_t)(outer + 1) : 2 * total;
    }
    if (st != DUQUAD_OK) return st;
    if (capped) return fail(ctx, DUQUAD_EMAXITER, "an inner solve hit inner_max before the eps_in test (result valid)");
    return DUQUAD_OK;
}

duquad_status duquad_solve_eps(duquad_ctx *ctx, int32_t alg, int32_t outer, int32_t inner_max, double eps_in,
                               double sigma_L, duquad_result *res) {
    if (!ctx) return fail(nullptr, DUQUAD_EINVAL, "ctx is NULL");
    if (!(eps_in > 0.0) || !(sigma_L > 0.0) || !std::isfinite(eps_in) || !std::isfinite(sigma_L))
        return fail(ctx, DUQUAD_EINVAL, "eps_in and sigma_L must be finite and > 0");
    if (ctx->emulated) return fail(ctx, DUQUAD_EINVAL, "emulated ranks: use duquad_solve_eps_emulated");
    if (outer < 1 || inner_max < 1) return fail(ctx, DUQUAD_EINVAL, "need outer_iters >= 1 and inner_max >= 1");
    if (!ctx->have_consts) return fail(ctx, DUQUAD_ESTATE, "constants not set (duquad_lipschitz or duquad_set_constants)");
    DevGuard guard(ctx->dev);
    duquad_status st = eps_begin(ctx, outer, eps_in, sigma_L);
    if (st != DUQUAD_OK) return st;
    st = solve_body(ctx, alg, outer, inner_max, res);
    return eps_end(ctx, outer, st, res);
}

duquad_status duquad_theory_schedule(int32_t alg, double eps, double R_d, double L_d, double L_in, double sigma_L,
                                     double D_U, double normG, double lambda_min_Q, double lambda_max_Q,
                                     duquad_schedule *out) {
    if (!out) return fail(nullptr, DUQUAD_EINVAL, "out is NULL");
    if (alg != DUQUAD_DGM && alg != DUQUAD_DFGM) return fail(nullptr, DUQUAD_EINVAL, "bad alg");
    const double v[] = {eps, R_d, L_d, L_in, sigma_L, D_U, normG, lambda_min_Q, lambda_max_Q};
    for (double x : v)
        if (!std::isfinite(x)) return fail(nullptr, DUQUAD_EINVAL, "non-finite schedule argument");
    if (!(eps > 0) || !(R_d > 0) || !(L_d > 0) || !(L_in > 0) || sigma_L < 0 || !(D_U > 0) || normG < 0 ||
        lambda_min_Q < 0 || lambda_max_Q < 0)
        return fail(nullptr, DUQUAD_EINVAL, "schedule arguments out of range");
    std::memset(out, 0, sizeof(*out));
    // counts are formed in double and clamped to [0, 2^62] before the integer conversion
    auto to_count = [](double x) { return x > 0.0 ? (int64_t)std::min(x, 4.6116860184273879e18) : (int64_t)0; };
    const double q = 8.0 * L_d * R_d * R_d / eps;                         // (choose_ein)
    if (alg == DUQUAD_DGM) {
        out->eps_in = eps / 4.0;
        out->k_out = to_count(std::ceil(q));
    } else {
        out->eps_in = eps * std::sqrt(eps) / (8.0 * R_d * std::sqrt(2.0 * L_d));
        out->k_out = to_count(std::ceil(std::sqrt(q)));
    }
    const double d2 = D_U * D_U;
    double kin;
    if (sigma_L > 0.0)
        kin = std::sqrt(L_in / sigma_L) * std::log(L_in * d2 / out->eps_in) + 1.0;
    else
        kin = std::sqrt(2.0 * L_in * d2 / out->eps_in);
    out->k_in = to_count(std::ceil(std::max(kin, 1.0)));
    out->rho_star = 8.0 * R_d * R_d / eps;
    // the log's argument is clamped to >= 1 (normG == 0 would give 0 * log 0 = NaN; an argument
    // below 1 a negative count)
    const double kt = sigma_L > 0.0 ? 16.0 * normG * R_d / std::sqrt(sigma_L * eps) *
                                          std::log(std::max(1.0, 8.0 * normG * D_U * R_d / eps))
                                    : 24.0 * normG * D_U * R_d / eps;
    out->k_total = to_count(std::floor(kt));
    // Case 1 (Q > 0, rho = 0) iff lambda_min(Q) > tau_pd = 1e-7 max(1, lambda_max(Q))
    // (SPEC.md:186's numerical threshold for the paper's dichotomy; reading c25)
    out->case_id = lambda_min_Q > 1e-7 * std::max(1.0, lambda_max_Q) ? 1 : 2;
    return DUQUAD_OK;
}

duquad_status duquad_local_ranges(const duquad_ctx *ctx, int64_t *r0, int64_t *nloc, int64_t *s0, int64_t *ploc) {
    if (!ctx) return fail(nullptr, DUQUAD_EINVAL, "ctx is NULL");
    if (r0) *r0 = ctx->Btot > 1 ? 0 : ctx->r0;
    if (nloc) *nloc = ctx->Btot > 1 ? ctx->n : ctx->nloc;
    if (s0) *s0 = ctx->Btot > 1 ? 0 : ctx->s0;
    if (ploc) *ploc = ctx->Btot > 1 ? ctx->p : ctx->ploc;
    return DUQUAD_OK;
}

duquad_status duquad_theory_bounds(int32_t alg, int64_t k, double L_d, double R_d, double eps_in,
                                   duquad_bounds *out) {
    if (!out) return fail(nullptr, DUQUAD_EINVAL, "out is NULL");
    if (alg != DUQUAD_DGM && alg != DUQUAD_DFGM) return fail(nullptr, DUQUAD_EINVAL, "bad alg");
    if (!std::isfinite(L_d) || !std::isfinite(R_d) || !std::isfinite(eps_in) || k < 1 || !(L_d > 0) || R_d < 0 ||
        eps_in < 0)
        return fail(nullptr, DUQUAD_EINVAL, "bounds arguments out of range");
    const double k1 = (double)k + 1.0, kk = (double)k;
    const bool fast = alg == DUQUAD_DFGM;                 // p(beta) = 2 for DFGM, 1 for DGM (Eq. pbetak)
    out->dual_gap = 4.0 * L_d * R_d * R_d / (fast ? k1 * k1 : k1) + 2.0 * (fast ? k1 : 1.0) * eps_in;
    out->drift = R_d + std::sqrt(kk * eps_in / L_d);
    out->feas_last = std::sqrt(2.0 * L_d * eps_in) + std::sqrt(2.0 * L_d * out->dual_gap);
    out->feas_avg = fast ? 8.0 * L_d * R_d / (kk * kk) + 8.0 * std::sqrt(L_d * eps_in / kk)
                         : 4.0 * L_d * R_d / kk + 2.0 * std::sqrt(L_d * eps_in / kk);
    return DUQUAD_OK;
}

duquad_status duquad_get_inner_counts(duquad_ctx *ctx, int32_t *counts, int32_t *converged, int32_t max_entries) {
    if (!ctx) return fail(nullptr, DUQUAD_EINVAL, "ctx is NULL");
    if (max_entries < 0) return fail(ctx, DUQUAD_EINVAL, "max_entries < 0");
    const int64_t m = std::min<int64_t>(max_entries, (int64_t)ctx->last_counts.size());
    for (int64_t j = 0; j < m; ++j) {
        if (counts) counts[j] = ctx->last_counts[j];
        if (converged) converged[j] = ctx->last_conv[j];
    }
    return DUQUAD_OK;
}

// device sizes of the state vectors (x, x_hat: n-vectors; mu, lambda_prev: p-vectors) in this
// context's layout (QP-major with strides ld / ldp for a batch)
static void state_sizes(const duquad_ctx *ctx, int64_t *nx, int64_t *nl) {
    const bool bt = ctx->Btot > 1;
    *nx = bt ? ctx->Bloc * ctx->ld : ctx->nloc;
    *nl = bt ? ctx->Bloc * std::max<int64_t>(ctx->ldp, 2) : ctx->ploc;
}

static duquad_status alloc_state(duquad_ctx *ctx) {
    int64_t nx, nl;
    state_sizes(ctx, &nx, &nl);
    if (!ctx->ck_x) CK(dalloc(&ctx->ck_x, nx));
    if (!ctx->ck_xh) CK(dalloc(&ctx->ck_xh, nx));
    if (!ctx->ck_mu) CK(dalloc(&ctx->ck_mu, nl));
    if (!ctx->ck_lp) CK(dalloc(&ctx->ck_lp, nl));
    return DUQUAD_OK;
}

// the state after outer iteration K of this solve: u_bar^K, mu^K, lambda^{K-1}, x_hat (enqueued)
static duquad_status save_checkpoint(duquad_ctx *ctx) {
    duquad_status st = alloc_state(ctx);
    if (st != DUQUAD_OK) return st;
    int64_t nx, nl;
    state_sizes(ctx, &nx, &nl);
    const bool bt = ctx->Btot > 1;
    const cudaMemcpyKind d2d = cudaMemcpyDeviceToDevice;
    if (nx > 0) {
        CK(cudaMemcpyAsync(ctx->ck_x, bt ? ctx->Xb : ctx->x, nx * sizeof(double), d2d, ctx->stream));
        CK(cudaMemcpyAsync(ctx->ck_xh, bt ? ctx->XHb : ctx->xhat, nx * sizeof(double), d2d, ctx->stream));
    }
    if (nl > 0) {
        CK(cudaMemcpyAsync(ctx->ck_mu, bt ? ctx->mub : ctx->mu, nl * sizeof(double), d2d, ctx->stream));
        CK(cudaMemcpyAsync(ctx->ck_lp, bt ? ctx->lpb : ctx->lam_prev, nl * sizeof(double), d2d, ctx->stream));
    }
    return DUQUAD_OK;
}

// caller layout <-> context layout of one state vector (len per QP, stride ld per QP in a batch)
static duquad_status state_copy(duquad_ctx *ctx, double *dst, const double *src, int64_t len, int64_t ld,
                                bool to_ctx, int32_t on_device) {
    const int64_t B = ctx->Btot > 1 ? ctx->Bloc : 1;
    if (len <= 0 || B <= 0) return DUQUAD_OK;
    const int64_t ldc = ctx->Btot > 1 ? ld : len;
    const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice
                                          : (to_ctx ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost);
    if (to_ctx)
        CK(cudaMemcpy2DAsync(dst, ldc * sizeof(double), src, len * sizeof(double), len * sizeof(double), B, kind,
                             ctx->stream));
    else
        CK(cudaMemcpy2DAsync(dst, len * sizeof(double), src, ldc * sizeof(double), len * sizeof(double), B, kind,
                             ctx->stream));
    return DUQUAD_OK;
}

duquad_status duquad_get_state(duquad_ctx *ctx, double *x, double *mu, double *lam_prev, double *x_avg,
                               int64_t *outer_done, double *S, int32_t on_device) {
    if (!ctx) return fail(nullptr, DUQUAD_EINVAL, "ctx is NULL");
    if (!ctx->ck_valid) return fail(ctx, DUQUAD_ESTATE, "no checkpoint: solve with options.checkpoint = 1 first");
    DevGuard guard(ctx->dev);
    const int64_t n = ctx->Btot > 1 ? ctx->n : ctx->nloc, p = ctx->Btot > 1 ? ctx->p : ctx->ploc;
    const int64_t sp = std::max<int64_t>(ctx->ldp, 2);
    duquad_status st;
    if (x && (st = state_copy(ctx, x, ctx->ck_x, n, ctx->ld, false, on_device)) != DUQUAD_OK) return st;
    if (x_avg && (st = state_copy(ctx, x_avg, ctx->ck_xh, n, ctx->ld, false, on_device)) != DUQUAD_OK) return st;
    if (mu && (st = state_copy(ctx, mu, ctx->ck_mu, p, sp, false, on_device)) != DUQUAD_OK) return st;
    if (lam_prev && (st = state_copy(ctx, lam_prev, ctx->ck_lp, p, sp, false, on_device)) != DUQUAD_OK) return st;
    CK(cudaStreamSynchronize(ctx->stream));
    if (outer_done) *outer_done = ctx->ck_j;
    if (S) *S = ctx->ck_S;
    return DUQUAD_OK;
}

duquad_status duquad_set_state(duquad_ctx *ctx, const double *x, const double *mu, const double *lam_prev,
                               const double *x_avg, int64_t outer_done, double S, int32_t on_device) {
    if (!ctx) return fail(nullptr, DUQUAD_EINVAL, "ctx is NULL");
    if (outer_done < 1 || !(S > 0) || !std::isfinite(S) || outer_done > (1 << 28))
        return fail(ctx, DUQUAD_EINVAL, "set_state: outer_done >= 1 and S > 0 (the averaging weight sum)");
    if (!x || !x_avg || (ctx->p > 0 && (!mu || !lam_prev)))
        return fail(ctx, DUQUAD_EINVAL, "set_state: x, x_avg, mu and lam_prev are all required");
    DevGuard guard(ctx->dev);
    if (on_device) CK(cudaDeviceSynchronize());   // caller's device buffers may still be in flight
    duquad_status st = alloc_state(ctx);
    if (st != DUQUAD_OK) return st;
    const int64_t n = ctx->Btot > 1 ? ctx->n : ctx->nloc, p = ctx->Btot > 1 ? ctx->p : ctx->ploc;
    const int64_t sp = std::max<int64_t>(ctx->ldp, 2);
    if ((st = state_copy(ctx, ctx->ck_x, x, n, ctx->ld, true, on_device)) != DUQUAD_OK) return st;
    if ((st = state_copy(ctx, ctx->ck_xh, x_avg, n, ctx->ld, true, on_device)) != DUQUAD_OK) return st;
    if (p > 0) {
        if ((st = state_copy(ctx, ctx->ck_mu, mu, p, sp, true, on_device)) != DUQUAD_OK) return st;
        if ((st = state_copy(ctx, ctx->ck_lp, lam_prev, p, sp, true, on_device)) != DUQUAD_OK) return st;
    }
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->ck_valid = true;
    ctx->ck_j = outer_done;
    ctx->ck_S = S;
    ctx->resume = true;
    return DUQUAD_OK;
}

static duquad_status solve_body(duquad_ctx *ctx, int32_t alg, int32_t outer, int32_t inner, duquad_result *res) {
    if (alg != DUQUAD_DGM && alg != DUQUAD_DFGM) return fail(ctx, DUQUAD_EINVAL, "bad alg");
    if (outer < 1 || inner < 1) return fail(ctx, DUQUAD_EINVAL, "need outer_iters >= 1 and inner_iters >= 1");
    if (!ctx->have_consts) return fail(ctx, DUQUAD_ESTATE, "constants not set (duquad_lipschitz or duquad_set_constants)");
    DevGuard guard(ctx->dev);
    cudaStream_t s = ctx->stream;
    const int K = outer, Kin = inner;
    std::vector<double> beta_in;
    {
        duquad_status st0 = solve_prepare(ctx, alg, K, Kin, beta_in);
        if (st0 != DUQUAD_OK) return st0;
    }
    duquad_status st;
    if ((st = allgather_y(ctx)) != DUQUAD_OK) return st;
    if (ctx->resumed && ctx->y_full2 && (st = allgather_vec(ctx, ctx->y_full2)) != DUQUAD_OK) return st;
    if (ctx->small && !ctx->eps_mode && !ctx->davg && !ctx->resumed && !ctx->opt.checkpoint &&
        small_smem_bytes(ctx->n, ctx->p, ctx->ld, ctx->ldp, K, Kin) <= ctx->small_smem) {   // whole solve in one CTA (K4)
        if (ctx->beta_cap < Kin + 1) {
            if (ctx->d_beta) cudaFree(ctx->d_beta);
            ctx->d_beta = nullptr;
            CK(cudaMalloc(&ctx->d_beta, (Kin + 1) * sizeof(double)));
            ctx->beta_cap = Kin + 1;
        }
        CK(cudaMemcpyAsync(ctx->d_beta, beta_in.data(), (Kin + 1) * sizeof(double), cudaMemcpyHostToDevice, s));
        SmallArgs sa{};
        sa.A = ctx->A;
        sa.GT = ctx->GT;
        sa.n = ctx->n;
        sa.p = ctx->p;
        sa.ld = ctx->ld;
        sa.ldp = ctx->ldp;
        sa.q = ctx->q;
        sa.lb = ctx->lb;
        sa.ub = ctx->ub;
        sa.g = ctx->g;
        sa.cone = ctx->cone;
        sa.K = K;
        sa.Kin = Kin;
        sa.beta_in = ctx->d_beta;
        sa.a = make_a(ctx);
        sa.b = make_b(ctx);
        sa.trace_lam = ctx->trace_lam;
        sa.trace_u = ctx->trace_u;
        sa.trace_max = ctx->trace_max;
        sa.x_out = ctx->x;
        sa.xhat_out = ctx->xhat;
        sa.y_out = ctx->y_full;
        sa.lam_out = ctx->lam_prev;
        sa.mu_out = ctx->mu;
        sa.x_init = ctx->init_x;
        sa.lam_init = ctx->init_lam;
        cudaEvent_t t0, t1;
        CK(cudaEventCreate(&t0));
        CK(cudaEventCreate(&t1));
        CK(cudaEventRecord(t0, s));
        CK(launch_small_solve(sa, small_smem_bytes(ctx->n, ctx->p, ctx->ld, ctx->ldp, K, Kin), s));
        CK(cudaEventRecord(t1, s));
        CK(cudaStreamSynchronize(s));
        int32_t flag = 0;
        CK(cudaMemcpy(&flag, ctx->d_flag, sizeof(flag), cudaMemcpyDeviceToHost));
        if (res) {
            std::memset(res, 0, sizeof(*res));
            float ms = 0.f;
            cudaEventElapsedTime(&ms, t0, t1);
            res->ms_device = ms;
            res->path = DUQUAD_PATH_SMALL;
            res->outer_iters = K;
            res->inner_iters_total = (int64_t)(K + 1) * Kin;
            res->kernel_launches = 2;
            res->matrix_passes = (int64_t)(K + 1) * Kin * 2;
            res->bytes_pass_a = 8.0 * ((double)(ctx->n + ctx->p) * ctx->n);   // from shared memory
            res->bytes_pass_b = 8.0 * ((double)ctx->n * ctx->p);
        }
        cudaEventDestroy(t0);
        cudaEventDestroy(t1);
        ctx->solved = true;
        if (flag) return fail(ctx, DUQUAD_ENONFINITE, "an iterate became non-finite");
        return DUQUAD_OK;
    }
    const bool tracing = ctx->trace_lam || ctx->trace_u;
    if (ctx->persist && !tracing && !ctx->eps_mode && !ctx->davg && !ctx->resumed && !ctx->opt.checkpoint) {   // the whole solve in one cooperative launch
        if (ctx->beta_cap < Kin + 1) {
            if (ctx->d_beta) cudaFree(ctx->d_beta);
            ctx->d_beta = nullptr;
            CK(cudaMalloc(&ctx->d_beta, (Kin + 1) * sizeof(double)));
            ctx->beta_cap = Kin + 1;
        }
        CK(cudaMemcpyAsync(ctx->d_beta, beta_in.data(), (Kin + 1) * sizeof(double), cudaMemcpyHostToDevice, s));
        cudaEvent_t t0, t1;
        CK(cudaEventCreate(&t0));
        CK(cudaEventCreate(&t1));
        CK(cudaEventRecord(t0, s));
        CK(launch_persist(make_a(ctx), make_b(ctx), ctx->d_beta, K, Kin, ctx->pbar, ctx->num_sms, ctx->persist_smem, s));
        CK(cudaEventRecord(t1, s));
        CK(cudaStreamSynchronize(s));
        int32_t flag = 0;
        CK(cudaMemcpy(&flag, ctx->d_flag, sizeof(flag), cudaMemcpyDeviceToHost));
        if (res) {
            std::memset(res, 0, sizeof(*res));
            float ms = 0.f;
            cudaEventElapsedTime(&ms, t0, t1);
            res->ms_device = ms;
            res->path = DUQUAD_PATH_PERSIST;
            res->outer_iters = K;
            res->inner_iters_total = (int64_t)(K + 1) * Kin;
            res->kernel_launches = 2;
            res->matrix_passes = (int64_t)(K + 1) * Kin * 2;
            const double nn = (double)ctx->n, pp = (double)ctx->p;
            res->bytes_pass_a = 8.0 * ((nn + pp) * nn + nn + nn + 3.0 * pp);
            res->bytes_pass_b = 8.0 * (nn * pp + pp + 8.0 * nn);
        }
        cudaEventDestroy(t0);
        cudaEventDestroy(t1);
        ctx->solved = true;
        if (flag) return fail(ctx, DUQUAD_ENONFINITE, "an iterate became non-finite");
        return DUQUAD_OK;
    }
    const bool graphs = ctx->opt.use_graphs && !tracing;
    const int j_timed = ctx->opt.time_passes ? std::max(1, (K + 1) / 2) : -1;
    std::vector<cudaEvent_t> ev;
    if (j_timed > 0) {
        ev.resize(4 * Kin);
        for (auto &e : ev) CK(cudaEventCreate(&e));
    }
    cudaGraphExec_t gexec = nullptr;
    cudaGraph_t graph = nullptr;
    if (graphs) {
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        st = run_outer(ctx, beta_in, Kin, -1, nullptr);
        cudaError_t e = cudaStreamEndCapture(s, &graph);
        if (st != DUQUAD_OK) return st;
        CK(e);
        CK(cudaGraphInstantiate(&gexec, graph, 0));
    }
    cudaEvent_t t0, t1;
    CK(cudaEventCreate(&t0));
    CK(cudaEventCreate(&t1));
    CK(cudaEventRecord(t0, s));
    const int nout = K + 1 + (ctx->davg ? 1 : 0);   // + the solve at the dual average
    for (int j = 1; j <= nout; ++j) {
        if (j == K + 1 && ctx->opt.checkpoint && (st = save_checkpoint(ctx)) != DUQUAD_OK) break;
        if (j == j_timed) {
            st = run_outer(ctx, beta_in, Kin, j, &ev);
        } else if (graphs) {
            cudaError_t e = cudaGraphLaunch(gexec, s);
            st = e == cudaSuccess ? DUQUAD_OK : fail(ctx, DUQUAD_ECUDA, std::string("cudaGraphLaunch: ") + cudaGetErrorString(e));
        } else {
            st = run_outer(ctx, beta_in, Kin, j, nullptr);
        }
        if (st != DUQUAD_OK) break;
    }
    CK(cudaEventRecord(t1, s));
    cudaError_t esync = cudaStreamSynchronize(s);
    if (gexec) cudaGraphExecDestroy(gexec);
    if (graph) cudaGraphDestroy(graph);
    if (st != DUQUAD_OK) return st;
    CK(esync);
    int32_t flag = 0;
    CK(cudaMemcpy(&flag, ctx->d_flag, sizeof(flag), cudaMemcpyDeviceToHost));
    if (res) {
        std::memset(res, 0, sizeof(*res));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, t0, t1);
        res->ms_device = ms;
        res->path = ctx->eqh ? (ctx->fused ? DUQUAD_PATH_EQ_H_FLOOR : DUQUAD_PATH_EQ_H)
                    : ctx->fused ? (ctx->rho0 ? DUQUAD_PATH_RHO0_FLOOR : DUQUAD_PATH_BYTE_FLOOR)
                    : ctx->rho0 ? DUQUAD_PATH_RHO0
                    : ctx->Btot > 1 ? DUQUAD_PATH_BATCHED
                    : ctx->format == DUQUAD_CSR ? DUQUAD_PATH_CSR : DUQUAD_PATH_TWO_PASS;
        res->sparse_kernels = ctx->format == DUQUAD_CSR ? (ctx->kind_a | (ctx->dia.nd > 0 ? 8 : 0) | (ctx->dia.sym ? 64 : 0)) | (ctx->kind_b << 4)
                                                        : 0;
        res->outer_iters = K;
        res->inner_iters_total = (int64_t)nout * Kin;
        res->kernel_launches = 1 + (int64_t)nout * (2 * Kin + 1);
        res->matrix_passes = (int64_t)nout * Kin * 2;
        const double nn = (double)ctx->n, nl = (double)ctx->nloc, pl = (double)ctx->ploc, pp = (double)ctx->p;
        if (ctx->fused) {      // byte floor: Q triangle (+ G once) streamed, workspace through L2
            // algorithmic bytes: Q triangle + G once + y; the epilogue: 7 vectors + the partials
            // (row-sharded: this rank's rows [qa, qb) of the triangle and its G rows)
            const double qa = (double)ctx->fz.qa, qb = (double)ctx->fz.qb;
            const double tri = (qb - qa) * nn - 0.5 * (qb * qb - qa * qa) + 0.5 * (qb - qa);
            const double wsb = 16.0 * ctx->fz.nt * (double)ctx->ld +
                               (double)ctx->fz.nq_ctas * ctx->fz.cslots * 4096.0 + (double)ctx->fz.ng * (double)ctx->ld;
            res->bytes_pass_a = 8.0 * (tri + (ctx->rho0 ? 0.0 : pl * nn) + nn);
            res->bytes_pass_b = 8.0 * (wsb + 8.0 * nn);
            if (ctx->rho0) {
                res->kernel_launches = 1 + (int64_t)nout * (2 * Kin + 3);
                res->matrix_passes = (int64_t)nout * (Kin + 2);
            }
        } else if (ctx->rho0) {       // K3 inner steps: Q only; per outer: one G pass and one G' pass
            res->kernel_launches = 1 + (int64_t)nout * (Kin + 3);
            res->matrix_passes = (int64_t)nout * (Kin + 2);
            res->bytes_pass_a = 8.0 * (nl * nn + nn + 8.0 * nl);   // "pass A" slot = the K3 step
            res->bytes_pass_b = 0.0;
        } else if (ctx->Btot > 1) {   // shared matrices (L2-resident) + per-QP vectors
            const double B = (double)ctx->Bloc;
            // flops the kernels execute (paired rows: [Q;G_t] and G_t', P = p/2; the algorithmic
            // 2B(n+p)n + 2Bnp of the unpaired step is what the step computes either way)
            const double pe = ctx->pairP ? (double)ctx->pairP : pp;
            res->flops_pass_a = 2.0 * (nn + pe) * nn * B;
            res->flops_pass_b = 2.0 * nn * pe * B;
            res->bytes_pass_a = 8.0 * ((nn + pp) * nn + B * (nn + nn + 3.0 * pp));
            res->bytes_pass_b = 8.0 * (nn * pp + B * (pp + 8.0 * nn));
        } else if (ctx->format == DUQUAD_CSR) {   // values + indices + row pointers + vectors
            res->bytes_pass_a = 12.0 * ctx->nnz_a + 4.0 * (nl + pl + 1) + 8.0 * (nn + nl + 3.0 * pl);
            res->bytes_pass_b = 12.0 * ctx->nnz_b + 4.0 * (nl + 1) + 8.0 * (pp + 8.0 * nl);
        } else {
            res->bytes_pass_a = 8.0 * ((nl + pl) * nn + nn + nl + 3.0 * pl);
            res->bytes_pass_b = 8.0 * (nl * pp + pp + 8.0 * nl);
        }
        if (j_timed > 0) {
            double sa = 0, sb = 0;
            for (int k = 0; k < Kin; ++k) {
                float a = 0.f, b = 0.f;
                cudaEventElapsedTime(&a, ev[4 * k], ev[4 * k + 1]);
                cudaEventElapsedTime(&b, ev[4 * k + 2], ev[4 * k + 3]);
                sa += a;
                sb += b;
            }
            res->ms_pass_a = sa / Kin;
            res->ms_pass_b = sb / Kin;
            res->n_timed_a = Kin;
            res->n_timed_b = Kin;
        }
    }
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    for (auto &e : ev) cudaEventDestroy(e);
    ctx->solved = true;
    if (ctx->opt.checkpoint && !flag) {
        ctx->ck_valid = true;
        ctx->ck_j = ctx->j0 + K;
        ctx->ck_S = ctx->S_end;
    }
    if (flag) return fail(ctx, DUQUAD_ENONFINITE, "an iterate became non-finite");
    return DUQUAD_OK;
}

// all-gather of replica buffer b across emulated ranks: device copies of every rank's slice
static duquad_status group_gather_impl(duquad_ctx **c, int P, int b);
static duquad_status group_gather(duquad_ctx **c, int P, int b) {
    duquad_status st = group_gather_impl(c, P, b);
    if (st != DUQUAD_OK || P == 1 || !c[0]->pend_decide) return st;
    // emulated all-reduce of the stop test's sum: ranks added in order, the result to every rank
    duquad_ctx *ctx = c[0];
    double *acc = c[0]->gm_part;   // scratch (the partial sums of the check kernel are consumed)
    CK(cudaMemcpyAsync(acc, c[0]->gm_tot, sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    for (int q = 1; q < P; ++q) CK(launch_vec_add(acc, c[q]->gm_tot, 1, ctx->stream));
    for (int r = 0; r < P; ++r) {
        CK(cudaMemcpyAsync(c[r]->gm_tot, acc, sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
        CK(launch_inner_decide(c[r]->gm_tot, c[r]->d_done, c[r]->eps_thresh2, c[r]->d_counts, c[r]->d_j,
                               ctx->stream));
        c[r]->pend_decide = false;
    }
    return DUQUAD_OK;
}

static duquad_status group_gather_impl(duquad_ctx **c, int P, int b) {
    if (b < 0 || P == 1) return DUQUAD_OK;
    duquad_ctx *ctx = c[0];
    if (b == G_RS) {   // reduce-scatter: slice r = sum over ranks q (in order) of fpart_q[slice r]
        const int64_t sl = ctx->n_slice;
        for (int r = 0; r < P; ++r) {
            CK(cudaMemcpyAsync(c[r]->rs_out, c[0]->fpart + r * sl, sl * sizeof(double), cudaMemcpyDeviceToDevice,
                               ctx->stream));
            for (int q = 1; q < P; ++q) CK(launch_vec_add(c[r]->rs_out, c[q]->fpart + r * sl, sl, ctx->stream));
        }
        return DUQUAD_OK;
    }
    const int64_t sl = gather_slice(ctx, b);
    for (int d = 0; d < P; ++d)
        for (int s = 0; s < P; ++s) {
            const int64_t off = b == G_W ? ctx->gs0[s] : s * sl, cnt = b == G_W ? ctx->gcnt[s] : sl;
            if (s != d && cnt > 0)
                CK(cudaMemcpyAsync(gather_ptr(c[d], b) + off, gather_ptr(c[s], b) + off, cnt * sizeof(double),
                                   cudaMemcpyDeviceToDevice, ctx->stream));
        }
    return DUQUAD_OK;
}

static duquad_status solve_emulated_impl(duquad_ctx **ctxs, int32_t P, int32_t alg, int32_t outer, int32_t inner);

duquad_status duquad_solve_eps_emulated(duquad_ctx **ctxs, int32_t P, int32_t alg, int32_t outer, int32_t inner_max,
                                        double eps_in, double sigma_L) {
    if (!ctxs || P < 1 || !ctxs[0]) return fail(nullptr, DUQUAD_EINVAL, "need P >= 1 contexts");
    if (!(eps_in > 0.0) || !(sigma_L > 0.0) || !std::isfinite(eps_in) || !std::isfinite(sigma_L))
        return fail(ctxs[0], DUQUAD_EINVAL, "eps_in and sigma_L must be finite and > 0");
    if (outer < 1 || inner_max < 1) return fail(ctxs[0], DUQUAD_EINVAL, "need outer_iters >= 1 and inner_max >= 1");
    for (int r = 0; r < P; ++r)
        if (!ctxs[r] || !ctxs[r]->have_consts || ctxs[r]->Btot > 1)
            return fail(ctxs[0], DUQUAD_EINVAL, "emulated eps_in group: set-up single-QP contexts with constants");
    DevGuard guard(ctxs[0]->dev);
    duquad_status st;
    for (int r = 0; r < P; ++r)
        if ((st = eps_begin(ctxs[r], outer, eps_in, sigma_L)) != DUQUAD_OK) return st;
    st = solve_emulated_impl(ctxs, P, alg, outer, inner_max);
    duquad_status out = DUQUAD_OK;
    for (int r = 0; r < P; ++r) {
        const duquad_status e = eps_end(ctxs[r], outer, st, nullptr);
        if (out == DUQUAD_OK) out = e;
    }
    return out;
}

duquad_status duquad_solve_emulated(duquad_ctx **ctxs, int32_t P, int32_t alg, int32_t outer, int32_t inner) {
    if (ctxs && P >= 1)
        for (int r = 0; r < P; ++r)
            if (ctxs[r]) ctxs[r]->eps_mode = false;
    return solve_emulated_impl(ctxs, P, alg, outer, inner);
}

static duquad_status solve_emulated_impl(duquad_ctx **ctxs, int32_t P, int32_t alg, int32_t outer, int32_t inner) {
    if (!ctxs || P < 1) return fail(nullptr, DUQUAD_EINVAL, "need P >= 1 contexts");
    for (int r = 0; r < P; ++r) {
        duquad_ctx *c = ctxs[r];
        if (!c) return fail(nullptr, DUQUAD_EINVAL, "null context");
        if (c->world != P || c->rank != r || (P > 1 && !c->emulated) || c->stream != ctxs[0]->stream ||
            c->dev != ctxs[0]->dev || c->Btot > 1 || c->small || c->n != ctxs[0]->n || c->p != ctxs[0]->p)
            return fail(ctxs[0], DUQUAD_EINVAL,
                        "emulated group: contexts must be ranks 0..P-1 of one row-sharded problem with "
                        "emulate_ranks = 1 and the same device and stream (rank " + std::to_string(r) +
                            ": world " + std::to_string(c->world) + ", rank " + std::to_string(c->rank) +
                            ", emulated " + std::to_string(c->emulated) + ", small " + std::to_string(c->small) + ")");
        if (!c->have_consts) return fail(ctxs[0], DUQUAD_ESTATE, "constants not set");
    }
    if (alg != DUQUAD_DGM && alg != DUQUAD_DFGM) return fail(ctxs[0], DUQUAD_EINVAL, "bad alg");
    if (outer < 1 || inner < 1) return fail(ctxs[0], DUQUAD_EINVAL, "need outer_iters >= 1 and inner_iters >= 1");
    duquad_ctx *ctx = ctxs[0];
    DevGuard guard(ctx->dev);
    const int K = outer, Kin = inner;
    std::vector<double> beta_in;
    duquad_status st;
    for (int r = 0; r < P; ++r)
        if ((st = solve_prepare(ctxs[r], alg, K, Kin, beta_in)) != DUQUAD_OK) return st;
    if ((st = group_gather(ctxs, P, G_Y)) != DUQUAD_OK) return st;
    if (ctx->resumed && ctx->y_full2 && (st = group_gather(ctxs, P, G_Y2)) != DUQUAD_OK) return st;
    for (int j = 1; j <= K + 1 + (ctx->davg ? 1 : 0); ++j) {
        if (j == K + 1)
            for (int r = 0; r < P; ++r)
                if (ctxs[r]->opt.checkpoint && (st = save_checkpoint(ctxs[r])) != DUQUAD_OK) return st;
        for (int ph = 0; ph < num_phases(ctx, Kin); ++ph) {
            int gb = G_NONE;
            for (int r = 0; r < P; ++r)
                if ((st = outer_phase(ctxs[r], beta_in, Kin, j, ph, nullptr, &gb)) != DUQUAD_OK) return st;
            if ((st = group_gather(ctxs, P, gb)) != DUQUAD_OK) return st;
        }
    }
    CK(cudaStreamSynchronize(ctx->stream));
    int32_t any = 0;
    for (int r = 0; r < P; ++r) {
        int32_t flag = 0;
        CK(cudaMemcpy(&flag, ctxs[r]->d_flag, sizeof(flag), cudaMemcpyDeviceToHost));
        any |= flag;
        ctxs[r]->solved = true;
        if (ctxs[r]->opt.checkpoint && !flag) {
            ctxs[r]->ck_valid = true;
            ctxs[r]->ck_j = ctxs[r]->j0 + K;
            ctxs[r]->ck_S = ctxs[r]->S_end;
        }
    }
    if (any) return fail(ctx, DUQUAD_ENONFINITE, "an iterate became non-finite");
    return DUQUAD_OK;
}

static duquad_status get_result_batched(duquad_ctx *ctx, double *x_last, double *x_avg, double *lam,
                                        int32_t on_device);

duquad_status duquad_get_result(duquad_ctx *ctx, double *x_last, double *x_avg, double *lam, int32_t on_device) {
    if (!ctx) return fail(nullptr, DUQUAD_EINVAL, "ctx is NULL");
    if (!ctx->solved) return fail(ctx, DUQUAD_ESTATE, "no solve has run");
    DevGuard guard(ctx->dev);
    if (ctx->Btot > 1) return get_result_batched(ctx, x_last, x_avg, lam, on_device);
    const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (x_last) CK(cudaMemcpyAsync(x_last, ctx->x, ctx->nloc * sizeof(double), kind, ctx->stream));
    if (x_avg) CK(cudaMemcpyAsync(x_avg, ctx->xhat, ctx->nloc * sizeof(double), kind, ctx->stream));
    if (lam && ctx->ploc > 0) CK(cudaMemcpyAsync(lam, ctx->lam_prev, ctx->ploc * sizeof(double), kind, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return DUQUAD_OK;
}

static duquad_status get_result_batched(duquad_ctx *ctx, double *x_last, double *x_avg, double *lam,
                                        int32_t on_device) {
    const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    const int64_t n = ctx->n, p = ctx->p, B = ctx->Bloc, sp = std::max<int64_t>(ctx->ldp, 2);
    if (B > 0) {
        if (x_last)
            CK(cudaMemcpy2DAsync(x_last, n * 8, ctx->Xb, ctx->ld * 8, n * 8, B, kind, ctx->stream));
        if (x_avg)
            CK(cudaMemcpy2DAsync(x_avg, n * 8, ctx->XHb, ctx->ld * 8, n * 8, B, kind, ctx->stream));
        if (lam && p > 0) CK(cudaMemcpy2DAsync(lam, p * 8, ctx->lpb, sp * 8, p * 8, B, kind, ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
    return DUQUAD_OK;
}

duquad_status duquad_residuals(duquad_ctx *ctx, int32_t which, double *F, double *dist, double *lag) {
    if (!ctx) return fail(nullptr, DUQUAD_EINVAL, "ctx is NULL");
    if (!ctx->solved) return fail(ctx, DUQUAD_ESTATE, "no solve has run");
    if (which != 0 && which != 1) return fail(ctx, DUQUAD_EINVAL, "which must be 0 (x_last) or 1 (x_avg)");
    if (ctx->Btot > 1) return fail(ctx, DUQUAD_EINVAL, "residuals: single QP only");
    DevGuard guard(ctx->dev);
    cudaStream_t s = ctx->stream;
    duquad_status st;
    const double *xv = which == 0 ? ctx->x : ctx->xhat;
    double *yl = ctx->y_full + ctx->rank * ctx->n_slice;
    CK(cudaMemcpyAsync(yl, xv, ctx->nloc * sizeof(double), cudaMemcpyDeviceToDevice, s));
    if ((st = allgather_y(ctx)) != DUQUAD_OK) return st;
    PassAArgs a = make_a(ctx);
    a.lin_coef = 1.0;
    CK(launch_pass_a(a, MODE_LIN, ctx->cfg_a, s));          // qy = Q x, w_local = G x
    CK(launch_residual_partial(xv, ctx->qy, ctx->q, ctx->nloc, ctx->w_full + ctx->s0, ctx->g,
                               ctx->lam_prev, ctx->cone, ctx->ploc, ctx->rho, ctx->partials, s));
    double *acc = ctx->scal + SC_TMP;
    CK(launch_reduce_final(ctx->partials, kRedGrid, 5, acc, s));
    if ((st = allreduce_sum(ctx, acc, 5)) != DUQUAD_OK) return st;
    double h[5];
    CK(cudaMemcpyAsync(h, acc, sizeof(h), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (F) *F = h[0];
    if (dist) *dist = std::sqrt(h[1]);
    if (lag) *lag = ctx->rho > 0 ? h[0] + 0.5 * ctx->rho * h[2] - h[3] / (2.0 * ctx->rho) : h[0] + h[4];
    return DUQUAD_OK;
}

duquad_status duquad_solve_monitored(duquad_ctx *ctx, int32_t alg, int32_t outer_max, int32_t inner_iters,
                                     int32_t check_every, int32_t which, double eps, double F_star,
                                     duquad_monitor *mon, double *history, duquad_result *res) {
    if (!ctx) return fail(nullptr, DUQUAD_EINVAL, "ctx is NULL");
    if (outer_max < 1 || check_every < 1 || (which != 0 && which != 1) || !(eps > 0) || std::isinf(F_star))
        return fail(ctx, DUQUAD_EINVAL, "solve_monitored: outer_max, check_every >= 1; which 0/1; eps > 0; F_star finite or NaN");
    if (ctx->Btot > 1 || ctx->davg)
        return fail(ctx, DUQUAD_EINVAL, "solve_monitored: single QP, no dual_average");
    if (ctx->emulated) return fail(ctx, DUQUAD_EINVAL, "solve_monitored: not on emulated ranks");
    ctx->eps_mode = false;
    const int32_t ck_opt = ctx->opt.checkpoint;
    ctx->opt.checkpoint = 1;   // every segment ends with a snapshot the next one continues from
    duquad_monitor m{};
    duquad_result seg{};
    duquad_status st = DUQUAD_OK;
    int64_t done = 0;
    while (done < outer_max) {
        const int32_t K = (int32_t)std::min<int64_t>(check_every, outer_max - done);
        if (done > 0) ctx->resume = true;   // continue from the previous segment's checkpoint
        if ((st = solve_body(ctx, alg, K, inner_iters, &seg)) != DUQUAD_OK) break;
        done += K;
        m.inner_total += seg.inner_iters_total;
        m.passes_total += seg.matrix_passes;
        // residuals of both iterates; lag of x_last = u_bar(lambda^j) is the inexact dual value
        double F[2], d[2], lg[2];
        if ((st = duquad_residuals(ctx, 0, &F[0], &d[0], &lg[0])) != DUQUAD_OK) break;
        if ((st = duquad_residuals(ctx, 1, &F[1], &d[1], &lg[1])) != DUQUAD_OK) break;
        m.F = F[which];
        m.dist = d[which];
        m.dual = lg[0];
        if (history) {
            double *h = history + 8 * (int64_t)m.checks;
            h[0] = (double)(ctx->ck_j);
            h[1] = lg[0];
            h[2] = F[0];
            h[3] = F[1];
            h[4] = d[0];
            h[5] = d[1];
            h[6] = (double)m.inner_total;
            h[7] = (double)m.passes_total;
        }
        ++m.checks;
        const bool obj_ok = std::isnan(F_star) ? std::fabs(m.F - m.dual) <= eps * (1.0 + std::fabs(m.F))
                                               : std::fabs(m.F - F_star) <= eps;
        if (m.dist <= eps && obj_ok) {
            m.converged = 1;
            break;
        }
    }
    ctx->opt.checkpoint = ck_opt;
    ctx->resume = false;
    m.outer_done = done;
    if (mon) *mon = m;
    if (res) *res = seg;
    return st;
}

}  // extern "C"
