// Batched (MPC-shaped) sm_100a kernels: B QPs sharing Q and G (SURVEY.md §8(a) row a9,
// BASELINE.json configs[3], north_star (c)).
//
// With B right-hand sides the two passes of an inner step are real dense contractions:
//   pass A:  [Q;G] (n+p x n) . Y (n x B)   -> QY, and per (row, QP) the w / DFOM epilogue
//   pass B:  G'    (n x p)   . W (p x B)   -> per (row, QP) the clamp / momentum / average epilogue
// run on the FP64 tensor pipe with DMMA (`mma.sync.aligned.m8n8k4.row.col.f64`, SASS DMMA.8x8x4;
// tcgen05.mma has no f64 kind, and the larger f64 mma shapes lower to the same DMMA.8x8x4).
// Per-QP vectors are stored QP-major (B x ld, zero-padded to a multiple of 32), which is exactly
// the "col" B-operand layout, so no transposes are needed.
//
// One persistent, warp-specialised CTA per SM.  CTA c owns a contiguous range of QP octets
// (8 QPs), so there is no inter-CTA traffic; it walks the range in groups of <= NT octets, the
// rows in blocks of 128 (16 m8 tiles) and the reduction dimension in BK = 32 chunks:
//   - 2 producer warps stream the A chunk (128 x 32) and the B chunk (8*NT x 32) of every step
//     into a STAGES-deep shared-memory ring with cp.async; each thread's copies arrive on the
//     stage's "full" mbarrier (cp.async.mbarrier.arrive.noinc);
//   - 8 math warps (two per SM sub-partition; warp w owns m8 tiles w and w + 8 of the block and
//     all octets of the group) issue the DMMAs and release the stage on its "empty" mbarrier;
//   - pass A: the math warps apply the epilogue themselves.  Outside the DFOM step it needs one
//     operand per element, h = mu + rho g (constant within an outer iteration); two staging warps
//     copy the block's h tile into shared memory while the math warps run the block's DMMAs, the
//     math warps overwrite it in place with qy / w and write it out in 64-byte runs (the DFOM
//     step itself runs out of line, dual_block);
//   - pass B (one row block, seven operands per element): the math warps park the C tile in
//     shared memory and 6 epilogue warps apply it while the math warps run the CTA's next group.
// The DMMA pipe is the bound: 1 DMMA.8x8x4 per 16 cycles per sub-partition (measured,
// scripts/dmma_bench.cu: 37 TFLOP/s at 1965 MHz, reached with one warp and 4 accumulators).
// Measured on config 3 (profiles/r01_summary.md): the earlier 2-CTA/SM tile kernel ran the
// pipe at 30 % in pass A; separate epilogue warps next to DMMA-issuing warps ran ~3x slower than
// alone, which is why pass A folds its (light) epilogue into the math warps.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#ifdef DUQUAD_BATCHED_TRACE
#include <cstdio>
#include <cstring>
#endif

#include "duquad_internal.h"
#include "epilogue.cuh"

namespace dq {

namespace {

constexpr int BK = 32;
constexpr int PADK = BK + 4;    // smem row pitch (doubles): the 8x4 fragment loads of a half-warp hit 32 banks
constexpr int kMathW = 8, kProdW = 2;
constexpr int kBlkM = 128;      // rows per block: 16 m8 tiles
constexpr int LDC = kBlkM + 2;  // tiles Cs[qp][row]; 2 LDC = 4 mod 16 doubles: fragment-order accesses are conflict-free
constexpr int kSmemCap = 225 * 1024;

template <int PASS, int NT, bool PAIR = false>
struct Geo {
    static constexpr int EPIW = PASS == 0 ? 2 : 6;   // pass A: 2 h-staging warps; pass B: 6 epilogue warps
    static constexpr int THREADS = 32 * (kMathW + kProdW + EPIW);
    static constexpr int BN = 8 * NT;
    static constexpr int SA = kBlkM * PADK, SB = BN * PADK;   // doubles per stage
    static constexpr int CS = BN * LDC;   // pass B: parked C tile; pass A: staged h tile (same shape)
    static constexpr int NCS = PAIR ? 2 : 1;   // pass A, paired rows: h tiles of the top and the bottom rows
    static constexpr int STAGES = (kSmemCap - 8 * NCS * CS - 128) / (8 * (SA + SB));
    static constexpr size_t SMEM = 8 * ((size_t)STAGES * (SA + SB) + NCS * CS) + 128;
    static_assert(STAGES >= 2, "ring too shallow");
};

__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp16(double *smem, const double *gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp8(double *smem, const double *gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(su32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
// arrives once this thread's earlier cp.async copies have landed (init count includes it)
__device__ __forceinline__ void mbar_arrive_cp(uint64_t *b) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}

#ifdef DUQUAD_BATCHED_TRACE   // instrumentation build only: per-block timeline of CTA 0
__device__ unsigned long long g_btrace[8 * 64];
__device__ unsigned long long g_ctatrace[2 * 256];   // per CTA: start, end (globaltimer)
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define BTRACE(slot, cond)                                                             \
    do {                                                                               \
        if ((cond) && blockIdx.x == 0 && (threadIdx.x & 31) == 0) {                    \
            unsigned long long t_;                                                     \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                     \
            g_btrace[slot] = t_;                                                       \
        }                                                                              \
    } while (0)
#else
#define BTRACE(slot, cond) \
    do {                   \
    } while (0)
#endif

struct Group {
    int64_t q0;   // first QP
    int nq, nc;   // valid QPs, octets
};
// CTA c owns octets [c*ncol8/grid, (c+1)*ncol8/grid) and walks them in ng groups of <= NT octets,
// the larger groups first (the last group's epilogue is the one left exposed).
struct Range {
    int64_t o0, len;
    int ng;
};
template <int NT>
__device__ __forceinline__ Range cta_range(const BatchedArgs &a) {
    Range r;
    r.o0 = (int64_t)blockIdx.x * a.ncol8 / gridDim.x;
    r.len = ((int64_t)blockIdx.x + 1) * a.ncol8 / gridDim.x - r.o0;
    r.ng = (int)((r.len + NT - 1) / NT);
    return r;
}
__device__ __forceinline__ Group group_of(const BatchedArgs &a, const Range &r, int k) {
    const int64_t c0 = r.o0 + ((int64_t)k * r.len + r.ng - 1) / r.ng;
    const int64_t c1 = r.o0 + ((int64_t)(k + 1) * r.len + r.ng - 1) / r.ng;
    Group g;
    g.q0 = 8 * c0;
    g.nc = (int)(c1 - c0);
    const int64_t nq = a.N - g.q0 < 8 * (c1 - c0) ? a.N - g.q0 : 8 * (c1 - c0);
    g.nq = nq > 0 ? (int)nq : 0;
    return g;
}

struct MathCtx {
    const double *As, *Bs;
    double *Cs, *Cs2;
    uint64_t *full, *empty, *cs_full, *cs_empty;
    uint32_t s, blk;
    int nkc, warp, lane;
};

// The K loop of one row block on math warp `warp`: m8 tiles warp and warp + 8 (TWO) or warp only,
// C octets; every DMMA unconditional so the loop body carries no per-instruction guards.
template <int ST, int SA, int SB, int C, bool TWO>
__device__ __forceinline__ void kloop(MathCtx &x, double (&acc)[2][C][2]) {
    const int fr = x.lane >> 2, fk = x.lane & 3;
#pragma unroll
    for (int j = 0; j < C; ++j) acc[0][j][0] = acc[0][j][1] = acc[1][j][0] = acc[1][j][1] = 0.0;
    for (int kc = 0; kc < x.nkc; ++kc, ++x.s) {
        const int slot = (int)(x.s % ST);
        mbar_wait(x.full + slot, (x.s / ST) & 1);
        const double *as = x.As + slot * SA + (8 * x.warp + fr) * PADK + fk;
        const double *bs = x.Bs + slot * SB + fr * PADK + fk;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double bf[C];
#pragma unroll
            for (int j = 0; j < C; ++j) bf[j] = bs[j * 8 * PADK + kk];
            const double a0 = as[kk];
            const double a1 = TWO ? as[64 * PADK + kk] : 0.0;
#pragma unroll
            for (int j = 0; j < C; ++j) {
                dmma(acc[0][j][0], acc[0][j][1], a0, bf[j]);
                if (TWO) dmma(acc[1][j][0], acc[1][j][1], a1, bf[j]);
            }
        }
        mbar_arrive(x.empty + slot);
    }
}

// The DFOM step for paired rows (G row k + P = -G row k): the block's reduced row k carries
// s = G_k u_bar; row k takes r = s + g_k, row k + P takes r = -s + g_{k+P} (bitwise the unpaired
// product, -s being exact), each with epilogue.cuh's dfom_row; the output is d_k = w_k - w_{k+P}
// (the operand of pass B's G_t' d).
__device__ __noinline__ void dual_block_pair(const double *Cs, const double *g, double *mu, double *lam_prev,
                                             double *hh, double *w, double *qy, const uint8_t *cone, double rho,
                                             double step, int project_dual, double beta_out, double *lam_hat,
                                             int mu_hat, double lhat_w, int64_t sn, int64_t sp, int64_t nq,
                                             int64_t M, int64_t q0, int nqp, int64_t m0, int ne, int ni, int warp,
                                             int lane, int64_t P, int64_t sw) {
    const int fr = lane >> 2, fk = lane & 3;
    for (int i = 0; i < ni; ++i) {
        const int rl = 8 * (warp + 8 * i) + fr;
        const int64_t row = m0 + rl;
        if (row >= M) continue;
        if (row < nq) {   // Q row: qy
            for (int e = 0; e < ne; ++e) {
                const int qp = 8 * (e >> 1) + 2 * fk + (e & 1);
                if (qp < nqp) qy[(q0 + qp) * sn + row] = Cs[qp * LDC + rl];
            }
            continue;
        }
        const int64_t k = row - nq;
        const uint8_t c0 = cone[k], c1 = cone[k + P];
        constexpr int E = 4;
        for (int e0 = 0; e0 < ne; e0 += E) {
            double gv[2][E], mv[2][E], lv[2][E];
#pragma unroll
            for (int u = 0; u < E; ++u) {
                const int e = e0 + u, qp = 8 * (e >> 1) + 2 * fk + (e & 1);
                if (e < ne && qp < nqp) {
                    const int64_t off = (q0 + qp) * sp + k;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        gv[h][u] = g[off + h * P];
                        mv[h][u] = mu[off + h * P];
                        lv[h][u] = lam_prev[off + h * P];
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < E; ++u) {
                const int e = e0 + u, qp = 8 * (e >> 1) + 2 * fk + (e & 1);
                if (e < ne && qp < nqp) {
                    const int64_t off = (q0 + qp) * sp + k;
                    const double s = Cs[qp * LDC + rl];
                    double wv[2];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const uint8_t c = h ? c1 : c0;
                        const double r = (h ? -s : s) + gv[h][u];
                        double lam;
                        double m = dfom_row(r, mv[h][u], lv[h][u], c, rho, step, project_dual, beta_out, lam);
                        if (lhat_w != 0.0) {   // DGM dual averaging
                            OuterA oa{1, beta_out, mu_hat, lhat_w};
                            double lh;
                            m = dual_average(lam_hat[off + h * P], lam, m, oa, lh);
                            lam_hat[off + h * P] = lh;
                        }
                        lam_prev[off + h * P] = lam;
                        mu[off + h * P] = m;
                        hh[off + h * P] = m + rho * gv[h][u];
                        wv[h] = rho > 0.0 ? proj_polar(m + rho * r, c) : m;
                    }
                    w[(q0 + qp) * sw + k] = wv[0] - wv[1];
                }
            }
        }
    }
}

// The DFOM step of pass A (first inner step of an outer iteration) for the elements of
// one math warp, whose accumulators are parked in the tile Cs[qp][row - m0]: epilogue.cuh's
// dfom_row per element, operands of 7 elements per lane-row loaded before any is used.  Out of
// line: it runs on 1 launch in K_in and must not cost the hot loop registers.
__device__ __noinline__ void dual_block(const double *Cs, const double *g, double *mu, double *lam_prev, double *hh,
                                        double *w, double *qy, const uint8_t *cone, double rho, double step,
                                        int project_dual, double beta_out, double *lam_hat, int mu_hat,
                                        double lhat_w, int64_t sn, int64_t sp, int64_t nq,
                                        int64_t M, int64_t q0, int nqp, int64_t m0, int ne, int ni, int warp,
                                        int lane) {
    const int fr = lane >> 2, fk = lane & 3;
    for (int i = 0; i < ni; ++i) {
        const int rl = 8 * (warp + 8 * i) + fr;
        const int64_t row = m0 + rl;
        if (row >= M) continue;
        if (row < nq) {   // Q row: qy
            for (int e = 0; e < ne; ++e) {
                const int qp = 8 * (e >> 1) + 2 * fk + (e & 1);
                if (qp < nqp) qy[(q0 + qp) * sn + row] = Cs[qp * LDC + rl];
            }
            continue;
        }
        const int64_t k = row - nq;
        const uint8_t c = cone[k];
        constexpr int E = 7;
        for (int e0 = 0; e0 < ne; e0 += E) {
            double gv[E], mv[E], lv[E];
#pragma unroll
            for (int u = 0; u < E; ++u) {
                const int e = e0 + u, qp = 8 * (e >> 1) + 2 * fk + (e & 1);
                if (e < ne && qp < nqp) {
                    const int64_t off = (q0 + qp) * sp + k;
                    gv[u] = g[off];
                    mv[u] = mu[off];
                    lv[u] = lam_prev[off];
                }
            }
#pragma unroll
            for (int u = 0; u < E; ++u) {
                const int e = e0 + u, qp = 8 * (e >> 1) + 2 * fk + (e & 1);
                if (e < ne && qp < nqp) {
                    const int64_t off = (q0 + qp) * sp + k;
                    const double r = Cs[qp * LDC + rl] + gv[u];
                    double lam;
                    double m = dfom_row(r, mv[u], lv[u], c, rho, step, project_dual, beta_out, lam);
                    if (lhat_w != 0.0) {   // DGM dual averaging
                        OuterA oa{1, beta_out, mu_hat, lhat_w};
                        double lh;
                        m = dual_average(lam_hat[off], lam, m, oa, lh);
                        lam_hat[off] = lh;
                    }
                    lam_prev[off] = lam;
                    mu[off] = m;
                    hh[off] = m + rho * gv[u];
                    w[off] = rho > 0.0 ? proj_polar(m + rho * r, c) : m;
                }
            }
        }
    }
}

// ---------------------------------------------------------------- pass A: block with in-register epilogue
// Fragment element (i, j, h) of lane (fr, fk): row m0 + 8 (warp + 8 i) + fr, QP q0 + 8 j + 2 fk + h.
// Arithmetic: epilogue.cuh's, with [mu + rho (s + g)]_{K°} regrouped as [h + rho s]_{K°} outside
// the DFOM step (reading c22); h comes from the tile the producers staged in x.Cs
// (Hs[qp][row - m0]).
template <int ST, int SA, int SB, int C, bool TWO, bool PAIR>
__device__ __forceinline__ void block_a(MathCtx &x, const BatchedArgs &args, const Group &gr, int64_t m0,
                                        const OuterA &o) {
    constexpr int NI = TWO ? 2 : 1;
    const PassAArgs &A = args.a;
    const int fr = x.lane >> 2, fk = x.lane & 3;
    const double rho = A.rho;
    int64_t row[NI];
    int kr[NI];   // G-row index, -1 for a Q row, -2 beyond M
    uint8_t cn[NI], cb[NI];   // cone tags of the G row (paired: of its top and bottom rows)
#pragma unroll
    for (int i = 0; i < NI; ++i) {
        row[i] = m0 + 8 * (x.warp + 8 * i) + fr;
        kr[i] = row[i] >= args.M ? -2 : row[i] < A.nq ? -1 : (int)(row[i] - A.nq);
        cn[i] = kr[i] >= 0 ? A.cone[kr[i]] : 0;   // lands during the K loop
        cb[i] = PAIR && kr[i] >= 0 ? A.cone[kr[i] + args.pairP] : 0;
    }
    double acc[2][C][2];
    BTRACE(8 * (x.blk & 63) + 0, x.warp == 0);
    kloop<ST, SA, SB, C, TWO>(x, acc);
    BTRACE(8 * (x.blk & 63) + 1, x.warp == 0);
    mbar_wait(x.cs_full, x.blk & 1);   // the h tile of this block
    BTRACE(8 * (x.blk & 63) + 3, x.warp == 0);
    if (!o.dual) {
        // (1) results in place in the tile: Hs[qp][r] := qy (Q row) or w (G row); immediate offsets.
        // Paired rows: the tiles hold h of the top and of the bottom row; d = w_top - w_bottom, the
        // bottom row's product being -s (exactly the unpaired one)
        double *hs = x.Cs + (2 * fk) * LDC + 8 * x.warp + fr;
        const double *hs2 = x.Cs2 + (2 * fk) * LDC + 8 * x.warp + fr;
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            const bool q_row = kr[i] == -1;
#pragma unroll
            for (int j = 0; j < C; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    double *e = hs + (8 * j + h) * LDC + 64 * i;
                    const double sv = acc[i][j][h];
                    if (PAIR) {
                        const double hb = hs2[(8 * j + h) * LDC + 64 * i];
                        const double wt = rho > 0.0 ? proj_polar(*e + rho * sv, cn[i]) : *e;
                        const double wb = rho > 0.0 ? proj_polar(hb + rho * (-sv), cb[i]) : hb;
                        *e = q_row ? sv : wt - wb;
                    } else {
                        *e = q_row ? sv : rho > 0.0 ? proj_polar(*e + rho * sv, cn[i]) : *e;
                    }
                }
        }
        __syncwarp();
        BTRACE(8 * (x.blk & 63) + 7, x.warp == 0);
        // (2) the warp's rows to global: lane -> (QP it * 4 + lane / 8, row lane % 8), 64-byte runs
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            const int rl = 8 * (x.warp + 8 * i) + (x.lane & 7);   // block row of this lane
            const int64_t r = m0 + rl;
            if (r < args.M) {
                const bool q_row = r < A.nq;
                const int64_t ld = q_row ? args.sn : args.sw;
                double *dst = (q_row ? A.qy + r : A.w + (r - A.nq)) + (gr.q0 + (x.lane >> 3)) * ld;
                const double *src = x.Cs + (x.lane >> 3) * LDC + rl;
                const int64_t step = 4 * ld;
#pragma unroll 4
                for (int qp = x.lane >> 3; qp < gr.nq; qp += 4, dst += step, src += 4 * LDC) *dst = *src;
            }
        }
    } else {   // the DFOM step (first inner step of an outer iteration), epilogue.cuh's dfom_row
        // park the accumulators in the (unused) h tile first, so they are not live across the loads
#pragma unroll
        for (int j = 0; j < C; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int i = 0; i < NI; ++i) x.Cs[(8 * j + 2 * fk + h) * LDC + (int)(row[i] - m0)] = acc[i][j][h];
        __syncwarp();
        if (PAIR)   // reduced row k is G row k (s) and G row k + P (-s, exactly)
            dual_block_pair(x.Cs, A.g, A.mu, A.lam_prev, A.h, A.w, A.qy, A.cone, rho, A.step, A.project_dual,
                            o.beta_out, A.lam_hat, o.mu_hat, o.lhat_w, args.sn, args.sp, A.nq, args.M, gr.q0, gr.nq,
                            m0, 2 * C, TWO ? 2 : 1, x.warp, x.lane, args.pairP, args.sw);
        else
            dual_block(x.Cs, A.g, A.mu, A.lam_prev, A.h, A.w, A.qy, A.cone, rho, A.step, A.project_dual, o.beta_out,
                       A.lam_hat, o.mu_hat, o.lhat_w, args.sn, args.sp, A.nq, args.M, gr.q0, gr.nq, m0, 2 * C,
                       TWO ? 2 : 1, x.warp, x.lane);
    }
    mbar_arrive(x.cs_empty);
    BTRACE(8 * (x.blk & 63) + 2, x.warp == 0);
    ++x.blk;
}

// ---------------------------------------------------------------- pass B: block parked in smem
template <int ST, int SA, int SB, int C, bool TWO>
__device__ __forceinline__ void block_b(MathCtx &x) {
    const int fr = x.lane >> 2, fk = x.lane & 3;
    double acc[2][C][2];
    BTRACE(8 * (x.blk & 63) + 0, x.warp == 0);
    kloop<ST, SA, SB, C, TWO>(x, acc);
    BTRACE(8 * (x.blk & 63) + 1, x.warp == 0);
    // park the C tile QP-major (fragment: row fr, cols 2fk, 2fk+1 of each 8x8 tile)
    mbar_wait(x.cs_empty, (x.blk & 1) ^ 1);
    BTRACE(8 * (x.blk & 63) + 2, x.warp == 0);
#pragma unroll
    for (int j = 0; j < C; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            x.Cs[(8 * j + 2 * fk + h) * LDC + 8 * x.warp + fr] = acc[0][j][h];
            if (TWO) x.Cs[(8 * j + 2 * fk + h) * LDC + 8 * (x.warp + 8) + fr] = acc[1][j][h];
        }
    mbar_arrive(x.cs_full);
    ++x.blk;
}

template <int PASS, int NT, bool PAIR, int C>
__device__ __forceinline__ void block_sel(MathCtx &x, const BatchedArgs &args, const Group &gr, int64_t m0,
                                          const OuterA &o) {
    using GE = Geo<PASS, NT, PAIR>;
    const bool two = m0 + 8 * (x.warp + 8) < args.M;
    if (gr.nc == C) {
        if (PASS == 0) {
            if (two)
                block_a<GE::STAGES, GE::SA, GE::SB, C, true, PAIR>(x, args, gr, m0, o);
            else
                block_a<GE::STAGES, GE::SA, GE::SB, C, false, PAIR>(x, args, gr, m0, o);
        } else {
            if (two)
                block_b<GE::STAGES, GE::SA, GE::SB, C, true>(x);
            else
                block_b<GE::STAGES, GE::SA, GE::SB, C, false>(x);
        }
    } else if constexpr (C > 1) {
        block_sel<PASS, NT, PAIR, C - 1>(x, args, gr, m0, o);
    }
}

// Pass B epilogue (one block of one group, from the parked C tile): x+ = clamp(y - (qy + q + G'w)
// / L_in), momentum, running average.  Lanes own rows m0 + lane + 32 t, so
// the bounds are loaded once per block; epilogue.cuh's arithmetic expression for expression.
constexpr int RPL = kBlkM / 32;
__device__ __forceinline__ void epi_block_b(const BatchedArgs &args, const double *Cs, int64_t m0, const Group &gr,
                                            int wid, int nwk, int lane, double avg_w) {
    const PassBArgs &B = args.b;
    const double L = B.L_in, beta = B.beta_in;
    const bool last = B.last_inner != 0;
    int jj[RPL];
    double lbv[RPL], ubv[RPL];
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
        const int64_t j = m0 + lane + 32 * t;
        jj[t] = j < args.M ? (int)j : -1;
        lbv[t] = jj[t] >= 0 ? B.lb[j] : 0.0;
        ubv[t] = jj[t] >= 0 ? B.ub[j] : 0.0;
    }
    bool bad = false;
    for (int col = wid; col < gr.nq; col += nwk) {
        if (args.done_b && args.done_b[gr.q0 + col]) continue;   // eps_in mode: this QP's inner solve stopped
        const int64_t off = (gr.q0 + col) * args.sn;
        const double *qyp = B.qy + off, *qp = B.q + off;
        double *xp = B.x + off, *yp = B.y + off, *hp = B.xhat + off;
        const double *cs = Cs + col * LDC + lane;
        double vq[RPL], vqy[RPL], vx[RPL], vy[RPL], vh[RPL];
#pragma unroll
        for (int t = 0; t < RPL; ++t)
            if (jj[t] >= 0) {
                vqy[t] = qyp[jj[t]];
                vq[t] = qp[jj[t]];
                vx[t] = xp[jj[t]];
                vy[t] = yp[jj[t]];
                vh[t] = avg_w != 0.0 ? hp[jj[t]] : 0.0;
            }
#pragma unroll
        for (int t = 0; t < RPL; ++t)
            if (jj[t] >= 0) {
                const double grad = (vqy[t] + vq[t]) + cs[32 * t];
                const double xn = fmin(fmax(vy[t] - grad / L, lbv[t]), ubv[t]);
                const double yn = last ? xn : xn + beta * (xn - vx[t]);
                if (avg_w != 0.0) hp[jj[t]] = vh[t] + avg_w * (xn - vh[t]);
                xp[jj[t]] = xn;
                yp[jj[t]] = yn;
                bad |= !isfinite(xn) || !isfinite(yn);
                if (args.gm_b) {   // eps_in mode: (y - x+)^2, this column's rows
                    const double dd = vy[t] - xn;
                    vh[t] = dd * dd;
                }
            } else {
                vh[t] = 0.0;
            }
        if (args.gm_b) {   // the QP's sum: rows in lane order, blocks in order (one warp per column)
            double gsum = 0.0;
#pragma unroll
            for (int t = 0; t < RPL; ++t) gsum += vh[t];
            gsum = warp_sum(gsum);
            if (lane == 0) atomicAdd(&args.gm_b[gr.q0 + col], gsum);
        }
    }
    if (bad) *B.flag = 1;
}

// C[m][b] = sum_k A[m][k] * Bop[b][k];  A: M x K row-major (lda), Bop: N x K (ldb), K padded to BK.
template <int PASS, int NT, bool PAIR>
__global__ void __launch_bounds__(Geo<PASS, NT, PAIR>::THREADS, 1) k_batched(const BatchedArgs args) {
    using GE = Geo<PASS, NT, PAIR>;
    constexpr int ST = GE::STAGES;
    extern __shared__ __align__(16) double smem[];
    double *As = smem;
    double *Bs = As + ST * GE::SA;
    double *Cs = Bs + ST * GE::SB;
    double *Cs2 = Cs + (GE::NCS - 1) * GE::CS;   // paired rows: the bottom rows' h tile
    uint64_t *bars = reinterpret_cast<uint64_t *>(Cs + GE::NCS * GE::CS);
    uint64_t *full = bars, *empty = bars + ST, *cs_full = bars + 2 * ST, *cs_empty = cs_full + 1;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#ifdef DUQUAD_BATCHED_TRACE
    if (tid == 0 && blockIdx.x < 256) g_ctatrace[2 * blockIdx.x] = gtimer();
#endif
    if (tid == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(full + s, kProdW * 32);
            mbar_init(empty + s, kMathW * 32);
        }
        // pass B: C tile math -> epilogue warps; pass A: h tile producers -> math warps
        mbar_init(cs_full, PASS == 0 ? GE::EPIW * 32 : kMathW * 32);
        mbar_init(cs_empty, PASS == 0 ? kMathW * 32 : GE::EPIW * 32);
    }
    __syncthreads();
    const int nmb = (int)((args.M + kBlkM - 1) / kBlkM), nkc = (int)(args.K / BK);
    const Range rg = cta_range<NT>(args);
    // the producers' A operand (the shared matrix: never written by a solve) of the first ST ring
    // chunks, before the PDL dependency wait (epilogue.cuh): the ring fill overlaps the previous
    // kernel's tail; the B operand (the iterates) and everything else come after it
    const bool producer = warp >= kMathW && warp < kMathW + kProdW;
    const int pt = tid - 32 * kMathW;
    auto issue_a = [&](int64_t m0, int kc, int slot) {
        const int rows = (int)(args.M - m0 < kBlkM ? args.M - m0 : kBlkM);
        double *as = As + slot * GE::SA;
        const double *ag = args.Aop + m0 * args.lda + (int64_t)kc * BK;
        for (int i = pt; i < rows * (BK / 2); i += 32 * kProdW) {
            const int r = i / (BK / 2), c = (i % (BK / 2)) * 2;
            cp16(as + r * PADK + c, ag + r * args.lda + c);
        }
    };
    uint32_t pre = 0;   // chunks whose A part is in flight already
    if (producer) {
        for (int k = 0; k < rg.ng && pre < (uint32_t)ST; ++k) {
            if (group_of(args, rg, k).nq == 0) continue;
            for (int mb = 0; mb < nmb && pre < (uint32_t)ST; ++mb)
                for (int kc = 0; kc < nkc && pre < (uint32_t)ST; ++kc, ++pre) issue_a((int64_t)mb * kBlkM, kc, (int)pre);
        }
    }
    pdl_wait();
    pdl_trigger();
    if (args.ndone && *args.ndone >= args.N) {   // eps_in mode: every QP's inner solve has stopped
        if (producer) asm volatile("cp.async.wait_all;" ::: "memory");
        return;
    }
    const OuterA o = PASS == 0 ? outer_a(args.a, MODE_SOLVE) : OuterA{0, 0.0};

    if (warp < kMathW) {   // ------------------------------------------------ math warps
        MathCtx x{As, Bs, Cs, Cs2, full, empty, cs_full, cs_empty, 0u, 0u, nkc, warp, lane};
        for (int k = 0; k < rg.ng; ++k) {
            const Group gr = group_of(args, rg, k);
            if (gr.nq == 0) continue;
            for (int mb = 0; mb < nmb; ++mb) block_sel<PASS, NT, PAIR, NT>(x, args, gr, (int64_t)mb * kBlkM, o);
        }
    } else if (producer) {   // ------------------------------------------------------ producer warps
        uint32_t s = 0;
        for (int k = 0; k < rg.ng; ++k) {
            const Group gr = group_of(args, rg, k);
            if (gr.nq == 0) continue;
            for (int mb = 0; mb < nmb; ++mb) {
                const int64_t m0 = (int64_t)mb * kBlkM;
                for (int kc = 0; kc < nkc; ++kc, ++s) {
                    const int slot = (int)(s % ST);
                    mbar_wait(empty + slot, ((s / ST) & 1) ^ 1);
                    BTRACE(8 * ((mb + k * nmb) & 63) + 6, kc == 0 && warp == kMathW);
                    if (s >= pre) issue_a(m0, kc, slot);
                    double *bs = Bs + slot * GE::SB;
                    const double *bg = args.Bop + gr.q0 * args.ldb + (int64_t)kc * BK;
                    for (int i = pt; i < gr.nq * (BK / 2); i += 32 * kProdW) {
                        const int r = i / (BK / 2), c = (i % (BK / 2)) * 2;
                        cp16(bs + r * PADK + c, bg + r * args.ldb + c);
                    }
                    mbar_arrive_cp(full + slot);
                }
            }
        }
    } else if (PASS == 0) {   // ----------------------------------------------- h-staging warps (pass A)
        // the block's h tile Hs[qp][row - m0] (G rows; none on DFOM-step launches), QP columns
        // split over the staging warps; Hs is free once the math warps wrote the previous block out
        const int st = tid - 32 * (kMathW + kProdW), nst = 32 * GE::EPIW;
        uint32_t hb = 0;
        for (int k = 0; k < rg.ng; ++k) {
            const Group gr = group_of(args, rg, k);
            if (gr.nq == 0) continue;
            for (int mb = 0; mb < nmb; ++mb, ++hb) {
                const int64_t m0 = (int64_t)mb * kBlkM;
                const int64_t r0 = m0 > args.a.nq ? m0 : args.a.nq;
                const int64_t r1 = args.M < m0 + kBlkM ? args.M : m0 + kBlkM;
                mbar_wait(cs_empty, (hb & 1) ^ 1);
                BTRACE(8 * (hb & 63) + 4, warp == kMathW + kProdW);
                if (!o.dual && r1 > r0) {
                    const int nr = (int)(r1 - r0), k0 = (int)(r0 - args.a.nq), d0 = (int)(r0 - m0);
                    // paired rows: tile 2 holds h of the bottom rows k + P
                    for (int t = 0; t < GE::NCS; ++t) {
                        double *ct = t ? Cs2 : Cs;
                        const int kt = k0 + (t ? (int)args.pairP : 0);
                        if (((kt | d0 | (int)args.sp) & 1) == 0) {   // 16-byte pairs (+ an odd tail element)
                            const int np = (nr + 1) / 2;
                            for (int i = st; i < gr.nq * np; i += nst) {
                                const int c = i / np, r = 2 * (i % np);
                                const double *src = args.a.h + (gr.q0 + c) * args.sp + kt + r;
                                if (r + 1 < nr)
                                    cp16(ct + c * LDC + d0 + r, src);
                                else
                                    cp8(ct + c * LDC + d0 + r, src);
                            }
                        } else {
                            for (int i = st; i < gr.nq * nr; i += nst) {
                                const int c = i / nr, r = i % nr;
                                cp8(ct + c * LDC + d0 + r, args.a.h + (gr.q0 + c) * args.sp + kt + r);
                            }
                        }
                    }
                }
                mbar_arrive_cp(cs_full);
                BTRACE(8 * (hb & 63) + 5, warp == kMathW + kProdW);
            }
        }
    } else {   // ------------------------------------------------------------------ epilogue warps (pass B)
        const int wid = warp - kMathW - kProdW;
        const double avg_w = avg_weight(args.b, MODE_SOLVE);
        uint32_t blk = 0;
        for (int k = 0; k < rg.ng; ++k) {
            const Group gr = group_of(args, rg, k);
            if (gr.nq == 0) continue;
            for (int mb = 0; mb < nmb; ++mb) {
                mbar_wait(cs_full, blk & 1);
                BTRACE(8 * (blk & 63) + 4, wid == 0);
                epi_block_b(args, Cs, (int64_t)mb * kBlkM, gr, wid, GE::EPIW, lane, avg_w);
                BTRACE(8 * (blk & 63) + 5, wid == 0);
                mbar_arrive(cs_empty);
                ++blk;
            }
        }
    }
#ifdef DUQUAD_BATCHED_TRACE
    __syncthreads();
    if (tid == 0 && blockIdx.x < 256) g_ctatrace[2 * blockIdx.x + 1] = gtimer();
#endif
}

// Pass A reuses each (128 x 32) A chunk over 7 octets (56 QPs); pass B (one row block for
// n <= 128) uses 4-octet groups, two per CTA, so the epilogue of a CTA's first group overlaps
// the math of its second.
constexpr int kNTA = 7, kNTB = 4;

int g_num_sms = 0;   // grid cap: the SM count, or DUQUAD_BATCHED_CTAS (tests: several groups per CTA)

template <int PASS, int NT, bool PAIR>
cudaError_t launch_t(BatchedArgs a, cudaStream_t s) {
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
        if (const char *e = getenv("DUQUAD_BATCHED_CTAS"))
            if (atoi(e) > 0 && atoi(e) < g_num_sms) g_num_sms = atoi(e);
    }
    a.ncol8 = (a.N + 7) / 8;
    const int64_t nctas = a.ncol8 < g_num_sms ? a.ncol8 : g_num_sms;
    cudaError_t e = launch_ex(k_batched<PASS, NT, PAIR>, (unsigned)nctas, Geo<PASS, NT, PAIR>::THREADS,
                              Geo<PASS, NT, PAIR>::SMEM, s, a.pdl, 0, a);
    if (e) return e;
#ifdef DUQUAD_BATCHED_TRACE
    {
        unsigned long long h[8 * 64];
        cudaStreamSynchronize(s);
        cudaMemcpyFromSymbol(h, g_btrace, sizeof h);
        const unsigned long long t0 = h[0];
        for (int b = 0; b < 8 && h[8 * b]; ++b) {
            fprintf(stderr, "pass %c blk %d:", PASS == 0 ? 'A' : 'B', b);
            for (int c = 0; c < 8; ++c) fprintf(stderr, " %7.2f", h[8 * b + c] ? (double)(h[8 * b + c] - t0) / 1e3 : -1.0);
            fprintf(stderr, "\n");
        }
        memset(h, 0, sizeof h);
        cudaMemcpyToSymbol(g_btrace, h, sizeof h);
        unsigned long long c[2 * 256];
        cudaMemcpyFromSymbol(c, g_ctatrace, sizeof c);
        unsigned long long s0 = ~0ull, s1 = 0, e0 = ~0ull, e1 = 0;
        for (int b = 0; b < (int)nctas && b < 256; ++b) {
            s0 = c[2 * b] < s0 ? c[2 * b] : s0;
            s1 = c[2 * b] > s1 ? c[2 * b] : s1;
            e0 = c[2 * b + 1] < e0 ? c[2 * b + 1] : e0;
            e1 = c[2 * b + 1] > e1 ? c[2 * b + 1] : e1;
        }
        fprintf(stderr, "pass %c CTAs: start %.2f..%.2f us, end %.2f..%.2f us (from the first start; CTA 0 ends %.2f)\n",
                PASS == 0 ? 'A' : 'B', 0.0, (s1 - s0) / 1e3, (e0 - s0) / 1e3, (e1 - s0) / 1e3, (c[1] - s0) / 1e3);
    }
#endif
    return cudaGetLastError();
}

template <int PASS, int NT, bool PAIR>
cudaError_t configure_t() {
    return cudaFuncSetAttribute(k_batched<PASS, NT, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)Geo<PASS, NT, PAIR>::SMEM);
}

}  // namespace

cudaError_t configure_batched_kernels() {
    cudaError_t e;
    if ((e = configure_t<0, kNTA, false>())) return e;
    if ((e = configure_t<0, kNTA, true>())) return e;
    if ((e = configure_t<0, 5, true>())) return e;
    if ((e = configure_t<0, 4, true>())) return e;
    if ((e = configure_t<1, 7, false>())) return e;
    if ((e = configure_t<1, 3, false>())) return e;
    return configure_t<1, kNTB, false>();
}

cudaError_t launch_batched(const BatchedArgs &a, int pass, int mode, cudaStream_t s) {
    if (a.N <= 0 || a.M <= 0) return cudaSuccess;
    if (mode != MODE_SOLVE) return cudaErrorInvalidValue;   // the batched path runs solve passes only
    // group widths (octets per group): measurement overrides DUQUAD_NTA_PAIR / DUQUAD_NTB
    static const int nta_pair = getenv("DUQUAD_NTA_PAIR") ? atoi(getenv("DUQUAD_NTA_PAIR")) : kNTA;
    static const int ntb = getenv("DUQUAD_NTB") ? atoi(getenv("DUQUAD_NTB")) : kNTB;
    if (pass == 1) return ntb == 7 ? launch_t<1, 7, false>(a, s) : ntb == 3 ? launch_t<1, 3, false>(a, s)
                                                                             : launch_t<1, kNTB, false>(a, s);
    if (a.pairP > 0)
        return nta_pair == 5 ? launch_t<0, 5, true>(a, s) : nta_pair == 4 ? launch_t<0, 4, true>(a, s)
                                                                            : launch_t<0, kNTA, true>(a, s);
    return launch_t<0, kNTA, false>(a, s);
}

// eps_in mode (per QP): the stop test on the QP's sum of (y - x+)^2, then the sum is cleared
__global__ void k_batched_decide(double *gm_b, int32_t *done_b, int32_t *ndone, double thresh2, int32_t *counts,
                                 int64_t nc, const int32_t *d_j, int64_t B) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= B) return;
    if (!done_b[q]) {
        counts[q * nc + *d_j - 1] += 1;
        if (gm_b[q] <= thresh2) {
            done_b[q] = 1;
            atomicAdd(ndone, 1);
        }
    }
    gm_b[q] = 0.0;
}

// end of an inner solve in eps_in mode: y = x (warm start), running average, the QP's
// converged flag recorded and its stop flag cleared for the next outer iteration
__global__ void k_batched_finish(const double *x, double *y, double *xhat, int64_t n, int64_t sn, int64_t B,
                                 const OuterParam *ops, const int32_t *d_j, int32_t *done_b, int32_t *conv,
                                 int64_t nc) {
    const double w = ops[*d_j].avg_w;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < B * sn; t += (int64_t)gridDim.x * blockDim.x) {
        if (t % sn >= n) continue;
        const double xi = x[t];
        y[t] = xi;
        if (w != 0.0) xhat[t] = xhat[t] + w * (xi - xhat[t]);
    }
}

__global__ void k_batched_reset(int32_t *done_b, int32_t *ndone, int32_t *conv, int64_t nc, const int32_t *d_j,
                                int64_t B) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q < B) {
        conv[q * nc + *d_j - 1] = done_b[q];
        done_b[q] = 0;
    }
    if (q == 0) *ndone = 0;
}

cudaError_t launch_batched_decide(double *gm_b, int32_t *done_b, int32_t *ndone, double thresh2, int32_t *counts,
                                  int64_t nc, const int32_t *d_j, int64_t B, cudaStream_t s) {
    if (B > 0) k_batched_decide<<<(unsigned)((B + 255) / 256), 256, 0, s>>>(gm_b, done_b, ndone, thresh2, counts, nc, d_j, B);
    return cudaGetLastError();
}

cudaError_t launch_batched_finish(const double *x, double *y, double *xhat, int64_t n, int64_t sn, int64_t B,
                                  const OuterParam *ops, const int32_t *d_j, int32_t *done_b, int32_t *ndone,
                                  int32_t *conv, int64_t nc, cudaStream_t s) {
    if (B <= 0) return cudaSuccess;
    const int64_t m = B * sn;
    k_batched_finish<<<(unsigned)std::min<int64_t>(1184, (m + 255) / 256), 256, 0, s>>>(x, y, xhat, n, sn, B, ops, d_j,
                                                                                       done_b, conv, nc);
    k_batched_reset<<<(unsigned)((B + 255) / 256), 256, 0, s>>>(done_b, ndone, conv, nc, d_j, B);
    return cudaGetLastError();
}

// flag = 1 unless G row k + P == -G row k for every k < P (n columns, rows ld apart)
__global__ void k_check_pairs(const double *G, int64_t P, int64_t n, int64_t ld, int32_t *flag) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < P * n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = t / n, j = t % n;
        if (G[(k + P) * ld + j] != -G[k * ld + j]) *flag = 1;
    }
}

cudaError_t launch_check_pairs(const double *G, int64_t P, int64_t n, int64_t ld, int32_t *flag, cudaStream_t s) {
    if (P * n > 0) k_check_pairs<<<592, 256, 0, s>>>(G, P, n, ld, flag);
    return cudaGetLastError();
}

__global__ void k_batched_h(double *h, const double *mu, const double *g, double rho, int64_t p, int64_t sp,
                            int64_t B) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < B * sp && t % sp < p) h[t] = mu[t] + rho * g[t];
}

cudaError_t launch_batched_h(double *h, const double *mu, const double *g, double rho, int64_t p, int64_t sp,
                             int64_t B, cudaStream_t s) {
    const int64_t m = B * sp;
    if (m <= 0) return cudaSuccess;
    k_batched_h<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(h, mu, g, rho, p, sp, B);
    return cudaGetLastError();
}

__global__ void k_init_batched(double *x, double *y, double *xhat, const double *lb, const double *ub, int64_t n,
                               int64_t sn, double *mu, double *lam_prev, int64_t sp, int64_t B, int32_t *d_j,
                               int32_t *flag) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < B * sn) {
        const int64_t i = t % sn;
        const double x0 = i < n ? fmin(fmax(0.0, lb[i]), ub[i]) : 0.0;   // u_bar^0 = [0]_U
        x[t] = x0;
        y[t] = x0;
        xhat[t] = 0.0;
    }
    if (t < B * sp) {
        mu[t] = 0.0;
        lam_prev[t] = 0.0;
    }
    if (t == 0) {
        *d_j = 1;
        *flag = 0;
    }
}

cudaError_t launch_init_batched(double *x, double *y, double *xhat, const double *lb, const double *ub, int64_t n,
                                int64_t sn, double *mu, double *lam_prev, int64_t sp, int64_t B, int32_t *d_j,
                                int32_t *flag, cudaStream_t s) {
    const int64_t m = B * (sn > sp ? sn : sp);
    k_init_batched<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(x, y, xhat, lb, ub, n, sn, mu, lam_prev, sp, B,
                                                                d_j, flag);
    return cudaGetLastError();
}

}  // namespace dq
