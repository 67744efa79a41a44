// Byte-floor inner step for large dense QPs (SURVEY.md §8(a) "byte floor"; config 2).
//
// The two-pass step streams [Q;G] and G' = 8(n^2 + 2pn) bytes.  The method only needs
// 8(n(n+1)/2 + pn): Q is symmetric (Hessian) and G can be read once.  One streaming
// kernel (k_fused_stream) does both, then a small kernel (k_fused_epi) finishes the step.
//
// Data movement: every thread prefetches, with cp.async (LDGSTS), exactly the 16-byte pieces of
// the 4096-column row chunks it will itself consume, 7 chunks ahead (224 KB of ring per SM),
// into a private shared-memory ring -- the stream needs no barriers at all.  (Measured on B200:
// such a ring streams at ~7.2 TB/s, while cp.async.bulk (TMA) rings are bound by a per-copy
// cost: 3.7 TB/s with 8 KB copies, 6.6 TB/s with 16 KB copies.)  Thread t owns columns
// 2t, 2t+1 (+1024 k) of every chunk: their y values and column sums live in registers.
// 16 warps, 128 registers per thread.
//
//  * Q role (single CTAs): the upper triangle in tile columns of 4096, as the sequence
//    (J, r): J = 0..nt-1, r = 0..min(4096 (J+1), n)-1; row step (J, r) = columns
//    [max(4096 J, r), 4096 (J+1)) of row r.  Each element Q_rc (c >= r) is used twice: Q_rc y_c
//    into row r's dot (per-warp sums -> ws_rowp[J][warp][r]; no cross-warp sync) and Q_rc y_r into column c
//    (registers -> ws_col[cta][J - j0] when the CTA leaves tile column J).  The host cuts the
//    sequence into pieces of equal estimated time, max(bytes, per-step cost) summed.
//  * G role (CTA pairs = thread-block clusters of 2): rank c owns column block c
//    ([c W, (c+1) W)) of a range of G rows.  Per row: the block's partial dot -> the last warp to
//    post its partial (shared-memory counter) sends the CTA sum to every CTA of the cluster through distributed shared memory (st.async with mbarrier
//    complete_tx), adds the block partials in rank order and applies the pass-A epilogue (w_i =
//    [mu_i + rho r_i]_{K°}, incl. the fused DFOM step on the first inner step); all warps then
//    accumulate w_i G_i into register column sums from the row values they hold in registers
//    (the CTA's block of y sits in shared memory after a ring that is pure prefetch); the
//    first chunk of row i+1 is read and dotted before waiting for w_i, so the exchange hides
//    under the stream.
//  * k_fused_epi: grad_j = sum of the partials of column j in a fixed order (+ q_j), then the
//    pass-B epilogue (box projection, momentum, average).
// All sums are in a fixed order, so results are bitwise reproducible run to run (but not
// bitwise equal to the two-pass path: different summation order).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "duquad_internal.h"
#include "epilogue.cuh"

namespace dq {

namespace {

constexpr int kWarps = 16;
constexpr int kThreadsF = kWarps * 32;  // 4 warps per SMSP, 128 registers
constexpr int kChunk = 4096;            // columns per chunk (= Q tile width)
constexpr int kV = 4;                   // double2 per thread per chunk
constexpr int kSlots = 7;               // per-thread ring depth (chunks; 224 KB per CTA), Q role
// G role: a (kSlots - NCHG)-chunk ring + this CTA's block of y (NCHG chunks) in the same space
constexpr int kD = 8;                   // depth of the per-row buffers / barriers (G rows)
constexpr int kHdr = 3072;              // barriers + per-row buffers; header + ring = 227 KB
constexpr int kE_ = 16;                 // (= kE) per-row epilogue-operand buffers in the header
static_assert(128 + kD * 32 * 8 + kE_ * 5 * 8 <= kHdr, "header overflow");
static_assert(kThreadsF * kV * 2 == kChunk, "chunk = 512 threads x 8 doubles");

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t map_to_cta(uint32_t saddr, uint32_t cta) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(cta));
    return r;
}
// 8 bytes into another CTA's shared memory, completing 8 bytes of transaction count on its mbarrier:
// data and signal in one asynchronous operation, no fence.  (A remote mbarrier.arrive.release.cluster
// compiles to MEMBAR.ALL.GPU + ERRBAR -- microseconds per row.)
__device__ __forceinline__ void st_async_f64(uint32_t raddr, double v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr), "l"(
                     __double_as_longlong(v)),
                 "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ void cp16(uint32_t dst, const double *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// G rows' epilogue operands (g, mu, lambda_prev, cone, lam_hat) reach shared memory by cp.async,
// kEpiAhead rows ahead (DQ_EPI_ASYNC), instead of loads by thread 0 that stall warp 0 -- the warp
// every row's exchange waits for -- until they return (measured, DQ_TRACE_G: 20 % of warp 0's time)
#ifndef DQ_EPI_ASYNC
#define DQ_EPI_ASYNC 1
#endif
constexpr int kEpiAhead = 7;   // >= kSlotsG + 1: one ring group per row is the worst case (nch = 1)
constexpr int kE = kE_;        // per-row epilogue buffers: a slot is rewritten kE - kEpiAhead rows after its
                               // row, when every warp has long read it (a warp lags by at most one row)
static_assert(kEpiAhead + 2 <= kE, "per-row epilogue buffers in flight");
__device__ __forceinline__ void cp8s(double *smem, const double *gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp4s(void *smem, const uint32_t *gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
// the aligned 32-bit word holding the cone byte *c (decoded with the byte's offset in the word)
__device__ __forceinline__ uint32_t cone_word(const uint8_t *c) {
    return *reinterpret_cast<const uint32_t *>(reinterpret_cast<uintptr_t>(c) & ~(uintptr_t)3);
}

// column (relative to the chunk base) of element e (0..7) owned by thread t
__device__ __forceinline__ int own_col(int t, int e) { return (e >> 1) * 1024 + 2 * t + (e & 1); }

// fixed-tree sum of the 16 warp partials held by lanes 0..15
__device__ __forceinline__ double sum16(double v) {
    v += __shfl_xor_sync(0xffffffffu, v, 8);
    v += __shfl_xor_sync(0xffffffffu, v, 4);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    return v;
}

// w_i from r_i = G_i y + g_i: the pass-A epilogue value (epilogue.cuh, epi_a_store) without the
// store; `write` = this CTA commits mu / lambda (rank 0 of the pair only).
__device__ __forceinline__ double g_row_w(const PassAArgs &a, int64_t k, double s, const EpiA &e, const OuterA &o,
                                          bool write) {
    const double r = s + e.g;
    double m = e.mu;
    if (o.dual) {
        double lam;
        m = dfom_row(r, e.mu, e.lp, e.c, a.rho, a.step, a.project_dual, o.beta_out, lam);
        double lh = 0.0;
        if (o.lhat_w != 0.0) m = dual_average(e.lh, lam, m, o, lh);
        if (write) {
            a.lam_prev[k] = lam;
            a.mu[k] = m;
            if (o.lhat_w != 0.0) a.lam_hat[k] = lh;
        }
    }
    return a.rho > 0.0 ? proj_polar(m + a.rho * r, e.c) : m;
}

// Q tile column J: columns [a, b), rows 0..rows-1
struct Tile {
    int a, b, rows;
};
__device__ __forceinline__ Tile tile_of(const FusedArgs &f, int J) {
    Tile t;
    t.a = J * kChunk;
    t.b = t.a + kChunk < (int)f.ld ? t.a + kChunk : (int)f.ld;
    t.rows = t.b < (int)f.n ? t.b : (int)f.n;
    if (t.rows > (int)f.qb) t.rows = (int)f.qb;   // row-sharded: this rank's rows end at qb
    return t;
}

// NCHG: G chunks per column block (0: no G role in this launch -- Q only)
// Launched with a cluster dimension of 2 when there is a G role (pairs), 1 otherwise.
#ifdef DQ_TRACE_G   // instrumentation build only: cumulative per-role cycle counters, printed periodically
__device__ unsigned long long g_trg[8];   // G: wait, loop, epi-prefetch (warp 0), rows; Q: loop, steps
__device__ unsigned g_trlaunch;
#endif
#ifdef DQ_TRACE_ROLE   // instrumentation build only: per-CTA durations (globaltimer) of one launch
__device__ unsigned long long g_trd[2 * 160];
__device__ unsigned g_trrl;
#endif
template <int NCHG>
__global__ void __launch_bounds__(kThreadsF, 1) k_fused_stream(const FusedArgs f) {
    // PDL (epilogue.cuh): the Q role fills its ring with Q rows (never written by a solve) before
    // pdl_wait(); every other read and write of both roles comes after it
    constexpr int kSlotsG = kSlots - (NCHG > 0 ? NCHG : 1);
    extern __shared__ __align__(128) uint8_t fsm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int cta = blockIdx.x;
    // ---- shared memory: barriers + small per-row buffers (first 8 KB), then the ring
    uint64_t *xbar = reinterpret_cast<uint64_t *>(fsm);    // [kD] pair exchange (st.async bytes)
    double *xbuf = reinterpret_cast<double *>(fsm + 128);  // [kD][32] warp partials of a G row, rank-major
    double *epib = xbuf + kD * 32;                         // [kE][5] g, mu, lambda_prev, cone, lam_hat of the row
    const double2 *ring = reinterpret_cast<const double2 *>(fsm + kHdr) + tid;   // [kSlots][kV][512]
    const uint32_t ring_u32 = smem_u32(ring);
    auto slot_addr = [&](int s, int k) -> uint32_t { return ring_u32 + (uint32_t)((s * kV + k) * kThreadsF) * 16; };

#ifdef DQ_TRACE_ROLE
    unsigned long long trr_t0 = 0;
    unsigned trr_l = 0;
    if (tid == 0) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(trr_t0));
        trr_l = *(volatile unsigned *)&g_trrl;
    }
#endif
#ifdef DQ_TRACE_G
    if (cta == 0 && tid == 0) {
        const unsigned c = atomicAdd(&g_trlaunch, 1u);
        if (c % 4000 == 3999)
            printf("TRACE_G launches %u G: wait %llu loop %llu epipf %llu rows %llu | Q: loop %llu steps %llu\n", c + 1,
                   g_trg[0], g_trg[1], g_trg[2], g_trg[3], g_trg[4], g_trg[5]);
    }
    unsigned long long tr_wait = 0, tr_pf = 0, tr_t0 = clock64();
#endif
    if (tid == 0) {
        for (int s = 0; s < kD; ++s) mbar_init(&xbar[s], 1);   // warp 0's expect_tx + 32 x 8 bytes of st.async
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    cluster_sync_all();

    if (!(NCHG == 0 || cta < f.nq_ctas)) {
        pdl_wait();
        pdl_trigger();
        if (f.a.skip && *f.a.skip) return;   // eps_in mode: converged (uniform over the grid)
    }
    if (NCHG == 0 || cta < f.nq_ctas) {
        // ================================ Q role: triangle row steps (J, r) of this piece
        const FusedPiece pc = f.pieces[cta];
        int nsteps = 0;   // row steps of this piece
        for (int J = pc.j0; J <= pc.j1 && J < f.nt; ++J) {
            const Tile tj = tile_of(f, J);
            const int rb = J == pc.j0 ? pc.r0 : (int)f.qa, re = J == pc.j1 ? pc.r1 : tj.rows;
            nsteps += re > rb ? re - rb : 0;
        }
        const int c2t = 2 * tid;
        // prefetch cursor: kSlots steps ahead of the consumer, same sequence
        int p_left = nsteps, pJ = pc.j0, pr = pc.r0, ps = 0;
        Tile pt = tile_of(f, pJ);
        bool p_rag = pt.b - pt.a < kChunk;
        const double *prow = f.Q + (int64_t)(pr - f.qa) * f.ld + pt.a + c2t;   // f.Q row 0 = global row qa
        auto issue = [&]() {
            if (p_left > 0) {
                if (pr < pt.a && !p_rag) {   // off-diagonal full row step
#pragma unroll
                    for (int k = 0; k < kV; ++k) cp16(slot_addr(ps, k), prow + 1024 * k);
                } else {                     // diagonal (from column r) / ragged tile
                    const int st = pr > pt.a ? (pr & ~1) : pt.a;
#pragma unroll
                    for (int k = 0; k < kV; ++k) {
                        const int c = pt.a + c2t + 1024 * k;
                        if (c >= st && c < pt.b) cp16(slot_addr(ps, k), prow + 1024 * k);
                    }
                }
                --p_left;
                prow += f.ld;
                if (++pr == pt.rows) {
                    ++pJ;
                    pr = (int)f.qa;
                    pt = tile_of(f, pJ < f.nt ? pJ : 0);
                    p_rag = pt.b - pt.a < kChunk;
                    prow = f.Q + pt.a + c2t;
                }
            }
            cp_commit();
            if (++ps == kSlots) ps = 0;
        };
        for (int t = 0; t < kSlots; ++t) issue();   // Q rows: matrix data, before the dependency wait
        pdl_wait();
        pdl_trigger();
        if (f.a.skip && *f.a.skip) {   // eps_in mode: converged (uniform over the grid)
            cp_wait<0>();
            return;
        }
        int cs = 0;
        auto load_q = [&](double *q) {
#pragma unroll
            for (int k = 0; k < kV; ++k) {
                const double2 v = ring[(cs * kV + k) * kThreadsF];
                q[2 * k] = v.x;
                q[2 * k + 1] = v.y;
            }
            if (++cs == kSlots) cs = 0;
        };
        for (int J = pc.j0; J <= pc.j1 && J < f.nt; ++J) {
            const Tile t = tile_of(f, J);
            const int rb = J == pc.j0 ? pc.r0 : (int)f.qa, re = J == pc.j1 ? pc.r1 : t.rows;
            if (re <= rb) continue;
            const bool rag = t.b - t.a < kChunk;
            const int cb = t.a + c2t;   // column of element e: cb + (e >> 1) * 1024 + (e & 1)
            double yv[8], acc[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int c = cb + (e >> 1) * 1024 + (e & 1);
                yv[e] = c < t.b ? f.y[c] : 0.0;
                acc[e] = 0.0;
            }
            double *rowp = f.ws_rowp + ((int64_t)J * kWarps + warp) * f.ld;   // this warp's row partials
            // y_r for 32 rows at a time, one per lane (broadcast by shuffle)
            int ybase = rb;
            double ycache = rb + lane < t.rows ? f.y[rb + lane] : 0.0;
            int r = rb;
            // the row-pair butterfly is software-pipelined: pair i's sums are reduced after pair i+1's
            // FMAs, so its dependent shuffle chain overlaps independent work (same sums, same order)
            double p0 = 0.0, p1 = 0.0;
            int pr_ = -1;
            auto finish_pair = [&](double u0, double u1, int rr) {
                double mine = (lane & 16) ? u1 : u0;
                mine += __shfl_xor_sync(0xffffffffu, (lane & 16) ? u0 : u1, 16);
                mine += __shfl_xor_sync(0xffffffffu, mine, 8);
                mine += __shfl_xor_sync(0xffffffffu, mine, 4);
                mine += __shfl_xor_sync(0xffffffffu, mine, 2);
                mine += __shfl_xor_sync(0xffffffffu, mine, 1);
                if ((lane & 15) == 0) rowp[rr + (lane >> 4)] = mine;
            };
            for (; r + 1 < re; r += 2) {   // two row steps per iteration (independent chains)
                if (r + 1 - ybase >= 32) {
                    ybase = r;
                    ycache = r + lane < t.rows ? f.y[r + lane] : 0.0;
                }
                const double y0 = __shfl_sync(0xffffffffu, ycache, r - ybase);
                const double y1 = __shfl_sync(0xffffffffu, ycache, r + 1 - ybase);
                cp_wait<kSlots - 2>();
                double q0[8], q1[8];
                load_q(q0);
                load_q(q1);
                issue();
                issue();
                double a0 = 0.0, b0 = 0.0, a1 = 0.0, b1 = 0.0;
                if (r + 1 < t.a && !rag) {   // both rows above the diagonal tile: no masks
#pragma unroll
                    for (int e = 0; e < 8; e += 2) {
                        a0 = fma(q0[e], yv[e], a0);
                        b0 = fma(q0[e + 1], yv[e + 1], b0);
                        a1 = fma(q1[e], yv[e], a1);
                        b1 = fma(q1[e + 1], yv[e + 1], b1);
                        acc[e] = fma(q0[e], y0, acc[e]);
                        acc[e + 1] = fma(q0[e + 1], y0, acc[e + 1]);
                        acc[e] = fma(q1[e], y1, acc[e]);
                        acc[e + 1] = fma(q1[e + 1], y1, acc[e + 1]);
                    }
                } else if (!rag) {
                    // diagonal tile (40 % of the row steps at config 2): per 1024-column quarter k the
                    // warp's 64 columns [lo, lo + 64) are all right of both rows' diagonals, all left,
                    // or straddle -- a warp-uniform choice, so only the straddling quarter pays the
                    // per-element masks.  Same accumulators and order as the masked loop (a masked
                    // term adds an exact zero), so the sums are unchanged.
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int lo = t.a + 1024 * k + 64 * warp;
                        if (lo > r + 1) {
#pragma unroll
                            for (int e = 2 * k; e < 2 * k + 2; ++e) {
                                if (e & 1) {
                                    b0 = fma(q0[e], yv[e], b0);
                                    b1 = fma(q1[e], yv[e], b1);
                                } else {
                                    a0 = fma(q0[e], yv[e], a0);
                                    a1 = fma(q1[e], yv[e], a1);
                                }
                                acc[e] = fma(q0[e], y0, acc[e]);
                                acc[e] = fma(q1[e], y1, acc[e]);
                            }
                        } else if (lo + 63 >= r) {
#pragma unroll
                            for (int e = 2 * k; e < 2 * k + 2; ++e) {
                                const int c = cb + (e >> 1) * 1024 + (e & 1);
                                const double d0 = c >= r ? q0[e] : 0.0, d1 = c >= r + 1 ? q1[e] : 0.0;
                                if (e & 1) {
                                    b0 = fma(d0, yv[e], b0);
                                    b1 = fma(d1, yv[e], b1);
                                } else {
                                    a0 = fma(d0, yv[e], a0);
                                    a1 = fma(d1, yv[e], a1);
                                }
                                acc[e] = fma(c > r ? d0 : 0.0, y0, acc[e]);
                                acc[e] = fma(c > r + 1 ? d1 : 0.0, y1, acc[e]);
                            }
                        }
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const int c = cb + (e >> 1) * 1024 + (e & 1);
                        const bool in = c < t.b;
                        const double d0 = (in && c >= r) ? q0[e] : 0.0, d1 = (in && c >= r + 1) ? q1[e] : 0.0;
                        if (e & 1) {
                            b0 = fma(d0, yv[e], b0);
                            b1 = fma(d1, yv[e], b1);
                        } else {
                            a0 = fma(d0, yv[e], a0);
                            a1 = fma(d1, yv[e], a1);
                        }
                        acc[e] = fma(c > r ? d0 : 0.0, y0, acc[e]);
                        acc[e] = fma(c > r + 1 ? d1 : 0.0, y1, acc[e]);
                    }
                }
                // both row sums with one butterfly (lanes < 16 reduce row r, lanes >= 16 row r + 1),
                // the previous pair's first
                if (pr_ >= 0) finish_pair(p0, p1, pr_);
                p0 = a0 + b0;
                p1 = a1 + b1;
                pr_ = r;
            }
            if (pr_ >= 0) finish_pair(p0, p1, pr_);
            if (r < re) {   // last row of the segment
                if (r - ybase >= 32) {
                    ybase = r;
                    ycache = r + lane < t.rows ? f.y[r + lane] : 0.0;
                }
                const double y0 = __shfl_sync(0xffffffffu, ycache, r - ybase);
                cp_wait<kSlots - 1>();
                double q0[8];
                load_q(q0);
                issue();
                double a0 = 0.0;
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const int c = cb + (e >> 1) * 1024 + (e & 1);
                    const double d0 = (c < t.b && c >= r) ? q0[e] : 0.0;
                    a0 = fma(d0, yv[e], a0);
                    acc[e] = fma(c > r ? d0 : 0.0, y0, acc[e]);
                }
                a0 = warp_sum(a0);
                if (lane == 0) rowp[r] = a0;
            }
            // column sums of this tile column -> ws_col[cta][J - j0]
            double *dst = f.ws_col + ((int64_t)cta * f.cslots + (J - pc.j0)) * kChunk + c2t;
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (cb + (e >> 1) * 1024 + (e & 1) < t.b) dst[(e >> 1) * 1024 + (e & 1)] = acc[e];
        }
        cp_wait<0>();
#ifdef DQ_TRACE_G
        if (tid == 0) {
            atomicAdd(&g_trg[4], clock64() - tr_t0);
            atomicAdd(&g_trg[5], (unsigned long long)nsteps);
        }
#endif
    } else if constexpr (NCHG > 0) {
        // ================================ G role: pair gi owns rows [g0, g1); this CTA block `rank`
        const uint32_t rank = cluster_rank();
        const int a = (int)rank * f.W, b = rank == 1 ? (int)f.ld : f.W;
        const int nch = (b - a + kChunk - 1) / kChunk;
        const bool ragged = ((b - a) % kChunk) != 0;
        const int gi = (cta - f.nq_ctas) >> 1;
        const int64_t g0 = f.p * gi / f.ng, g1 = f.p * (gi + 1) / f.ng;
        const int nr = (int)(g1 - g0);
        // The G role keeps this CTA's block of y in shared memory (after a kSlotsG-slot ring) and
        // row values in registers between their dot and their w G, so every ring slot is refilled
        // as soon as it is read (kSlotsG chunks in flight).  Half-row lag: the first chunk of row
        // it+1 is read and dotted before waiting for w_it, which hides the cluster exchange.
        double2 *ysm = reinterpret_cast<double2 *>(fsm + kHdr + kSlotsG * kChunk * 8) + tid;   // [NCHG][kV][512]
        for (int m = 0; m < NCHG; ++m)
#pragma unroll
            for (int k = 0; k < kV; ++k) {
                const int c = a + m * kChunk + 2 * tid + 1024 * k;
                ysm[(m * kV + k) * kThreadsF] = (m < nch && c < b) ? *reinterpret_cast<const double2 *>(f.y + c)
                                                                    : make_double2(0.0, 0.0);
            }
        // the G loop is compiled twice: RAG (the rank's block ends in a partial chunk: per-element
        // masks on that chunk) and not (config 2: no masks at all in the hot loop)
        auto g_body = [&](auto rag_c) {
            constexpr bool RAG = decltype(rag_c)::value;
            int p_it = 0, p_m = 0, ps = 0;   // prefetch cursor
            auto issue = [&]() {
                if (p_it < nr) {
                    const double *row = f.G + (g0 + p_it) * f.ld;
    #pragma unroll
                    for (int k = 0; k < kV; ++k) {
                        const int c = a + p_m * kChunk + 2 * tid + 1024 * k;
                        if (!RAG || c < b) cp16(slot_addr(ps, k), row + c);
                    }
                    if (++p_m == nch) {
                        p_m = 0;
                        ++p_it;
                    }
                }
                cp_commit();
                if (++ps == kSlotsG) ps = 0;
            };
            for (int t = 0; t < kSlotsG; ++t) issue();
            double acc[NCHG][8];
    #pragma unroll
            for (int m = 0; m < NCHG; ++m)
    #pragma unroll
                for (int e = 0; e < 8; ++e) acc[m][e] = 0.0;
            int cs = 0;
            // read chunk m of the next row from the ring into v (slot refilled at once); its dot with y
            auto take = [&](int m, double *v, double part) -> double {
                cp_wait<kSlotsG - 1>();
                const bool rg = RAG && m == nch - 1;
    #pragma unroll
                for (int k = 0; k < kV; ++k) {
                    double2 q = ring[(cs * kV + k) * kThreadsF];
                    if (rg && a + m * kChunk + 2 * tid + 1024 * k >= b) q = make_double2(0.0, 0.0);   // not loaded
                    v[2 * k] = q.x;
                    v[2 * k + 1] = q.y;
                }
                issue();
                if (++cs == kSlotsG) cs = 0;
    #pragma unroll
                for (int k = 0; k < kV; ++k) {
                    const double2 yk = ysm[(m * kV + k) * kThreadsF];
                    part = fma(v[2 * k], yk.x, part);
                    part = fma(v[2 * k + 1], yk.y, part);
                }
                return part;
            };
            // Row finishing: the LAST warp to post its partial (shared-memory counter) forms the CTA sum
            // of the 16 warp partials (fixed tree) and sends it to every CTA of the cluster with
            // st.async (completing the rows' exchange barrier); every warp then forms w itself (row_w).
            // The epilogue operands of row it are prefetched into shared memory two rows ahead.
            const OuterA o = outer_a(f.a, MODE_SOLVE);
            const uint32_t xb_r = map_to_cta(smem_u32(xbuf), (uint32_t)(lane & 1));
            const uint32_t xm_r = map_to_cta(smem_u32(xbar), (uint32_t)(lane & 1));
            auto prefetch_epi = [&](int it) {
#ifdef DQ_TRACE_G
                const unsigned long long t0_ = clock64();
#endif
                if (tid == 0 && it < nr) {
                    const EpiA e = epi_a_load(f.a, MODE_SOLVE, f.a.nq + g0 + it, o);
                    double *eb = epib + (it % kE) * 5;
                    eb[0] = e.g;
                    eb[1] = e.mu;
                    eb[2] = e.lp;
                    *reinterpret_cast<uint32_t *>(eb + 3) = cone_word(f.a.cone + g0 + it);
                    eb[4] = e.lh;
                }
#ifdef DQ_TRACE_G
                __syncwarp();
                tr_pf += clock64() - t0_;
#endif
            };
#if DQ_EPI_ASYNC
            // the same operands with cp.async (thread 0), kEpiAhead rows ahead: nothing waits for
            // them here.  They join thread 0's next ring group; post(it) -- warp 0's arrive that
            // publishes row it's buffer -- comes after a take() whose cp_wait<kSlotsG - 1> retired
            // every group at least kSlotsG - 1 newer ones old, i.e. (one or more groups per row) the
            // group of row it's copies, issued kEpiAhead >= kSlotsG + 1 rows earlier.
            auto prefetch_epi_async = [&](int it) {
                if (tid == 0 && it < nr) {
                    const int64_t k = g0 + it;
                    double *eb = epib + (it % kE) * 5;
                    cp8s(eb + 0, f.a.g + k);
                    cp8s(eb + 1, f.a.mu + k);
                    if (o.dual) cp8s(eb + 2, f.a.lam_prev + k);
                    if (o.lhat_w != 0.0) cp8s(eb + 4, f.a.lam_hat + k);
                    cp4s(eb + 3, reinterpret_cast<const uint32_t *>(reinterpret_cast<uintptr_t>(f.a.cone + k) &
                                                                    ~(uintptr_t)3));
                }
            };
#endif
            // Row finishing without any intra-CTA hand-off: every warp sends its partial of the row to
            // both CTAs of the pair (st.async into xbuf[d][rank * 16 + warp], completing 8 bytes of the
            // row's exchange barrier there; warp 0 arms the barrier for all 32 partials), then waits for
            // the barrier and forms w itself: fixed butterfly over the 32 partials, pass-A epilogue.
            auto post = [&](int it, double part) {
                part = warp_sum(part);
                const int d = it % kD;
                if (lane < 2)   // lane c -> CTA c of the pair
                    st_async_f64(xb_r + (uint32_t)(d * 32 + (int)rank * kWarps + warp) * 8, part,
                                 xm_r + (uint32_t)d * 8);
                if (warp == 0 && lane == 0) mbar_arrive_expect_tx(&xbar[d], 2u * kWarps * 8u);
            };
            auto row_w = [&](int it) -> double {
                const int d = it % kD;
#ifdef DQ_TRACE_G
                const unsigned long long tw_ = clock64();
                mbar_wait(&xbar[d], (uint32_t)((it / kD) & 1));
                tr_wait += clock64() - tw_;
#else
                mbar_wait(&xbar[d], (uint32_t)((it / kD) & 1));
#endif
                double s_row = xbuf[d * 32 + lane];
                s_row += __shfl_xor_sync(0xffffffffu, s_row, 16);
                s_row += __shfl_xor_sync(0xffffffffu, s_row, 8);
                s_row += __shfl_xor_sync(0xffffffffu, s_row, 4);
                s_row += __shfl_xor_sync(0xffffffffu, s_row, 2);
                s_row += __shfl_xor_sync(0xffffffffu, s_row, 1);
                const double *eb = epib + (it % kE) * 5;
                EpiA e;
                e.g = eb[0];
                e.mu = eb[1];
                e.lp = eb[2];
                e.c = (uint8_t)(*reinterpret_cast<const uint32_t *>(eb + 3) >>
                                (8 * (reinterpret_cast<uintptr_t>(f.a.cone + g0 + it) & 3)));
                e.lh = eb[4];
                return g_row_w(f.a, g0 + it, s_row, e, o, rank == 0 && warp == 0 && lane == 0);
            };
#if DQ_EPI_ASYNC
            for (int r = 0; r < kEpiAhead; ++r) prefetch_epi(r);
#else
            prefetch_epi(0);
            prefetch_epi(1);
#endif
            double hold[NCHG][8];   // the current row's values (chunks 0..nch-1)
            if (nr > 0) {
                double part = 0.0;
    #pragma unroll
                for (int m = 0; m < NCHG; ++m)
                    if (m < nch) part = take(m, hold[m], part);
                post(0, part);
            }
            for (int it = 0; it < nr; ++it) {
                const bool nxt = it + 1 < nr;
#if DQ_EPI_ASYNC
                prefetch_epi_async(it + kEpiAhead);
#else
                prefetch_epi(it + 2);
#endif
                double next0[8];
                double part = 0.0;
                if (nxt) part = take(0, next0, part);                    // row it+1, chunk 0
                const double w = row_w(it);
    #pragma unroll
                for (int m = 0; m < NCHG; ++m)                              // w G of row it
    #pragma unroll
                    for (int e = 0; e < 8; ++e) acc[m][e] = fma(w, hold[m][e], acc[m][e]);
                if (nxt) {
    #pragma unroll
                    for (int e = 0; e < 8; ++e) hold[0][e] = next0[e];
    #pragma unroll
                    for (int m = 1; m < NCHG; ++m)
                        if (m < nch) part = take(m, hold[m], part);         // row it+1, chunks 1..
                    post(it + 1, part);
                }
            }
            cp_wait<0>();
#ifdef DQ_TRACE_G
            if (lane == 0) {
                atomicAdd(&g_trg[0], tr_wait);
                atomicAdd(&g_trg[1], clock64() - tr_t0);
                if (warp == 0) atomicAdd(&g_trg[2], tr_pf);
                if (warp == 0) atomicAdd(&g_trg[3], (unsigned long long)nr);
            }
#endif
            double *pt = f.ws_g + (int64_t)gi * f.ld;
    #pragma unroll
            for (int m = 0; m < NCHG; ++m)
    #pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const int c = a + m * kChunk + own_col(tid, e);
                    if (m < nch && c < b) pt[c] = acc[m][e];
                }
        };
        if (ragged)
            g_body(std::true_type{});
        else
            g_body(std::false_type{});
    }
    __syncthreads();
#ifdef DQ_TRACE_ROLE
    if (tid == 0) {
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (trr_l == 4050 && cta < 160) {   // an inner step without the DFOM step
            g_trd[2 * cta] = trr_t0;
            g_trd[2 * cta + 1] = t1;
        }
        __threadfence();
        if (cta == 0) atomicAdd(&g_trrl, 1u);   // launch counter (CTA 0 of each launch)
    }
#endif
    cluster_sync_all();   // no CTA leaves while its partner may still write its shared memory
}

// grad_j = sum of the partials of column j (fixed order) + q_j: the pass-B epilogue.
// Block: 32 columns x 8 slices; slice s sums list entries s, s + 8, ...; the 8 slice sums are
// added in slice order.  List of column j (tile column Jc = j / 4096):
//   ws_rowp[J][w][j] for J = Jc..nt-1, w = 0..15, then ws_col[c][Jc - j0(c)][j - 4096 Jc] for the Q CTAs c
//   with rows in tile column Jc, then ws_g[g][j] for the G pairs g.
constexpr int kEpiCols = 32, kEpiSlices = 8;
__global__ void __launch_bounds__(kEpiCols *kEpiSlices) k_fused_epi(const PassBArgs bl, const PassBArgs bs,
                                                                    const FusedArgs f) {
    pdl_wait();   // every read here depends on the stream kernel (PDL, epilogue.cuh)
    pdl_trigger();
    if (bl.skip && *bl.skip) return;
    __shared__ double part[kEpiSlices][kEpiCols];
    const int cl = threadIdx.x % kEpiCols, sl = threadIdx.x / kEpiCols;
    const int64_t j = (int64_t)blockIdx.x * kEpiCols + cl;
    const double avg_w = avg_weight(bl, MODE_SOLVE);
    const bool partial = f.partial != nullptr;   // row-sharded: the rank's partial n-vector, no epilogue
    const int64_t nr = partial ? f.n : bl.nrows;
    EpiB e{};
    if (!partial && sl == 0 && j < nr) e = epi_b_load(bl, MODE_SOLVE, j, avg_w);   // overlaps the partial loads
    double s = 0.0;
    if (j < nr) {
        const int Jc = (int)(j / kChunk);
        const int nrow = (j >= f.qa && j < f.qb) ? (f.nt - Jc) * kWarps : 0;   // row dots: this rank's rows
        const int lo = f.qlo[Jc], nqc = f.qhi[Jc] - f.qlo[Jc];
        const int64_t jr = j - (int64_t)Jc * kChunk;
        const int len = nrow + nqc + f.ng;
        auto at = [&](int t) -> const double * {
            if (t < nrow) return f.ws_rowp + ((int64_t)Jc * kWarps + t) * f.ld + j;
            if (t < nrow + nqc) {
                const int c = lo + (t - nrow);
                return f.ws_col + ((int64_t)c * f.cslots + (Jc - f.pieces[c].j0)) * kChunk + jr;
            }
            return f.ws_g + (int64_t)(t - nrow - nqc) * f.ld + j;
        };
        // sixteen list entries in flight per thread, the ragged last batch included (predicated,
        // zeros past the end: s + 0 = s), added in list order (the same sum, bit for bit)
        constexpr int U = 16;
        for (int t = sl; t < len; t += U * kEpiSlices) {
            double v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = t + u * kEpiSlices < len ? __ldcg(at(t + u * kEpiSlices)) : 0.0;
#pragma unroll
            for (int u = 0; u < U; ++u) s += v[u];
        }
    }
    part[sl][cl] = s;
    __syncthreads();
    if (sl == 0 && j < nr) {
        double t = part[0][cl];
#pragma unroll
        for (int q = 1; q < kEpiSlices; ++q) t += part[q][cl];
        if (partial) {
            f.partial[j] = t;
            return;
        }
        e.qy = t;
        epi_b_store(bs, MODE_SOLVE, j, 0.0, e, avg_w);
    }
}

// Row-sharded byte floor, after the reduce-scatter of the ranks' partial vectors: grad_j = sum_j + q_j
// and the pass-B epilogue on this rank's rows (the arithmetic of k_fused_epi's last step).
__global__ void k_slice_epi(const PassBArgs bl, const PassBArgs bs, const double *sum) {
    if (bl.skip && *bl.skip) return;
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= bl.nrows) return;
    const double avg_w = avg_weight(bl, MODE_SOLVE);
    EpiB e = epi_b_load(bl, MODE_SOLVE, j, avg_w);
    e.qy = sum[j];
    epi_b_store(bs, MODE_SOLVE, j, 0.0, e, avg_w);
}

__global__ void k_vec_add(double *dst, const double *src, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] += src[i];
}

#ifdef DQ_TRACE_ROLE
}  // namespace
}  // namespace dq
// instrumentation builds only: start / end globaltimer of every CTA of the recorded launch
extern "C" int duquad_debug_role_trace(unsigned long long *out, int n) {
    if (n > 2 * 160) n = 2 * 160;
    return (int)cudaMemcpyFromSymbol(out, dq::g_trd, n * sizeof(unsigned long long));
}
namespace dq {
namespace {
#endif
template <int NCHG>
cudaError_t launch_t(const FusedArgs &f, cudaStream_t s) {
    return launch_ex(k_fused_stream<NCHG>, f.nb, kThreadsF, f.smem, s, f.pdl, NCHG > 0 ? 2 : 1, f);
}

template <int NCHG>
cudaError_t configure_t(size_t smem) {
    cudaError_t e = cudaFuncSetAttribute(k_fused_stream<NCHG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e) return e;
    cudaFuncAttributes fa;
    if ((e = cudaFuncGetAttributes(&fa, k_fused_stream<NCHG>))) return e;
    if (fa.maxThreadsPerBlock < kThreadsF) {
        fprintf(stderr, "k_fused_stream<%d>: %d regs, maxThreadsPerBlock %d, local %zu\n", NCHG, fa.numRegs,
                fa.maxThreadsPerBlock, fa.localSizeBytes);
        return cudaErrorInvalidConfiguration;
    }
    return cudaSuccess;
}

}  // namespace

int fused_block_width(int64_t ld, int cg) { return (int)((ld + 32 * cg - 1) / (32 * cg) * 32); }
int fused_nchg(int64_t ld, int cg) { return (fused_block_width(ld, cg) + kChunk - 1) / kChunk; }
int fused_tiles(int64_t ld) { return (int)((ld + kChunk - 1) / kChunk); }
size_t fused_smem_bytes() { return kHdr + (size_t)kSlots * kChunk * 8; }
static_assert(kD * 8 <= 128 && 128 + kD * (32 + 5) * 8 <= kHdr, "header layout");
bool fused_supported(int64_t n, int64_t ld, size_t smem_optin) {
    int64_t nmin = 4096;   // below, the two-pass path is faster (tuning: DUQUAD_FUSED_NMIN)
    if (const char *ov = std::getenv("DUQUAD_FUSED_NMIN")) nmin = std::atoll(ov);
    return n >= nmin && fused_nchg(ld, 2) <= 2 && fused_tiles(ld) <= kFusedMaxTiles && fused_smem_bytes() <= smem_optin;
}

// Clusters of `cg` CTAs of the stream kernel that can be resident at once (0 on error).
int fused_max_clusters(int nchg, int cg, size_t smem) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cg * 256);
    cfg.blockDim = dim3(kThreadsF);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cg;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e;
    switch (nchg) {
        case 0: e = cudaOccupancyMaxActiveClusters(&n, k_fused_stream<0>, &cfg); break;
        case 1: e = cudaOccupancyMaxActiveClusters(&n, k_fused_stream<1>, &cfg); break;
        case 2: e = cudaOccupancyMaxActiveClusters(&n, k_fused_stream<2>, &cfg); break;
        default: return 0;
    }
    return e == cudaSuccess ? n : 0;
}

// Cut of the Q triangle sequence (J, r) into nq pieces of equal estimated time: a row step costs
// max(bytes, row_cost) (the per-step instruction cost dominates short steps near the diagonal);
// a step of a diagonal tile (masks on the straddling quarter, two rows of unequal length per pair)
// costs diag_fac * row_cost + diag_slope * bytes (fit to per-CTA end times of config 2,
// profiles/r02_role_trace3.txt: 1.145 and 0.0746).  qlo / qhi: the pieces with rows in each tile
// column; returns the most tile columns a piece spans.
int fused_partition(int64_t n, int64_t ld, int nq, double row_cost, double diag_fac, double diag_slope,
                    std::vector<FusedPiece> &pieces, int32_t *qlo, int32_t *qhi, int64_t qa, int64_t qb) {
    const int nt = fused_tiles(ld);
    // rows of tile column J in this rank's row range [qa, qb) (single GPU: [0, n)): [qa, rows(J))
    auto rows = [&](int J) -> int64_t {
        return std::min<int64_t>(std::min<int64_t>(std::min<int64_t>((int64_t)(J + 1) * kChunk, ld), n), qb);
    };
    auto cost = [&](int J, int64_t r) -> double {
        const int64_t a = (int64_t)J * kChunk, b = std::min<int64_t>(a + kChunk, ld);
        const int64_t st = r > a ? (r & ~1LL) : a;
        const double bytes = 8.0 * (double)(b - st);
        return r >= a ? diag_fac * row_cost + diag_slope * bytes : std::max(bytes, row_cost);
    };
    double total = 0.0;
    for (int J = 0; J < nt; ++J)
        for (int64_t r = qa; r < rows(J); ++r) total += cost(J, r);
    pieces.assign(nq, FusedPiece{0, 0, 0, 0});
    int J = 0;
    int64_t r = qa;
    double acc = 0.0;
    auto norm = [&]() {   // (J, r) past the end of tile column J -> next
        while (J < nt && r >= rows(J)) {
            ++J;
            r = qa;
        }
    };
    for (int c = 0; c < nq; ++c) {
        norm();
        pieces[c].j0 = J < nt ? J : nt - 1;
        pieces[c].r0 = J < nt ? (int32_t)r : (int32_t)rows(nt - 1);
        const double target = total * (c + 1) / nq;
        while (J < nt && (c == nq - 1 || acc + 0.5 * cost(J, r) < target)) {
            acc += cost(J, r);
            ++r;
            norm();
        }
        // exclusive end (j1, r1): r1 may equal rows(j1) only for the very end of the sequence
        if (J < nt) {
            pieces[c].j1 = J;
            pieces[c].r1 = (int32_t)r;
        } else {
            pieces[c].j1 = nt - 1;
            pieces[c].r1 = (int32_t)rows(nt - 1);
        }
    }
    int span = 1;
    for (int b = 0; b < kFusedMaxTiles; ++b) {
        qlo[b] = nq;
        qhi[b] = 0;
    }
    for (int c = 0; c < nq; ++c) {
        const FusedPiece &p = pieces[c];
        for (int b = p.j0; b <= p.j1 && b < nt; ++b) {
            const int64_t r0 = b == p.j0 ? p.r0 : qa;
            const int64_t r1 = b == p.j1 ? p.r1 : rows(b);
            if (r1 > r0) {
                qlo[b] = std::min(qlo[b], c);
                qhi[b] = std::max(qhi[b], c + 1);
                span = std::max(span, b - p.j0 + 1);
            }
        }
    }
    for (int b = 0; b < kFusedMaxTiles; ++b)
        if (qhi[b] <= qlo[b]) qlo[b] = qhi[b] = 0;
    return span;
}

cudaError_t configure_fused_kernels(int nchg, size_t smem) {
    cudaError_t e = configure_t<0>(smem);
    if (e) return e;
    switch (nchg) {
        case 0: return cudaSuccess;
        case 1: return configure_t<1>(smem);
        case 2: return configure_t<2>(smem);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_fused_stream(const FusedArgs &f, cudaStream_t s) {
    if (f.nq_ctas == f.nb) return launch_t<0>(f, s);
    switch (f.nchg) {
        case 1: return launch_t<1>(f, s);
        case 2: return launch_t<2>(f, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_slice_epi(const PassBArgs &bl, const PassBArgs &bs, const double *sum, cudaStream_t s) {
    if (bl.nrows > 0) k_slice_epi<<<(unsigned)((bl.nrows + 255) / 256), 256, 0, s>>>(bl, bs, sum);
    return cudaGetLastError();
}

cudaError_t launch_vec_add(double *dst, const double *src, int64_t n, cudaStream_t s) {
    if (n > 0) k_vec_add<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(dst, src, n);
    return cudaGetLastError();
}

cudaError_t launch_fused_epi(const PassBArgs &bl, const PassBArgs &bs, const FusedArgs &f, cudaStream_t s) {
    const int grid = (int)(((f.partial ? f.n : bl.nrows) + kEpiCols - 1) / kEpiCols);
    if (grid <= 0) return cudaSuccess;
    return launch_ex(k_fused_epi, grid, kEpiCols * kEpiSlices, 0, s, f.pdl, 0, bl, bs, f);
}

}  // namespace dq
