// Byte-floor inner step for large dense QPs (SURVEY.md §8(a) "byte floor"; config 2).
//
// The two-pass step streams [Q;G] and G' = 8(n^2 + 2pn) bytes.  The method only needs
// 8(n(n+1)/2 + pn): Q is symmetric (Hessian) and G can be read once.  One streaming
// kernel (k_fused_stream) does both, then a small kernel (k_fused_epi) finishes the step:
//
//  * Q role (single CTAs): the upper triangle, row by row, in 2048-column chunks moved by TMA
//    bulk copies (cp.async.bulk + mbarrier ring) into shared memory; y lives in shared memory.
//    Each element Q_ij (j >= i) is used twice: Q_ij y_j into row i's dot, Q_ij y_i into column j.
//    Column sums accumulate in registers (thread t owns 4 columns of every chunk); row dots are
//    warp-reduced per row and parked in shared memory.  Rows are assigned in pairs (i, n-1-i),
//    so every Q CTA streams the same number of bytes.
//  * G role (CTA pairs = thread-block clusters of 2 on 2 SMs): each CTA owns one column half.
//    Per G row: partial dot with y (the CTA's half of y is held in registers), CTA reduction,
//    exchange of the two half sums through distributed shared memory (st.shared::cluster +
//    remote mbarrier arrive), then r = G_i y + g_i -> w_i = [mu_i + rho r]_{K°} (the pass-A
//    epilogue incl. the fused DFOM step) and, with the row still in shared memory,
//    t += w_i G_i into register column accumulators.  G is read from HBM once.
//  * Every CTA writes its column sums to a workspace PT[col][cta] (L2-resident, 19 MB at
//    config 2); k_fused_epi sums the 148 partials of a column in a fixed order and applies the
//    pass-B epilogue (grad = Qy + t + q, box projection, momentum, average).
// All sums are in a fixed order, so results are bitwise reproducible (but not bitwise equal to
// the two-pass path: different summation order; parity with the oracle is ~1e-15).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "duquad_internal.h"
#include "epilogue.cuh"

namespace dq {

namespace {

constexpr int kCons = 512;              // threads (16 warps); warp 15 lane 0 also issues TMA
constexpr int kThreadsF = kCons;
constexpr int kChunk = 2048;            // doubles per chunk (16 KB)
constexpr int kSlotsG = 14;             // G role ring (3.5 half rows of 4 chunks, 224 KB)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
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
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAITC_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// TMA bulk copy global -> own shared memory, completion counted on `bar` (bytes % 16 == 0)
__device__ __forceinline__ void tma_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
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
__device__ __forceinline__ void st_remote_f64(uint32_t raddr, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(raddr), "d"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t raddr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(raddr) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ void consumer_bar() { asm volatile("bar.sync 1, %0;" ::"n"(kCons) : "memory"); }

// column of element k (0..3) owned by consumer thread t inside a chunk
__device__ __forceinline__ int own_col(int t, int k) { return (k >> 1) * 1024 + 2 * t + (k & 1); }

// w_i from r_i = G_i y + g_i: the pass-A epilogue value (epilogue.cuh, epi_a_store) without the
// store; `write` = this CTA commits mu / lambda (rank 0 of the pair only).
__device__ __forceinline__ double g_row_w(const PassAArgs &a, int64_t k, double s, const EpiA &e, const OuterA &o,
                                          bool write) {
    const double r = s + e.g;
    double m = e.mu;
    if (o.dual) {
        const double sl = a.rho > 0.0 ? proj_K(r + e.mu / a.rho, e.c) : 0.0;
        double lam = e.mu + a.step * (r - sl);
        if (a.project_dual && e.c == DUQUAD_CONE_NONPOS) lam = fmax(lam, 0.0);
        m = lam + o.beta_out * (lam - e.lp);
        if (write) {
            a.lam_prev[k] = lam;
            a.mu[k] = m;
        }
    }
    return a.rho > 0.0 ? proj_polar(m + a.rho * r, e.c) : m;
}

// Producer duty (TMA issue) is carried by lane 0 of warp kProdWarp, interleaved with its
// consumer work: chunk c + depth is issued right after every warp released chunc c, so the
// ring stays `depth` chunks ahead.  512 threads -> 128 registers per thread, no spills.
constexpr int kProdWarp = 15;

template <int NCHQ, int NCHG>
__global__ void __launch_bounds__(kCons, 1) __cluster_dims__(2, 1, 1) k_fused_stream(const FusedArgs f) {
    extern __shared__ __align__(128) uint8_t fsm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool prod = warp == kProdWarp && lane == 0;
    const int cta = blockIdx.x;
    const bool q_role = cta < f.nq_ctas;
    // ---- shared memory carve-up (first KB: barriers and small buffers)
    uint64_t *full = reinterpret_cast<uint64_t *>(fsm);              // [kSlotsG]
    uint64_t *empty = full + kSlotsG;                                 // [kSlotsG]
    uint64_t *xbar = empty + kSlotsG;                                 // [4] pair exchange
    double *xbuf = reinterpret_cast<double *>(xbar + 4);              // [4]
    double *red = xbuf + 4;                                           // [2][16]
    double *ring = reinterpret_cast<double *>(fsm + 1024);            // slots of kChunk doubles
    const int nsq = f.slots_q;
    double *ys = ring + (int64_t)nsq * kChunk;                        // Q role: y (ld doubles)
    double *rowbuf = ys + f.ld;                                       // Q role: [16][16]
    double *rowsum = rowbuf + 256;                                    // Q role: [rows]

    if (tid == 0) {
        for (int s = 0; s < kSlotsG; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kCons / 32);
        }
        for (int s = 0; s < 4; ++s) mbar_init(&xbar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (q_role)
        for (int64_t i = tid; i < f.ld / 2; i += kCons)
            reinterpret_cast<double2 *>(ys)[i] = reinterpret_cast<const double2 *>(f.y)[i];
    __syncthreads();
    cluster_sync_all();

    if (q_role) {
        // rows of this CTA: pairs (i, n-1-i), i = cta, cta + nq, ...  (balanced bytes)
        const int64_t n = f.n, half = (n + 1) / 2;
        auto row_of = [&](int64_t idx) -> int64_t {
            const int64_t pi = cta + (idx >> 1) * f.nq_ctas;
            return (idx & 1) ? n - 1 - pi : pi;
        };
        int64_t nrows = 0;
        for (int64_t pi = cta; pi < half; pi += f.nq_ctas) nrows += (n - 1 - pi != pi) ? 2 : 1;
        // producer cursor (row index, chunk) and its ring position
        int64_t p_idx = 0;
        int p_m = nrows > 0 ? (int)(row_of(0) / kChunk) : NCHQ;
        int p_s = 0;
        uint32_t p_ph = 0;
        auto produce_one = [&]() {   // issues the next chunk of the sequence, if any
            if (p_idx >= nrows) return;
            const int64_t r = row_of(p_idx);
            const int64_t c0 = (int64_t)p_m * kChunk;
            const int64_t start = p_m == r / kChunk ? (r & ~1LL) : c0;
            const int64_t end = c0 + kChunk < f.ld ? c0 + kChunk : f.ld;
            const uint32_t bytes = (uint32_t)((end - start) * 8);
            mbar_expect_tx(&full[p_s], bytes);
            tma_load(ring + p_s * kChunk + (start - c0), f.Q + r * f.ld + start, bytes, &full[p_s]);
            if (++p_s == nsq) {
                p_s = 0;
                p_ph ^= 1u;
            }
            if (++p_m == NCHQ) {
                ++p_idx;
                p_m = p_idx < nrows ? (int)(row_of(p_idx) / kChunk) : NCHQ;
            }
        };
        if (prod)
            for (int i = 0; i < nsq; ++i) produce_one();
        double acc[NCHQ][4];
#pragma unroll
        for (int m = 0; m < NCHQ; ++m)
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[m][k] = 0.0;
        int s = 0;
        uint32_t ph = 0;
        const int ld32 = (int)f.ld;
        const bool ragged = (f.ld % kChunk) != 0;
        const double2 *ys2 = reinterpret_cast<const double2 *>(ys);
        for (int64_t idx = 0; idx < nrows; ++idx) {
            const int r = (int)row_of(idx);
            const int m0 = r / kChunk;
            const double yr = ys[r];
            double rowacc = 0.0;
#pragma unroll
            for (int m = 0; m < NCHQ; ++m) {
                if (m < m0) continue;
                mbar_wait(&full[s], ph);
                const double2 *sl2 = reinterpret_cast<const double2 *>(ring + s * kChunk);
                const double2 qa = sl2[tid], qb = sl2[512 + tid];
                const int ca = m * kChunk + 2 * tid, cb = ca + 1024;
                if (m == m0 || (ragged && m == NCHQ - 1)) {      // triangle edge / row end: masks
                    const double qv[4] = {qa.x, qa.y, qb.x, qb.y};
                    const int cc[4] = {ca, ca + 1, cb, cb + 1};
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (cc[k] >= r && cc[k] < ld32) {
                            rowacc = fma(qv[k], ys[cc[k]], rowacc);
                            if (cc[k] > r) acc[m][k] = fma(qv[k], yr, acc[m][k]);
                        }
                } else {                                          // interior chunk: no masks
                    const double2 ya = ys2[ca >> 1], yb = ys2[cb >> 1];
                    rowacc = fma(qa.x, ya.x, rowacc);
                    rowacc = fma(qa.y, ya.y, rowacc);
                    rowacc = fma(qb.x, yb.x, rowacc);
                    rowacc = fma(qb.y, yb.y, rowacc);
                    acc[m][0] = fma(qa.x, yr, acc[m][0]);
                    acc[m][1] = fma(qa.y, yr, acc[m][1]);
                    acc[m][2] = fma(qb.x, yr, acc[m][2]);
                    acc[m][3] = fma(qb.y, yr, acc[m][3]);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
                if (prod) {                                       // refill this slot
                    mbar_wait(&empty[s], ph);
                    produce_one();
                }
                if (++s == nsq) {
                    s = 0;
                    ph ^= 1u;
                }
            }
            rowacc = warp_sum(rowacc);
            const int slot = (int)(idx & 15);
            if (lane == 0) rowbuf[slot * 16 + warp] = rowacc;
            if (slot == 15 || idx == nrows - 1) {   // flush: row dots of the last <= 16 rows
                consumer_bar();
                if (tid <= slot) {
                    double sr = 0.0;
#pragma unroll
                    for (int w = 0; w < 16; ++w) sr += rowbuf[tid * 16 + w];
                    rowsum[idx - slot + tid] = sr;
                }
                consumer_bar();
            }
        }
        // column sums -> workspace (this CTA's column of PT)
        double *pt = f.ws;
#pragma unroll
        for (int m = 0; m < NCHQ; ++m)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int64_t c = (int64_t)m * kChunk + own_col(tid, k);
                if (c < f.ld) pt[c * f.nb + cta] = acc[m][k];
            }
        consumer_bar();
        for (int64_t idx = tid; idx < nrows; idx += kCons) pt[row_of(idx) * f.nb + cta] += rowsum[idx];
    } else {
        // ---- G role: pair g owns rows [g0, g1); this CTA the column half `half_id`.
        // Per row: A = half sums (half 1 sends its sum to half 0); B = half 0 forms r, the
        // epilogue and w (and commits mu / lambda), sends w to half 1; both then accumulate
        // w G_i.  Software-pipelined: A(i+1) runs before B(i), hiding the exchange latency.
        const uint32_t half_id = cluster_rank();
        const bool h0 = half_id == 0;
        const int g = (cta - f.nq_ctas) >> 1;
        const int ng = (gridDim.x - f.nq_ctas) >> 1;
        const int64_t g0 = f.p * g / ng, g1 = f.p * (g + 1) / ng, nrow = g1 - g0;
        const int chunk0 = (int)half_id * NCHG;
        const int64_t nseq = nrow * NCHG;
        int64_t p_seq = 0;
        auto produce_one = [&]() {
            if (p_seq >= nseq) return;
            const int ps = (int)(p_seq % kSlotsG);
            const int64_t i = g0 + p_seq / NCHG;
            const int m = (int)(p_seq % NCHG);
            ++p_seq;
            const int64_t c0 = (int64_t)(chunk0 + m) * kChunk;
            const int64_t end = c0 + kChunk < f.ld ? c0 + kChunk : f.ld;
            if (end <= c0) {                   // chunk past the row end: an empty phase
                mbar_arrive(&full[ps]);
                return;
            }
            const uint32_t bytes = (uint32_t)((end - c0) * 8);
            mbar_expect_tx(&full[ps], bytes);
            tma_load(ring + ps * kChunk, f.G + i * f.ld + c0, bytes, &full[ps]);
        };
        if (prod)
            for (int i = 0; i < kSlotsG; ++i) produce_one();
        double yv[NCHG][4], acc[NCHG][4];
#pragma unroll
        for (int m = 0; m < NCHG; ++m)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int64_t c = (int64_t)(chunk0 + m) * kChunk + own_col(tid, k);
                yv[m][k] = c < f.ld ? f.y[c] : 0.0;
                acc[m][k] = 0.0;
            }
        const uint32_t x_remote = map_to_cta(smem_u32(xbuf), half_id ^ 1u);
        const uint32_t xb_remote = map_to_cta(smem_u32(xbar), half_id ^ 1u);
        const OuterA o = outer_a(f.a, MODE_SOLVE);
        const bool ragged_g = (int64_t)(chunk0 + NCHG) * kChunk > f.ld;
        auto stage_a = [&](int64_t it) -> double {     // this half's sum of row g0 + it
            double part = 0.0;
            int s = (int)((it * NCHG) % kSlotsG);
            uint32_t ph = (uint32_t)(((it * NCHG) / kSlotsG) & 1);
#pragma unroll
            for (int m = 0; m < NCHG; ++m) {
                mbar_wait(&full[s], ph);
                const double2 *sl2 = reinterpret_cast<const double2 *>(ring + s * kChunk);
                const double2 qa = sl2[tid], qb = sl2[512 + tid];
                if (ragged_g) {
                    const double qv[4] = {qa.x, qa.y, qb.x, qb.y};
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if ((int64_t)(chunk0 + m) * kChunk + own_col(tid, k) < f.ld)
                            part = fma(qv[k], yv[m][k], part);
                } else {
                    part = fma(qa.x, yv[m][0], part);
                    part = fma(qa.y, yv[m][1], part);
                    part = fma(qb.x, yv[m][2], part);
                    part = fma(qb.y, yv[m][3], part);
                }
                if (++s == kSlotsG) {
                    s = 0;
                    ph ^= 1u;
                }
            }
            part = warp_sum(part);
            if (lane == 0) red[(it & 1) * 16 + warp] = part;
            consumer_bar();
            double mine = 0.0;
#pragma unroll
            for (int w = 0; w < 16; ++w) mine += red[(it & 1) * 16 + w];
            if (!h0 && tid == 0) {
                st_remote_f64(x_remote + (uint32_t)(it & 3) * 8, mine);
                mbar_arrive_remote(xb_remote + (uint32_t)(it & 3) * 8);
            }
            return mine;
        };
        EpiA e_cur{}, e_next{};
        double mine_cur = 0.0;
        if (nrow > 0) {
            if (h0) e_cur = epi_a_load(f.a, MODE_SOLVE, f.a.nq + g0, o);
            mine_cur = stage_a(0);
        }
        for (int64_t it = 0; it < nrow; ++it) {
            double mine_next = 0.0;
            if (it + 1 < nrow) {
                if (h0) e_next = epi_a_load(f.a, MODE_SOLVE, f.a.nq + g0 + it + 1, o);
                mine_next = stage_a(it + 1);
            }
            // stage B(it)
            mbar_wait_cluster(&xbar[it & 3], (uint32_t)((it >> 2) & 1));
            double w;
            if (h0) {
                const double s_row = mine_cur + xbuf[it & 3];     // half 0 + half 1
                w = g_row_w(f.a, g0 + it, s_row, e_cur, o, tid == 0);
                if (tid == 0) {
                    st_remote_f64(x_remote + (uint32_t)(it & 3) * 8, w);
                    mbar_arrive_remote(xb_remote + (uint32_t)(it & 3) * 8);
                }
            } else {
                w = xbuf[it & 3];
            }
            int s = (int)((it * NCHG) % kSlotsG);
            uint32_t ph = (uint32_t)(((it * NCHG) / kSlotsG) & 1);
#pragma unroll
            for (int m = 0; m < NCHG; ++m) {
                const double2 *sl2 = reinterpret_cast<const double2 *>(ring + s * kChunk);
                const double2 qa = sl2[tid], qb = sl2[512 + tid];
                const double qv[4] = {qa.x, qa.y, qb.x, qb.y};
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (!ragged_g || (int64_t)(chunk0 + m) * kChunk + own_col(tid, k) < f.ld)
                        acc[m][k] = fma(w, qv[k], acc[m][k]);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
                if (prod) {                                       // refill this slot
                    mbar_wait(&empty[s], ph);
                    produce_one();
                }
                if (++s == kSlotsG) {
                    s = 0;
                    ph ^= 1u;
                }
            }
            e_cur = e_next;
            mine_cur = mine_next;
        }
        // column sums of this half -> workspace; zeros for the other half
        double *pt = f.ws;
#pragma unroll
        for (int m = 0; m < NCHG; ++m)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int64_t c = (int64_t)(chunk0 + m) * kChunk + own_col(tid, k);
                const int64_t co = (int64_t)((half_id ^ 1) * NCHG + m) * kChunk + own_col(tid, k);
                if (c < f.ld) pt[c * f.nb + cta] = acc[m][k];
                if (co < f.ld) pt[co * f.nb + cta] = 0.0;
            }
    }
    __syncthreads();
    cluster_sync_all();   // no CTA leaves while its partner may still write its shared memory
}

// grad_j = sum_b PT[j][b] (= Qy_j + t_j) + q_j: the pass-B epilogue, one warp per row j.
// bl / bs: epilogue views for load / store (they differ only in y when y ping-pongs).
__global__ void __launch_bounds__(256) k_fused_epi(const PassBArgs bl, const PassBArgs bs,
                                                   const double *__restrict__ ws, int nb) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
    const double avg_w = avg_weight(bl, MODE_SOLVE);
    for (int64_t j = warp; j < bl.nrows; j += nwarps) {
        EpiB e{};
        if (lane == 0) e = epi_b_load(bl, MODE_SOLVE, j, avg_w);
        double s = 0.0;
        for (int c = lane; c < nb; c += 32) s += ws[j * nb + c];
        s = warp_sum(s);
        if (lane == 0) {
            e.qy = s;
            epi_b_store(bs, MODE_SOLVE, j, 0.0, e, avg_w);
        }
    }
}

template <int NCHQ>
cudaError_t launch_t(const FusedArgs &f, cudaStream_t s) {
    constexpr int NCHG = (NCHQ + 1) / 2;
    k_fused_stream<NCHQ, NCHG><<<f.nb, kThreadsF, f.smem, s>>>(f);
    return cudaGetLastError();
}

template <int NCHQ>
cudaError_t configure_t(size_t smem) {
    constexpr int NCHG = (NCHQ + 1) / 2;
    cudaError_t e = cudaFuncSetAttribute(k_fused_stream<NCHQ, NCHG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e) return e;
    cudaFuncAttributes fa;
    if ((e = cudaFuncGetAttributes(&fa, k_fused_stream<NCHQ, NCHG>))) return e;
    if (fa.maxThreadsPerBlock < kThreadsF) {
        fprintf(stderr, "k_fused_stream<%d>: %d regs, maxThreadsPerBlock %d, local %zu\n", NCHQ, fa.numRegs,
                fa.maxThreadsPerBlock, fa.localSizeBytes);
        return cudaErrorInvalidConfiguration;
    }
    return cudaSuccess;
}

}  // namespace

// Q-role ring slots that fit next to y and the row buffers in `optin` bytes (0: does not fit).
int fused_q_slots(int64_t ld, int64_t rows_per_q_cta, size_t optin) {
    const int64_t fixed = 1024 + ld * 8 + 256 * 8 + rows_per_q_cta * 8;
    const int64_t s = ((int64_t)optin - fixed) / (kChunk * 8);
    return s < 3 ? 0 : (s > 8 ? 8 : (int)s);
}

// Shared memory of the stream kernel: barriers (1 KB) + max(Q role: ring + y + row buffers,
// G role: 14-slot ring).
size_t fused_smem_bytes(int64_t ld, int64_t rows_per_q_cta, int slots_q) {
    const size_t q = (size_t)slots_q * kChunk * 8 + (size_t)ld * 8 + 256 * 8 + (size_t)rows_per_q_cta * 8;
    const size_t g = (size_t)kSlotsG * kChunk * 8;
    return 1024 + (q > g ? q : g);
}

int fused_nchq(int64_t ld) { return (int)((ld + kChunk - 1) / kChunk); }

cudaError_t configure_fused_kernels(int nchq, size_t smem) {
    switch (nchq) {
        case 2: return configure_t<2>(smem);
        case 3: return configure_t<3>(smem);
        case 4: return configure_t<4>(smem);
        case 5: return configure_t<5>(smem);
        case 6: return configure_t<6>(smem);
        case 7: return configure_t<7>(smem);
        case 8: return configure_t<8>(smem);
        case 9: return configure_t<9>(smem);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_fused_stream(const FusedArgs &f, cudaStream_t s) {
    switch (f.nchq) {
        case 2: return launch_t<2>(f, s);
        case 3: return launch_t<3>(f, s);
        case 4: return launch_t<4>(f, s);
        case 5: return launch_t<5>(f, s);
        case 6: return launch_t<6>(f, s);
        case 7: return launch_t<7>(f, s);
        case 8: return launch_t<8>(f, s);
        case 9: return launch_t<9>(f, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_fused_epi(const PassBArgs &bl, const PassBArgs &bs, const double *ws, int nb, int grid,
                             cudaStream_t s) {
    k_fused_epi<<<grid, 256, 0, s>>>(bl, bs, ws, nb);
    return cudaGetLastError();
}

}  // namespace dq
