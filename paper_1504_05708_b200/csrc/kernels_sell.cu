// Lane-per-row sparse kernels of the DuQuad inner step (config 4):
// SELL-32 for rows of nearly equal length, thread-per-row CSR for short rows of unequal length.
//
// Both run the same two passes and row epilogues (epilogue.cuh) as the sub-warp CSR kernels
// (kernels_csr.cu), with one lane per row, so the epilogue's vector accesses are coalesced and
// each lane sums its row's nonzeros in their CSR order: the row sums do not depend on the storage
// (SELL or CSR) or on the row sharding.
//
// SELL-32: 32 consecutive rows form a slice, and the k-th nonzero of every row of the slice sits
// in one 32-wide column, so every matrix load of a warp is one coalesced 256-byte (values) /
// 128-byte (indices) request and the slice width is warp-uniform (no divergence).  A slice costs
// one load round (U >= the slice width) and one gather round; no row pointer is on the critical
// path.  Padding entries carry value 0 and a valid column of the same row (an exact zero term).
// Used when the padding stays small (config 4's pass A: Q rows of 11 and G rows of 8 nonzeros).
//
// Thread-per-row CSR: lane l of a warp owns row base + l and walks its own nonzeros.  A warp's 32
// rows are contiguous in memory, so the lanes' scattered loads hit the same L1 lines round after
// round (L1-allocating loads, L2 evict-first); no padding and no row permutation.  Used when rows
// are short but unequal (config 4's pass B: G' rows with Poisson(4) nonzeros, where SELL-32
// would pad 2.2x and a length-sorted SELL scatters the heavy pass-B epilogue).
//
// The paper's observation that sparse data make the method cheap (P:1272-1274, P:1317-1319:
// "only sparse matrix-vector products") is where these layouts pay: the matrix stream is bound by
// HBM bandwidth rather than by the latency of the sub-warp kernels' row-pointer -> index chain.
#include <cuda_runtime.h>
#include <thrust/device_ptr.h>
#include <thrust/execution_policy.h>
#include <thrust/extrema.h>
#include <thrust/reduce.h>
#include <thrust/scan.h>

#include <algorithm>

#include "duquad_internal.h"
#include "epilogue.cuh"

namespace dq {

namespace {

constexpr int kLaneThreads = 256;
#ifndef DQ_LANE_MINB   // minimum resident blocks per SM of the lane kernels (register cap)
#define DQ_LANE_MINB 1
#endif
#ifndef DQ_SELLA_MINB  // SELL pass A: its solve-mode epilogue (the DFOM step) alone would take ~80
#define DQ_SELLA_MINB 4 // registers (2-3 CTAs/SM); capped at 64 for 4 CTAs/SM
#endif

__device__ __forceinline__ uint64_t evict_first() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// streamed once (SELL): bypass L1
__device__ __forceinline__ double ld_na_f64(const double *p, uint64_t pol) {
    double r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ int32_t ld_na_i32(const int32_t *p, uint64_t pol) {
    int32_t r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}
// re-read by neighbouring lanes in later rounds (thread-per-row CSR): allocate in L1
__device__ __forceinline__ double ld_l1_f64(const double *p, uint64_t pol) {
    double r;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ int32_t ld_l1_i32(const int32_t *p, uint64_t pol) {
    int32_t r;
    asm("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}

// row of lane `lane` of slice s (-1: an empty lane of a segment's last slice)
__device__ __forceinline__ int64_t sell_row(const SellMat &m, int64_t s, int lane) {
    if (s < m.nsl_q) {
        const int64_t r = s * 32 + lane;
        return r < m.nq ? r : -1;
    }
    const int64_t r = m.nq + (s - m.nsl_q) * 32 + lane;
    return r < m.rows ? r : -1;
}

// lane's row . v over the slice [base, base + 32 w): nonzeros in CSR order, U loads per round
template <int U>
__device__ __forceinline__ double sell_dot(const SellMat &m, int64_t base, int w, int lane,
                                           const double *__restrict__ v, uint64_t pol) {
    double acc = 0.0;
    const double *va = m.val + base + lane;
    const int32_t *ci = m.col + base + lane;
    for (int k0 = 0; k0 < w; k0 += U) {
        int32_t c[U];
        double a[U], x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const bool ok = k0 + u < w;   // warp-uniform
            c[u] = ok ? ld_na_i32(ci + (int64_t)(k0 + u) * 32, pol) : 0;
            a[u] = ok ? ld_na_f64(va + (int64_t)(k0 + u) * 32, pol) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = k0 + u < w ? __ldg(v + c[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (k0 + u < w) acc = fma(a[u], x[u], acc);
    }
    return acc;
}

// lane's own CSR row [lo, lo + len) . v, rounds of U nonzeros (the warp's longest row bounds the
// trip count; lanes past their row end are predicated off)
template <int U>
__device__ __forceinline__ double rowt_dot(const int32_t *__restrict__ ci, const double *__restrict__ va, int32_t lo,
                                           int32_t len, const double *__restrict__ v, uint64_t pol) {
    const int32_t wl = __reduce_max_sync(0xffffffffu, len);
    double acc = 0.0;
    for (int k0 = 0; k0 < wl; k0 += U) {
        int32_t c[U];
        double a[U], x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const bool ok = k0 + u < len;
            c[u] = ok ? ld_l1_i32(ci + lo + k0 + u, pol) : -1;
            a[u] = ok ? ld_l1_f64(va + lo + k0 + u, pol) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = c[u] >= 0 ? __ldg(v + c[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (c[u] >= 0) acc = fma(a[u], x[u], acc);
    }
    return acc;
}

// lane's row of the DIA Q block (local row i, global row gi): the diagonals in ascending column
// order, rounds of U, no index loads (the y loads of a round are contiguous per diagonal)
template <int U>
__device__ __forceinline__ double dia_dot(const DiaMat &d, int64_t i, const double *__restrict__ v, uint64_t pol) {
    const int64_t gi = d.r0 + i;
    double acc = 0.0;
    for (int k0 = 0; k0 < d.nd; k0 += U) {
        double a[U], x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int k = k0 + u;
            if (k < d.nd) {   // warp-uniform
                int64_t c = gi + d.off[k];
                c = c < 0 ? 0 : (c >= d.n ? d.n - 1 : c);   // outside the matrix: the stored value is 0
                a[u] = ld_na_f64(d.val + (int64_t)k * d.ldv + i, pol);
                x[u] = __ldg(v + c);
            } else {
                a[u] = 0.0;
                x[u] = 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (k0 + u < d.nd) acc = fma(a[u], x[u], acc);
    }
    return acc;
}

// symmetric half band (DiaMat.sym): row i's lower entries Q[gi, gi-o] = Q[gi-o, gi] read from the
// stored upper diagonals shifted by o, then its upper entries; both in ascending column order, so
// the row sum is bitwise the full band's / the CSR kernels' for a bitwise symmetric Q.  One DRAM
// round per row (rounds of DU: config 4's 5 + 6 loads): the upper round re-reads lines the lower
// round has just pulled into L1.
template <int DU>
__device__ __forceinline__ double dia_dot_sym(const DiaMat &d, int64_t i, const double *__restrict__ v,
                                              uint64_t pol) {
    const int64_t gi = d.r0 + i;
    const double *base = d.val + d.halo + i;
    double acc = 0.0;
    const int k1 = d.off[0] == 0 ? 1 : 0;          // lower half: the strictly positive offsets,
    for (int k0 = d.nd - 1; k0 >= k1; k0 -= DU) {  // widest first (ascending columns)
        double a[DU], x[DU];
#pragma unroll
        for (int u = 0; u < DU; ++u) {
            const int k = k0 - u;
            if (k >= k1) {   // warp-uniform
                const int o = d.off[k];
                const int64_t c = gi - o;
                a[u] = ld_l1_f64(base + (int64_t)k * d.ldv - o, pol);
                x[u] = __ldg(v + (c < 0 ? 0 : c));                // before column 0: stored 0
            } else {
                a[u] = 0.0;
                x[u] = 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < DU; ++u)
            if (k0 - u >= k1) acc = fma(a[u], x[u], acc);
    }
    for (int k0 = 0; k0 < d.nd; k0 += DU) {        // upper half, ascending offsets
        double a[DU], x[DU];
#pragma unroll
        for (int u = 0; u < DU; ++u) {
            const int k = k0 + u;
            if (k < d.nd) {
                const int64_t c = gi + d.off[k];
                a[u] = ld_l1_f64(base + (int64_t)k * d.ldv, pol);
                x[u] = __ldg(v + (c >= d.n ? d.n - 1 : c));   // past the last column: stored 0
            } else {
                a[u] = 0.0;
                x[u] = 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < DU; ++u)
            if (k0 + u < d.nd) acc = fma(a[u], x[u], acc);
    }
    return acc;
}

#ifndef DQ_SELL_MIX
#define DQ_SELL_MIX 1
#endif
#ifndef DQ_DIA_DU
#define DQ_DIA_DU 6
#endif

template <int MODE, int U>
__global__ void __launch_bounds__(kLaneThreads, DQ_SELLA_MINB) k_pass_a_sell(const PassAArgs a) {
    pdl_wait();   // everything below reads iterates or writes (PDL, epilogue.cuh)
    pdl_trigger();
    if (a.skip && *a.skip) return;
    const SellMat &m = a.sell;
    const int lane = threadIdx.x & 31;
    // sub-ranges: Q rows only [0, nq), G rows only [nq, rows), or all (segments never share a slice)
    const int64_t s_lo = a.row_begin >= m.nq ? m.nsl_q : 0;
    const int64_t s_hi = a.row_end <= m.nq ? m.nsl_q : m.nsl;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const OuterA o = outer_a(a, MODE);
    const uint64_t pol = evict_first();
    // whole range: Q and G slices interleaved in proportion (DQ_SELL_MIX), so the DIA Q rows (one
    // DRAM round each) and the G rows (index -> gather chains) are in flight together
    const bool mix = DQ_SELL_MIX && s_lo == 0 && s_hi == m.nsl && m.nsl_q > 0 && m.nsl > m.nsl_q;
    for (int64_t t = s_lo + warp; t < s_hi; t += nwarps) {
        int64_t s = t;
        if (mix) {
            const int64_t qb = t * m.nsl_q / m.nsl, qn = (t + 1) * m.nsl_q / m.nsl;
            s = qn > qb ? qb : m.nsl_q + (t - qb);
        }
        const int64_t r = sell_row(m, s, lane);
        const int64_t base = m.sptr[s];
        const int w = (int)((m.sptr[s + 1] - base) >> 5);
        EpiA e{};
        if (r >= 0) e = epi_a_load(a, MODE, r, o);
        const double acc = (s < m.nsl_q && a.dia.nd > 0)
                               ? (a.dia.sym ? dia_dot_sym<DQ_DIA_DU>(a.dia, s * 32 + lane, a.y, pol)
                                            : dia_dot<U>(a.dia, s * 32 + lane, a.y, pol))
                               : sell_dot<U>(m, base, w, lane, a.y, pol);
        if (r >= 0) epi_a_store(a, MODE, r, acc, e, o);
    }
}

template <int MODE, int U>
__global__ void __launch_bounds__(kLaneThreads, DQ_LANE_MINB) k_pass_b_sell(const PassBArgs b) {
    pdl_wait();
    pdl_trigger();
    if (b.skip && *b.skip) return;
    const SellMat &m = b.sell;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const double avg_w = avg_weight(b, MODE);
    const uint64_t pol = evict_first();
    for (int64_t s = warp; s < m.nsl; s += nwarps) {
        const int64_t j = sell_row(m, s, lane);
        const int64_t base = m.sptr[s];
        const int w = (int)((m.sptr[s + 1] - base) >> 5);
        EpiB e{};
        if (j >= 0) e = epi_b_load(b, MODE, j, avg_w);
        const double t = sell_dot<U>(m, base, w, lane, b.w, pol);
        if (j >= 0) epi_b_store(b, MODE, j, t, e, avg_w);
    }
}

template <int MODE, int U>
__global__ void __launch_bounds__(kLaneThreads, DQ_LANE_MINB) k_pass_a_rowt(const PassAArgs a) {
    pdl_wait();   // everything below reads iterates or writes (PDL, epilogue.cuh)
    pdl_trigger();
    if (a.skip && *a.skip) return;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const OuterA o = outer_a(a, MODE);
    const uint64_t pol = evict_first();
    for (int64_t base = a.row_begin + warp * 32; base < a.row_end; base += nwarps * 32) {
        const int64_t r = base + lane;
        const bool v = r < a.row_end;
        const int32_t lo = v ? a.rp[r] : 0, len = v ? a.rp[r + 1] - lo : 0;
        EpiA e{};
        if (v) e = epi_a_load(a, MODE, r, o);
        const double acc = rowt_dot<U>(a.ci, a.va, lo, len, a.y, pol);
        if (v) epi_a_store(a, MODE, r, acc, e, o);
    }
}

template <int MODE, int U>
__global__ void __launch_bounds__(kLaneThreads, DQ_LANE_MINB) k_pass_b_rowt(const PassBArgs b) {
    pdl_wait();
    pdl_trigger();
    if (b.skip && *b.skip) return;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const double avg_w = avg_weight(b, MODE);
    const uint64_t pol = evict_first();
    for (int64_t base = warp * 32; base < b.nrows; base += nwarps * 32) {
        const int64_t j = base + lane;
        const bool v = j < b.nrows;
        const int32_t lo = v ? b.rp[j] : 0, len = v ? b.rp[j + 1] - lo : 0;
        EpiB e{};
        if (v) e = epi_b_load(b, MODE, j, avg_w);
        const double t = rowt_dot<U>(b.ci, b.va, lo, len, b.w, pol);
        if (v) epi_b_store(b, MODE, j, t, e, avg_w);
    }
}

// ------------------------------------------------------------------ layout construction
__global__ void k_row_len(const int32_t *rp, int64_t rows, int32_t *len) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < rows) len[i] = rp[i + 1] - rp[i];
}

// 32 x the longest row of every slice (slices never straddle the two segments)
__global__ void k_slice_width(const int32_t *len, int64_t rows, int64_t nq, int64_t nsl_q, int64_t nsl,
                              int64_t *width) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= nsl) return;
    const int64_t r0 = s < nsl_q ? s * 32 : nq + (s - nsl_q) * 32;
    const int64_t r1 = s < nsl_q ? (r0 + 32 < nq ? r0 + 32 : nq) : (r0 + 32 < rows ? r0 + 32 : rows);
    int32_t w = 0;
    for (int64_t r = r0; r < r1; ++r) w = max(w, len[r]);
    width[s] = 32 * (int64_t)w;
}

__global__ void k_sell_fill(const int32_t *rp, const int32_t *ci, const double *va, int64_t rows, int64_t nq,
                            int64_t nsl_q, int64_t nsl, const int64_t *sptr, double *sv, int32_t *sc) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nsl * 32) return;
    const int64_t s = t >> 5, l = t & 31;
    const int64_t r = s < nsl_q ? (s * 32 + l < nq ? s * 32 + l : -1)
                                : (nq + (s - nsl_q) * 32 + l < rows ? nq + (s - nsl_q) * 32 + l : -1);
    const int32_t b = r >= 0 ? rp[r] : 0, len = r >= 0 ? rp[r + 1] - b : 0;
    const int32_t pad_col = len > 0 ? ci[b + len - 1] : 0;
    const int64_t base = sptr[s], w = (sptr[s + 1] - base) >> 5;
    for (int64_t k = 0; k < w; ++k) {
        sv[base + k * 32 + l] = k < len ? va[b + k] : 0.0;
        sc[base + k * 32 + l] = k < len ? ci[b + k] : pad_col;
    }
}

inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

template <typename K>
int occ_of(K kern) {
    int b = 0;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, kLaneThreads, 0) == cudaSuccess && b > 0 ? b : 1;
}

}  // namespace

void sell_free(SellStore *st) {
    if (st->val) cudaFree(st->val);
    if (st->col) cudaFree(st->col);
    if (st->sptr) cudaFree(st->sptr);
    *st = SellStore{};
}

cudaError_t sparse_plan(const int32_t *rp, int64_t rows, int64_t nq, SparsePlan *plan, cudaStream_t s) {
    *plan = SparsePlan{};
    plan->nsl_q = (nq + 31) / 32;
    plan->nsl = plan->nsl_q + (rows - nq + 31) / 32;
    if (rows <= 0) return cudaSuccess;
    int32_t *len = nullptr;
    int64_t *width = nullptr;
    cudaError_t e = cudaMalloc(&len, rows * sizeof(int32_t));
    if (!e) e = cudaMalloc(&width, (plan->nsl + 1) * sizeof(int64_t));
    if (!e) {
        k_row_len<<<nblk(rows, 256), 256, 0, s>>>(rp, rows, len);
        k_slice_width<<<nblk(plan->nsl, 256), 256, 0, s>>>(len, rows, nq, plan->nsl_q, plan->nsl, width);
        e = cudaGetLastError();
    }
    if (!e) {
        thrust::device_ptr<int64_t> wp(width);
        thrust::device_ptr<int32_t> lp(len);
        plan->padded = thrust::reduce(thrust::cuda::par.on(s), wp, wp + plan->nsl, (int64_t)0);
        plan->max_len = *thrust::max_element(thrust::cuda::par.on(s), lp, lp + rows);
        e = cudaGetLastError();
    }
    if (len) cudaFree(len);
    if (width) cudaFree(width);
    return e;
}

cudaError_t sell_build(const int32_t *rp, const int32_t *ci, const double *va, int64_t rows, int64_t nq,
                       const SparsePlan &plan, SellStore *out, cudaStream_t s) {
    *out = SellStore{};
    const int64_t nsl_q = plan.nsl_q, nsl = plan.nsl;
    if (rows <= 0 || nsl <= 0) return cudaSuccess;
    SellStore st{};
    st.nsl = nsl;
    st.nsl_q = nsl_q;
    st.nq = nq;
    st.rows = rows;
    st.padded = plan.padded;
    cudaError_t e = cudaMalloc(&st.sptr, (nsl + 1) * sizeof(int64_t));
    if (!e) e = cudaMalloc(&st.val, std::max<int64_t>(plan.padded, 2) * sizeof(double));
    if (!e) e = cudaMalloc(&st.col, std::max<int64_t>(plan.padded, 2) * sizeof(int32_t));
    int32_t *len = nullptr;
    if (!e) e = cudaMalloc(&len, rows * sizeof(int32_t));
    if (!e) {
        k_row_len<<<nblk(rows, 256), 256, 0, s>>>(rp, rows, len);
        k_slice_width<<<nblk(nsl, 256), 256, 0, s>>>(len, rows, nq, nsl_q, nsl, st.sptr);
        e = cudaMemsetAsync(st.sptr + nsl, 0, sizeof(int64_t), s);
    }
    if (!e) {
        thrust::device_ptr<int64_t> sp(st.sptr);
        thrust::exclusive_scan(thrust::cuda::par.on(s), sp, sp + nsl + 1, sp);
        k_sell_fill<<<nblk(nsl * 32, 256), 256, 0, s>>>(rp, ci, va, rows, nq, nsl_q, nsl, st.sptr, st.val, st.col);
        e = cudaGetLastError();
    }
    if (!e) e = cudaStreamSynchronize(s);
    if (len) cudaFree(len);
    if (e) {
        sell_free(&st);
        return e;
    }
    *out = st;
    return cudaSuccess;
}

// ------------------------------------------------------------------ DIA (banded Q rows)
namespace {
constexpr int kDiaWin = 64;   // column offsets considered: [-64, 64]
__global__ void k_dia_hist(const int32_t *rp, const int32_t *ci, int64_t rows, int64_t r0, int32_t *hist,
                           int32_t *bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= rows) return;
    int32_t prev = -1;
    for (int32_t e = rp[i]; e < rp[i + 1]; ++e) {
        const int64_t off = (int64_t)ci[e] - (r0 + i);
        if (off < -kDiaWin || off > kDiaWin || ci[e] == prev) {   // wide band or a duplicate column
            *bad = 1;
            return;
        }
        prev = ci[e];
        atomicAdd(&hist[off + kDiaWin], 1);
    }
}
__global__ void k_dia_fill(const int32_t *rp, const int32_t *ci, const double *va, int64_t rows, int64_t r0,
                           const int32_t *slot, int64_t ldv, double *val) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= rows) return;
    for (int32_t e = rp[i]; e < rp[i + 1]; ++e) val[(int64_t)slot[ci[e] - (r0 + i) + kDiaWin] * ldv + i] = va[e];
}
// symmetric half band from the full band (full diagonals f = 0..nd-1, offsets ascending and
// symmetric: diagonal f's mirror is nd-1-f).  Stored diagonal k (offset o = off[kf0 + k] >= 0):
// sv[k][halo + i] = full[kf0 + k][i]; for o > 0 the lower entry full[nd-1-kf0-k][i] = Q[gi, gi-o]
// either fills the halo (i - o < 0: row gi - o is not in the slice) or must equal the stored upper
// entry of row i - o bitwise (else *bad = 1 and the full band is kept)
__global__ void k_dia_sym(const double *full, int64_t ldf, int32_t nd, int32_t kf0, const int32_t *off_s, int32_t ns,
                          int64_t rows, int64_t halo, int64_t ldv, double *sv, int32_t *bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= rows) return;
    for (int k = 0; k < ns; ++k) {
        const int o = off_s[k];
        sv[(int64_t)k * ldv + halo + i] = full[(int64_t)(kf0 + k) * ldf + i];
        if (o == 0) continue;
        const double lo = full[(int64_t)(nd - 1 - kf0 - k) * ldf + i];
        if (i - o < 0) sv[(int64_t)k * ldv + halo + i - o] = lo;
        else if (lo != full[(int64_t)(kf0 + k) * ldf + i - o]) *bad = 1;
    }
}
}  // namespace

cudaError_t dia_build(const int32_t *rp, const int32_t *ci, const double *va, int64_t rows, int64_t r0, int64_t n,
                      int64_t nnz, double max_pad, bool allow_sym, DiaMat *out, double **val, cudaStream_t s) {
    *out = DiaMat{};
    *val = nullptr;
    if (rows <= 0 || nnz <= 0) return cudaSuccess;
    int32_t *hist = nullptr, *slot = nullptr;
    cudaError_t e = cudaMalloc(&hist, (2 * kDiaWin + 2) * sizeof(int32_t));
    if (!e) e = cudaMalloc(&slot, (2 * kDiaWin + 1) * sizeof(int32_t));
    if (!e) e = cudaMemsetAsync(hist, 0, (2 * kDiaWin + 2) * sizeof(int32_t), s);
    int32_t h[2 * kDiaWin + 2];
    if (!e) {
        k_dia_hist<<<nblk(rows, 256), 256, 0, s>>>(rp, ci, rows, r0, hist, hist + 2 * kDiaWin + 1);
        e = cudaMemcpyAsync(h, hist, sizeof(h), cudaMemcpyDeviceToHost, s);
    }
    if (!e) e = cudaStreamSynchronize(s);
    DiaMat d{};
    int32_t sl[2 * kDiaWin + 1];
    bool ok = !e && h[2 * kDiaWin + 1] == 0;
    if (ok) {
        for (int o = 0; o <= 2 * kDiaWin; ++o) {
            sl[o] = -1;
            if (h[o] > 0) {
                if (d.nd == kDiaMax) {
                    ok = false;
                    break;
                }
                sl[o] = d.nd;
                d.off[d.nd++] = o - kDiaWin;
            }
        }
    }
    d.ldv = (rows + 31) / 32 * 32;
    ok = ok && d.nd > 0 && (double)d.nd * (double)rows <= max_pad * (double)nnz;
    if (ok) {
        e = cudaMemcpyAsync(slot, sl, sizeof(sl), cudaMemcpyHostToDevice, s);
        if (!e) e = cudaMalloc(val, (size_t)d.nd * d.ldv * sizeof(double));
        if (!e) e = cudaMemsetAsync(*val, 0, (size_t)d.nd * d.ldv * sizeof(double), s);
        if (!e) {
            k_dia_fill<<<nblk(rows, 256), 256, 0, s>>>(rp, ci, va, rows, r0, slot, d.ldv, *val);
            e = cudaGetLastError();
        }
        if (!e) e = cudaStreamSynchronize(s);
        d.val = *val;
        d.r0 = r0;
        d.n = n;
        // symmetric half band: offsets symmetric about 0 with at least one off-diagonal
        bool symm = allow_sym && !e && d.off[d.nd - 1] > 0;
        for (int k = 0; symm && k < d.nd; ++k) symm = d.off[k] == -d.off[d.nd - 1 - k];
        if (symm) {
            DiaMat h = d;
            const int32_t kf0 = d.nd / 2;   // first offset >= 0 (the offsets are symmetric)
            h.nd = d.nd - kf0;
            for (int k = 0; k < h.nd; ++k) h.off[k] = d.off[kf0 + k];
            h.halo = h.off[h.nd - 1];
            h.ldv = (rows + h.halo + 31) / 32 * 32;
            h.sym = 1;
            double *sv = nullptr;
            int32_t bad = 0;
            e = cudaMemcpyAsync(slot, h.off, h.nd * sizeof(int32_t), cudaMemcpyHostToDevice, s);
            if (!e) e = cudaMemsetAsync(hist, 0, sizeof(int32_t), s);
            if (!e) e = cudaMalloc(&sv, (size_t)h.nd * h.ldv * sizeof(double));
            if (!e) e = cudaMemsetAsync(sv, 0, (size_t)h.nd * h.ldv * sizeof(double), s);
            if (!e) {
                k_dia_sym<<<nblk(rows, 256), 256, 0, s>>>(*val, d.ldv, d.nd, kf0, slot, h.nd, rows, h.halo, h.ldv,
                                                          sv, hist);
                e = cudaGetLastError();
            }
            if (!e) e = cudaMemcpyAsync(&bad, hist, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
            if (!e) e = cudaStreamSynchronize(s);
            if (!e && !bad) {
                cudaFree(*val);
                *val = sv;
                h.val = sv;
                d = h;
            } else if (sv) {
                cudaFree(sv);
            }
        }
        if (!e) *out = d;
    }
    cudaFree(hist);
    cudaFree(slot);
    if (e && *val) {
        cudaFree(*val);
        *val = nullptr;
    }
    return e;
}

SellMat sell_view(const SellStore &st) {
    SellMat m{};
    m.val = st.val;
    m.col = st.col;
    m.sptr = st.sptr;
    m.nsl = st.nsl;
    m.nsl_q = st.nsl_q;
    m.nq = st.nq;
    m.rows = st.rows;
    return m;
}

// Load-round width: 4 for both kinds, whatever the row lengths.  Measured on config 4
// (scripts/sparse_sweep.py, profiles/r02_sparse_sweep*.jsonl): SELL pass A (slices of width 11 / 8)
// 50.3 us at U = 4, 52.0 at 8, 60.7 at 12, 62.1 at 16 (with DIA for the Q rows: 45.6 at 4, 46.7 at
// 8) -- the kernel is bound by memory-level parallelism, and fewer registers per lane (more
// resident warps) beat fewer rounds per slice; thread-per-row pass B 31.9 us at U = 4, 32.3 at 8.
int lane_unroll(int kind, int64_t max_width, double mean_len) {
    (void)kind;
    (void)max_width;
    (void)mean_len;
    return 4;
}

#define DQ_LANE_DISPATCH(KERN, MODE, U, GRID, ARG)                                         \
    switch (U) {                                                                            \
        case 4: return launch_ex(KERN<MODE, 4>, GRID, kLaneThreads, 0, s, cfg.pdl, 0, ARG);   \
        case 8: return launch_ex(KERN<MODE, 8>, GRID, kLaneThreads, 0, s, cfg.pdl, 0, ARG);   \
        case 12: return launch_ex(KERN<MODE, 12>, GRID, kLaneThreads, 0, s, cfg.pdl, 0, ARG); \
        default: return launch_ex(KERN<MODE, 16>, GRID, kLaneThreads, 0, s, cfg.pdl, 0, ARG); \
    }

int lane_blocks_per_sm(int pass, int kind, int u) {
    if (pass == 0) {
        if (kind == SPK_SELL)
            return u == 4 ? occ_of(k_pass_a_sell<MODE_SOLVE, 4>) : u == 8 ? occ_of(k_pass_a_sell<MODE_SOLVE, 8>)
                   : u == 12 ? occ_of(k_pass_a_sell<MODE_SOLVE, 12>) : occ_of(k_pass_a_sell<MODE_SOLVE, 16>);
        return u == 4 ? occ_of(k_pass_a_rowt<MODE_SOLVE, 4>) : occ_of(k_pass_a_rowt<MODE_SOLVE, 8>);
    }
    if (kind == SPK_SELL)
        return u == 4 ? occ_of(k_pass_b_sell<MODE_SOLVE, 4>) : u == 8 ? occ_of(k_pass_b_sell<MODE_SOLVE, 8>)
               : u == 12 ? occ_of(k_pass_b_sell<MODE_SOLVE, 12>) : occ_of(k_pass_b_sell<MODE_SOLVE, 16>);
    return u == 4 ? occ_of(k_pass_b_rowt<MODE_SOLVE, 4>) : occ_of(k_pass_b_rowt<MODE_SOLVE, 8>);
}

cudaError_t launch_pass_a_lane(const PassAArgs &a, int mode, const LaunchCfg &cfg, cudaStream_t s) {
    if (a.row_end <= a.row_begin) return cudaSuccess;
    if (a.sp_kind == SPK_SELL) {
        if (mode == MODE_SOLVE) {
            DQ_LANE_DISPATCH(k_pass_a_sell, MODE_SOLVE, a.sp_u, cfg.grid, a);
        } else {
            DQ_LANE_DISPATCH(k_pass_a_sell, MODE_LIN, a.sp_u, cfg.grid, a);
        }
    } else if (mode == MODE_SOLVE) {
        if (a.sp_u == 4) return launch_ex(k_pass_a_rowt<MODE_SOLVE, 4>, cfg.grid, kLaneThreads, 0, s, cfg.pdl, 0, a);
        else return launch_ex(k_pass_a_rowt<MODE_SOLVE, 8>, cfg.grid, kLaneThreads, 0, s, cfg.pdl, 0, a);
    } else {
        if (a.sp_u == 4) return launch_ex(k_pass_a_rowt<MODE_LIN, 4>, cfg.grid, kLaneThreads, 0, s, cfg.pdl, 0, a);
        else return launch_ex(k_pass_a_rowt<MODE_LIN, 8>, cfg.grid, kLaneThreads, 0, s, cfg.pdl, 0, a);
    }
    return cudaGetLastError();
}

cudaError_t launch_pass_b_lane(const PassBArgs &b, int mode, const LaunchCfg &cfg, cudaStream_t s) {
    if (b.nrows <= 0) return cudaSuccess;
    if (b.sp_kind == SPK_SELL) {
        if (mode == MODE_SOLVE) {
            DQ_LANE_DISPATCH(k_pass_b_sell, MODE_SOLVE, b.sp_u, cfg.grid, b);
        } else {
            DQ_LANE_DISPATCH(k_pass_b_sell, MODE_LIN, b.sp_u, cfg.grid, b);
        }
    } else if (mode == MODE_SOLVE) {
        if (b.sp_u == 4) return launch_ex(k_pass_b_rowt<MODE_SOLVE, 4>, cfg.grid, kLaneThreads, 0, s, cfg.pdl, 0, b);
        else return launch_ex(k_pass_b_rowt<MODE_SOLVE, 8>, cfg.grid, kLaneThreads, 0, s, cfg.pdl, 0, b);
    } else {
        if (b.sp_u == 4) return launch_ex(k_pass_b_rowt<MODE_LIN, 4>, cfg.grid, kLaneThreads, 0, s, cfg.pdl, 0, b);
        else return launch_ex(k_pass_b_rowt<MODE_LIN, 8>, cfg.grid, kLaneThreads, 0, s, cfg.pdl, 0, b);
    }
    return cudaGetLastError();
}

}  // namespace dq
