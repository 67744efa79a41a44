// SELL-32 sm_100a kernels of the sparse DuQuad inner step (config 4).
//
// The same two passes and row epilogues (epilogue.cuh) as the CSR kernels, with the matrix
// stored slice-major: 32 consecutive (or, after a windowed sort by length, length-grouped) rows
// form a slice, and the k-th nonzero of every row of the slice sits in one 32-wide column, so
// a warp owns a slice, lane l owns row l of it, and every matrix load of the warp is one
// coalesced 256-byte (values) / 128-byte (indices) request.  The slice width is warp-uniform:
// no divergence, no row-pointer load on the critical path (the CSR kernels' row-pointer ->
// index -> gather chain), and each lane sums its row's nonzeros in their CSR order, so the row
// sums do not depend on the slicing or on the row sharding.  Padding entries carry value 0 and a
// valid column of the same row (their product adds an exact zero).
//
// The paper's observation that sparse data make the method cheap (P:1272-1274, P:1317-1319:
// "only sparse matrix-vector products") is where this layout pays: the matrix stream is bound by
// HBM bandwidth, not by the latency of the index chain.
#include <cuda_runtime.h>
#include <thrust/device_ptr.h>
#include <thrust/execution_policy.h>
#include <thrust/extrema.h>
#include <thrust/reduce.h>
#include <thrust/scan.h>
#include <thrust/sequence.h>
#include <thrust/sort.h>

#include <algorithm>

#include "duquad_internal.h"
#include "epilogue.cuh"

namespace dq {

namespace {

constexpr int kSellThreads = 256;
constexpr int kSellU = 8;   // nonzeros per lane in flight per round (loads issued together)

__device__ __forceinline__ uint64_t sell_evict_first() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ double sell_ld_f64(const double *p, uint64_t pol) {
    double r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ int32_t sell_ld_i32(const int32_t *p, uint64_t pol) {
    int32_t r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}

// row of lane `lane` of slice s (-1: an empty lane of a segment's last slice)
__device__ __forceinline__ int64_t sell_row(const SellMat &m, int64_t s, int lane) {
    if (m.row) return m.row[s * 32 + lane];
    if (s < m.nsl_q) {
        const int64_t r = s * 32 + lane;
        return r < m.nq ? r : -1;
    }
    const int64_t r = m.nq + (s - m.nsl_q) * 32 + lane;
    return r < m.rows ? r : -1;
}

// lane's row . v over the slice [base, base + 32 w): nonzeros in CSR order, U loads in flight
__device__ __forceinline__ double sell_dot(const SellMat &m, int64_t base, int w, int lane,
                                           const double *__restrict__ v, uint64_t pol) {
    double acc = 0.0;
    const double *va = m.val + base + lane;
    const int32_t *ci = m.col + base + lane;
    for (int k0 = 0; k0 < w; k0 += kSellU) {
        int32_t c[kSellU];
        double a[kSellU], x[kSellU];
#pragma unroll
        for (int u = 0; u < kSellU; ++u) {
            const bool ok = k0 + u < w;   // warp-uniform
            c[u] = ok ? sell_ld_i32(ci + (int64_t)(k0 + u) * 32, pol) : 0;
            a[u] = ok ? sell_ld_f64(va + (int64_t)(k0 + u) * 32, pol) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kSellU; ++u) x[u] = k0 + u < w ? __ldg(v + c[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < kSellU; ++u)
            if (k0 + u < w) acc = fma(a[u], x[u], acc);
    }
    return acc;
}

template <int MODE>
__global__ void __launch_bounds__(kSellThreads) k_pass_a_sell(const PassAArgs a) {
    if (a.skip && *a.skip) return;
    const SellMat &m = a.sell;
    const int lane = threadIdx.x & 31;
    // sub-ranges: Q rows only [0, nq), G rows only [nq, rows), or all (segments never share a slice)
    const int64_t s_lo = a.row_begin >= m.nq ? m.nsl_q : 0;
    const int64_t s_hi = a.row_end <= m.nq ? m.nsl_q : m.nsl;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const OuterA o = outer_a(a, MODE);
    const uint64_t pol = sell_evict_first();
    for (int64_t s = s_lo + warp; s < s_hi; s += nwarps) {
        const int64_t r = sell_row(m, s, lane);
        EpiA e{};
        if (r >= 0) e = epi_a_load(a, MODE, r, o);
        const int64_t base = m.sptr[s];
        const int w = (int)((m.sptr[s + 1] - base) >> 5);
        const double acc = sell_dot(m, base, w, lane, a.y, pol);
        if (r >= 0) epi_a_store(a, MODE, r, acc, e, o);
    }
}

template <int MODE>
__global__ void __launch_bounds__(kSellThreads) k_pass_b_sell(const PassBArgs b) {
    if (b.skip && *b.skip) return;
    const SellMat &m = b.sell;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const double avg_w = avg_weight(b, MODE);
    const uint64_t pol = sell_evict_first();
    for (int64_t s = warp; s < m.nsl; s += nwarps) {
        const int64_t j = sell_row(m, s, lane);
        EpiB e{};
        if (j >= 0) e = epi_b_load(b, MODE, j, avg_w);
        const int64_t base = m.sptr[s];
        const int w = (int)((m.sptr[s + 1] - base) >> 5);
        const double t = sell_dot(m, base, w, lane, b.w, pol);
        if (j >= 0) epi_b_store(b, MODE, j, t, e, avg_w);
    }
}

// ------------------------------------------------------------------ layout construction
__global__ void k_row_len(const int32_t *rp, int64_t rows, int32_t *len) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < rows) len[i] = rp[i + 1] - rp[i];
}

// sort keys: (window, -length); windows of `sigma` rows never straddle the two segments
__global__ void k_sort_keys(const int32_t *len, int64_t rows, int64_t nq, int64_t sigma, int64_t *keys) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= rows) return;
    const int64_t wq = (nq + sigma - 1) / sigma;
    const int64_t win = i < nq ? i / sigma : wq + (i - nq) / sigma;
    keys[i] = (win << 32) | (int64_t)(0x7fffffff - len[i]);
}

// row id of every (slice, lane) position from the sorted order (perm[t] = t-th row in sort order)
__global__ void k_slot_rows(const int32_t *perm, int64_t rows, int64_t nq, int64_t nsl_q, int64_t nsl,
                            int32_t *row) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nsl * 32) return;
    const int64_t s = t >> 5, l = t & 31;
    int64_t pos;
    bool ok;
    if (s < nsl_q) {
        pos = s * 32 + l;
        ok = pos < nq;
    } else {
        pos = nq + (s - nsl_q) * 32 + l;
        ok = pos < rows;
    }
    row[t] = ok ? (perm ? perm[pos] : (int32_t)pos) : -1;
}

__global__ void k_slice_width(const int32_t *row, const int32_t *len, int64_t nsl, int64_t *width) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= nsl) return;
    int32_t w = 0;
    for (int l = 0; l < 32; ++l) {
        const int32_t r = row[s * 32 + l];
        if (r >= 0) w = max(w, len[r]);
    }
    width[s] = 32 * (int64_t)w;
}

__global__ void k_sell_fill(const int32_t *rp, const int32_t *ci, const double *va, const int32_t *row,
                            const int64_t *sptr, int64_t nsl, double *sv, int32_t *sc) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nsl * 32) return;
    const int64_t s = t >> 5, l = t & 31;
    const int32_t r = row[t];
    const int32_t b = r >= 0 ? rp[r] : 0, len = r >= 0 ? rp[r + 1] - b : 0;
    const int32_t pad_col = len > 0 ? ci[b + len - 1] : 0;
    const int64_t base = sptr[s], w = (sptr[s + 1] - base) >> 5;
    for (int64_t k = 0; k < w; ++k) {
        sv[base + k * 32 + l] = k < len ? va[b + k] : 0.0;
        sc[base + k * 32 + l] = k < len ? ci[b + k] : pad_col;
    }
}

inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

template <typename T>
cudaError_t zalloc(T **p, int64_t count) {
    *p = nullptr;
    return cudaMalloc((void **)p, (size_t)std::max<int64_t>(count, 2) * sizeof(T));
}

// padded element count of the layout whose slot rows are in `row`
cudaError_t padded_count(const int32_t *row, const int32_t *len, int64_t nsl, int64_t *width, int64_t *total,
                         cudaStream_t s) {
    k_slice_width<<<nblk(std::max<int64_t>(nsl, 1), 256), 256, 0, s>>>(row, len, nsl, width);
    cudaError_t e = cudaGetLastError();
    if (e) return e;
    thrust::device_ptr<int64_t> wp(width);
    *total = nsl > 0 ? thrust::reduce(thrust::cuda::par.on(s), wp, wp + nsl, (int64_t)0) : 0;
    return cudaGetLastError();
}

}  // namespace

void sell_free(SellStore *st) {
    if (st->val) cudaFree(st->val);
    if (st->col) cudaFree(st->col);
    if (st->sptr) cudaFree(st->sptr);
    if (st->row) cudaFree(st->row);
    *st = SellStore{};
}

cudaError_t sell_build(const int32_t *rp, const int32_t *ci, const double *va, int64_t rows, int64_t nq,
                       int64_t nnz, double max_pad, SellStore *out, bool *ok, cudaStream_t s) {
    *ok = false;
    *out = SellStore{};
    const int64_t nsl_q = (nq + 31) / 32, nsl = nsl_q + (rows - nq + 31) / 32;
    if (rows <= 0 || nsl <= 0) return cudaSuccess;
    cudaError_t e;
    int32_t *len = nullptr, *row_id = nullptr, *row_srt = nullptr, *perm = nullptr;
    int64_t *width = nullptr, *keys = nullptr;
    auto cleanup = [&]() {
        for (void *q : {(void *)len, (void *)row_id, (void *)row_srt, (void *)perm, (void *)width, (void *)keys})
            if (q) cudaFree(q);
    };
    if ((e = zalloc(&len, rows)) || (e = zalloc(&row_id, nsl * 32)) || (e = zalloc(&width, nsl + 1))) {
        cleanup();
        return e;
    }
    k_row_len<<<nblk(rows, 256), 256, 0, s>>>(rp, rows, len);
    k_slot_rows<<<nblk(nsl * 32, 256), 256, 0, s>>>(nullptr, rows, nq, nsl_q, nsl, row_id);
    int64_t pad_id = 0, pad_srt = INT64_MAX;
    if ((e = padded_count(row_id, len, nsl, width, &pad_id, s))) {
        cleanup();
        return e;
    }
    // rows of unequal lengths: group them by length inside windows of 1024 rows (32 slices), so a
    // slice's rows have nearly equal lengths; the epilogue's scattered row accesses stay inside a
    // window (32 KB of each n-vector)
    constexpr int64_t kSigma = 1024;
    const bool try_sort = (double)pad_id > 1.05 * (double)nnz + 32.0 * 32.0;
    if (try_sort) {
        if ((e = zalloc(&keys, rows)) || (e = zalloc(&perm, rows)) || (e = zalloc(&row_srt, nsl * 32))) {
            cleanup();
            return e;
        }
        k_sort_keys<<<nblk(rows, 256), 256, 0, s>>>(len, rows, nq, kSigma, keys);
        thrust::device_ptr<int64_t> kp(keys);
        thrust::device_ptr<int32_t> pp(perm);
        thrust::sequence(thrust::cuda::par.on(s), pp, pp + rows);
        thrust::stable_sort_by_key(thrust::cuda::par.on(s), kp, kp + rows, pp);
        k_slot_rows<<<nblk(nsl * 32, 256), 256, 0, s>>>(perm, rows, nq, nsl_q, nsl, row_srt);
        if ((e = padded_count(row_srt, len, nsl, width, &pad_srt, s))) {
            cleanup();
            return e;
        }
    }
    const bool sorted = pad_srt < pad_id;
    const int64_t padded = sorted ? pad_srt : pad_id;
    if ((double)padded > max_pad * (double)nnz + 32.0 * 32.0) {   // too ragged: keep the CSR kernels
        cleanup();
        return cudaGetLastError();
    }
    if (!sorted && (e = padded_count(row_id, len, nsl, width, &pad_id, s))) {   // widths of the kept layout
        cleanup();
        return e;
    }
    SellStore st{};
    st.nsl = nsl;
    st.nsl_q = nsl_q;
    st.nq = nq;
    st.rows = rows;
    st.padded = padded;
    if ((e = zalloc(&st.sptr, nsl + 1)) || (e = zalloc(&st.val, padded)) || (e = zalloc(&st.col, padded))) {
        sell_free(&st);
        cleanup();
        return e;
    }
    {
        thrust::device_ptr<int64_t> wp(width), sp(st.sptr);
        cudaMemsetAsync(width + nsl, 0, sizeof(int64_t), s);
        thrust::exclusive_scan(thrust::cuda::par.on(s), wp, wp + nsl + 1, sp);
    }
    const int32_t *slot_rows = sorted ? row_srt : row_id;
    k_sell_fill<<<nblk(nsl * 32, 256), 256, 0, s>>>(rp, ci, va, slot_rows, st.sptr, nsl, st.val, st.col);
    if ((e = cudaGetLastError())) {
        sell_free(&st);
        cleanup();
        return e;
    }
    if (sorted) {   // keep the slot -> row map; the identity layout computes it
        st.row = row_srt;
        row_srt = nullptr;
    }
    e = cudaStreamSynchronize(s);
    cleanup();
    if (e) {
        sell_free(&st);
        return e;
    }
    *out = st;
    *ok = true;
    return cudaSuccess;
}

SellMat sell_view(const SellStore &st) {
    SellMat m{};
    m.val = st.val;
    m.col = st.col;
    m.sptr = st.sptr;
    m.row = st.row;
    m.nsl = st.nsl;
    m.nsl_q = st.nsl_q;
    m.nq = st.nq;
    m.rows = st.rows;
    return m;
}

int sell_blocks_per_sm(int pass) {
    int b = 0;
    cudaError_t e = pass == 0 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_pass_a_sell<MODE_SOLVE>,
                                                                               kSellThreads, 0)
                              : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_pass_b_sell<MODE_SOLVE>,
                                                                               kSellThreads, 0);
    return e == cudaSuccess && b > 0 ? b : 1;
}

cudaError_t launch_pass_a_sell(const PassAArgs &a, int mode, const LaunchCfg &cfg, cudaStream_t s) {
    if (a.row_end <= a.row_begin) return cudaSuccess;
    if (mode == MODE_SOLVE)
        k_pass_a_sell<MODE_SOLVE><<<cfg.grid, kSellThreads, 0, s>>>(a);
    else
        k_pass_a_sell<MODE_LIN><<<cfg.grid, kSellThreads, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_pass_b_sell(const PassBArgs &b, int mode, const LaunchCfg &cfg, cudaStream_t s) {
    if (b.nrows <= 0) return cudaSuccess;
    if (mode == MODE_SOLVE)
        k_pass_b_sell<MODE_SOLVE><<<cfg.grid, kSellThreads, 0, s>>>(b);
    else
        k_pass_b_sell<MODE_LIN><<<cfg.grid, kSellThreads, 0, s>>>(b);
    return cudaGetLastError();
}

}  // namespace dq
