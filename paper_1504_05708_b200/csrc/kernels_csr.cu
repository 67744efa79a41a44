// CSR sm_100a kernels of the DuQuad hot path (config 4).
//
// Same two passes and the same epilogues (epilogue.cuh) as the dense path, with
// the row products done as SpMV: a group of GS lanes owns a row (GS a power of
// two chosen from the mean nnz per row), lanes stride its nonzeros, the group
// reduces with a fixed xor-shuffle tree.  Values and column indices are
// streamed with L1-bypassing, L2-evict-first loads; the dense vector (y for
// pass A, w for pass B; 8 MB / 4 MB at config 4) is gathered through L1/L2
// and stays resident in the 126 MB L2.  The paper notes this is where the
// method is cheap ("only sparse matrix-vector products").
#include <cuda_runtime.h>
#include <thrust/binary_search.h>
#include <thrust/device_ptr.h>
#include <thrust/execution_policy.h>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>
#include <thrust/sort.h>

#include <algorithm>

#include "duquad_internal.h"
#include "epilogue.cuh"

namespace dq {

namespace {

constexpr int kCsrThreads = 256;

__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ double ld_stream_f64(const double *p, uint64_t pol) {
    double r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ int32_t ld_stream_i32(const int32_t *p, uint64_t pol) {
    int32_t r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}

template <int GS>
__device__ __forceinline__ double csr_row_dot(const int32_t *__restrict__ ci, const double *__restrict__ va,
                                              const double *__restrict__ v, int32_t lo, int32_t hi, int gl) {
    // 4 nonzeros per lane per round: all index/value loads issued, then all gathers, then the
    // FMAs in nonzero order (same per-lane summation order as a plain loop)
    constexpr int U = 4;
    const uint64_t pol = evict_first_policy();
    double s = 0.0;
    for (int32_t e0 = lo + gl; e0 < hi; e0 += U * GS) {
        int32_t c[U];
        double a[U], x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t e = e0 + u * GS;
            const bool ok = e < hi;
            c[u] = ok ? ld_stream_i32(ci + e, pol) : -1;
            a[u] = ok ? ld_stream_f64(va + e, pol) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = c[u] >= 0 ? __ldg(v + c[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (c[u] >= 0) s = fma(a[u], x[u], s);
    }
    return s;
}

// Two rows per lane group per round, their loads interleaved (latency of the row-pointer ->
// index -> gather chain is the limiter of a memory-bound SpMV, not bandwidth).  Each row keeps
// the summation order of csr_row_dot.
template <int GS>
__device__ __forceinline__ void csr_row_dot2(const int32_t *__restrict__ ci, const double *__restrict__ va,
                                             const double *__restrict__ v, int32_t lo0, int32_t hi0, int32_t lo1,
                                             int32_t hi1, int gl, double &s0, double &s1) {
    constexpr int U = 4;
    const uint64_t pol = evict_first_policy();
    s0 = 0.0;
    s1 = 0.0;
    for (int32_t e0 = lo0 + gl, e1 = lo1 + gl; e0 < hi0 || e1 < hi1; e0 += U * GS, e1 += U * GS) {
        int32_t c0[U], c1[U];
        double a0[U], a1[U], x0[U], x1[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t f0 = e0 + u * GS, f1 = e1 + u * GS;
            c0[u] = f0 < hi0 ? ld_stream_i32(ci + f0, pol) : -1;
            c1[u] = f1 < hi1 ? ld_stream_i32(ci + f1, pol) : -1;
            a0[u] = f0 < hi0 ? ld_stream_f64(va + f0, pol) : 0.0;
            a1[u] = f1 < hi1 ? ld_stream_f64(va + f1, pol) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            x0[u] = c0[u] >= 0 ? __ldg(v + c0[u]) : 0.0;
            x1[u] = c1[u] >= 0 ? __ldg(v + c1[u]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (c0[u] >= 0) s0 = fma(a0[u], x0[u], s0);
            if (c1[u] >= 0) s1 = fma(a1[u], x1[u], s1);
        }
    }
}

template <int MODE, int GS>
// (kCsrThreads, 4): <= 64 registers, 4 resident CTAs per SM (was 3 at 76): more rows in flight
__global__ void __launch_bounds__(kCsrThreads, 4) k_pass_a_csr(const PassAArgs a) {
    pdl_wait();   // everything below reads iterates or writes (PDL, epilogue.cuh)
    pdl_trigger();
    if (a.skip && *a.skip) return;
    const int lane = threadIdx.x & 31, gl = lane & (GS - 1), gw = lane / GS;
    const int64_t gpw = 32 / GS;   // lane groups per warp; a warp covers 2 * gpw consecutive rows
    const int64_t warp_id = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
    const int64_t rows = a.row_end - a.row_begin;
    const OuterA o = outer_a(a, MODE);
    for (int64_t base = warp_id * 2 * gpw; base < rows; base += nwarps * 2 * gpw) {
        const int64_t i0 = base + gw, i1 = base + gpw + gw;
        const bool v0 = i0 < rows, v1 = i1 < rows;
        const int64_t r0 = a.row_begin + i0, r1 = a.row_begin + i1;
        EpiA e0{}, e1{};
        if (gl == 0) {
            if (v0) e0 = epi_a_load(a, MODE, r0, o);
            if (v1) e1 = epi_a_load(a, MODE, r1, o);
        }
        double s0, s1;
        csr_row_dot2<GS>(a.ci, a.va, a.y, v0 ? a.rp[r0] : 0, v0 ? a.rp[r0 + 1] : 0, v1 ? a.rp[r1] : 0,
                         v1 ? a.rp[r1 + 1] : 0, gl, s0, s1);
        s0 = group_sum<GS>(s0);
        s1 = group_sum<GS>(s1);
        if (gl == 0) {
            if (v0) epi_a_store(a, MODE, r0, s0, e0, o);
            if (v1) epi_a_store(a, MODE, r1, s1, e1, o);
        }
    }
}

template <int MODE, int GS>
__global__ void __launch_bounds__(kCsrThreads) k_pass_b_csr(const PassBArgs b) {
    pdl_wait();
    pdl_trigger();
    if (b.skip && *b.skip) return;
    const int lane = threadIdx.x & 31, gl = lane & (GS - 1), gw = lane / GS;
    const int64_t gpw = 32 / GS;
    const int64_t warp_id = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
    const double avg_w = avg_weight(b, MODE);
    // G' rows are short (config 4: Poisson(4) nonzeros): one row per lane group measured faster
    const int64_t stride = nwarps * gpw;
    int64_t base = warp_id * gpw;
    int32_t lo = 0, hi = 0, lon = 0, hin = 0;
    if (base + gw < b.nrows) {
        lo = b.rp[base + gw];
        hi = b.rp[base + gw + 1];
    }
    for (; base < b.nrows; base += stride) {
        const int64_t j = base + gw;
        const bool valid = j < b.nrows;
        if (base + stride + gw < b.nrows) {   // next iteration's row pointers, one iteration ahead
            lon = b.rp[base + stride + gw];
            hin = b.rp[base + stride + gw + 1];
        }
        EpiB e{};
        double t = 0.0;
        if (valid) {
            if (gl == 0) e = epi_b_load(b, MODE, j, avg_w);
            t = csr_row_dot<GS>(b.ci, b.va, b.w, lo, hi, gl);
        }
        t = group_sum<GS>(t);
        if (valid && gl == 0) epi_b_store(b, MODE, j, t, e, avg_w);
        lo = lon;
        hi = hin;
    }
}

template <typename K>
int occ(K kern) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, kCsrThreads, 0) != cudaSuccess || b < 1) b = 1;
    return b;
}

template <int MODE>
cudaError_t dispatch_a(const PassAArgs &a, const LaunchCfg &cfg, cudaStream_t s) {
    switch (a.gs) {
        case 2: return launch_ex(k_pass_a_csr<MODE, 2>, cfg.grid, kCsrThreads, 0, s, cfg.pdl, 0, a);
        case 4: return launch_ex(k_pass_a_csr<MODE, 4>, cfg.grid, kCsrThreads, 0, s, cfg.pdl, 0, a);
        case 8: return launch_ex(k_pass_a_csr<MODE, 8>, cfg.grid, kCsrThreads, 0, s, cfg.pdl, 0, a);
        case 16: return launch_ex(k_pass_a_csr<MODE, 16>, cfg.grid, kCsrThreads, 0, s, cfg.pdl, 0, a);
        default: return launch_ex(k_pass_a_csr<MODE, 32>, cfg.grid, kCsrThreads, 0, s, cfg.pdl, 0, a);
    }
    return cudaGetLastError();
}

template <int MODE>
cudaError_t dispatch_b(const PassBArgs &b, const LaunchCfg &cfg, cudaStream_t s) {
    switch (b.gs) {
        case 2: return launch_ex(k_pass_b_csr<MODE, 2>, cfg.grid, kCsrThreads, 0, s, cfg.pdl, 0, b);
        case 4: return launch_ex(k_pass_b_csr<MODE, 4>, cfg.grid, kCsrThreads, 0, s, cfg.pdl, 0, b);
        case 8: return launch_ex(k_pass_b_csr<MODE, 8>, cfg.grid, kCsrThreads, 0, s, cfg.pdl, 0, b);
        case 16: return launch_ex(k_pass_b_csr<MODE, 16>, cfg.grid, kCsrThreads, 0, s, cfg.pdl, 0, b);
        default: return launch_ex(k_pass_b_csr<MODE, 32>, cfg.grid, kCsrThreads, 0, s, cfg.pdl, 0, b);
    }
    return cudaGetLastError();
}

__global__ void k_rebase(int32_t *dst, const int32_t *src, int64_t count, int32_t sub, int32_t add) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < count) dst[i] = src[i] - sub + add;
}

__global__ void k_check_csr(const int32_t *rp, const int32_t *ci, const double *va, int64_t rows, int64_t cols,
                            int64_t nnz, int32_t *flag) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t0 == 0 && (rp[0] != 0 || rp[rows] != nnz)) *flag = 1;
    for (int64_t i = t0; i < rows; i += stride)
        if (rp[i] > rp[i + 1]) *flag = 1;
    for (int64_t e = t0; e < nnz; e += stride)
        if (ci[e] < 0 || ci[e] >= cols || !isfinite(va[e])) *flag = 1;
}

// Q and its transpose T (both sorted CSR, same nnz): identical row pointers and column indices,
// values equal to 1e-12 relative (the dense path's k_check_sym tolerance)
__global__ void k_csr_sym_cmp(const int32_t *rp, const int32_t *ci, const double *va, const int32_t *trp,
                              const int32_t *tci, const double *tva, int64_t rows, int64_t nnz, int32_t *flag) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (int64_t i = t0; i <= rows; i += stride)
        if (rp[i] != trp[i]) *flag = 3;
    for (int64_t e = t0; e < nnz; e += stride) {
        const double a = va[e], b = tva[e];
        if (ci[e] != tci[e] || fabs(a - b) > 1e-12 * (fabs(a) + fabs(b))) *flag = 3;
    }
}

__global__ void k_expand_rows(const int32_t *rp, int64_t rows, int64_t *keys, const int32_t *ci) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= rows) return;
    for (int32_t e = rp[r]; e < rp[r + 1]; ++e) keys[e] = (int64_t)ci[e] * rows + r;   // (column, row)
}

__global__ void k_split_keys(const int64_t *keys, int64_t rows, int64_t nnz, int32_t *ci_t) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e < nnz) ci_t[e] = (int32_t)(keys[e] % rows);
}

struct TimesRows {
    int64_t rows, c0;
    __host__ __device__ int64_t operator()(int64_t j) const { return (c0 + j) * rows; }
};

__global__ void k_sub_i64_to_i32(const int64_t *src, int64_t count, int64_t sub, int32_t *dst) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < count) dst[i] = (int32_t)(src[i] - sub);
}

inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

}  // namespace

// resident CTAs per SM of the solve-mode pass kernels for group size gs (the grid is sized to whole
// waves: a grid-stride loop over rows, so a partial last wave would idle SMs)
int csr_blocks_per_sm(int pass, int gs) {
    if (pass == 0) {
        switch (gs) {
            case 2: return occ(k_pass_a_csr<MODE_SOLVE, 2>);
            case 4: return occ(k_pass_a_csr<MODE_SOLVE, 4>);
            case 8: return occ(k_pass_a_csr<MODE_SOLVE, 8>);
            case 16: return occ(k_pass_a_csr<MODE_SOLVE, 16>);
            default: return occ(k_pass_a_csr<MODE_SOLVE, 32>);
        }
    }
    switch (gs) {
        case 2: return occ(k_pass_b_csr<MODE_SOLVE, 2>);
        case 4: return occ(k_pass_b_csr<MODE_SOLVE, 4>);
        case 8: return occ(k_pass_b_csr<MODE_SOLVE, 8>);
        case 16: return occ(k_pass_b_csr<MODE_SOLVE, 16>);
        default: return occ(k_pass_b_csr<MODE_SOLVE, 32>);
    }
}

int csr_group_size(double m) {
    int gs = 2;
    while (gs < 32 && gs * 3 < m) gs *= 2;
    return gs;
}

cudaError_t launch_pass_a_csr(const PassAArgs &a, int mode, const LaunchCfg &cfg, cudaStream_t s) {
    if (a.row_end <= a.row_begin) return cudaSuccess;
    return mode == MODE_SOLVE ? dispatch_a<MODE_SOLVE>(a, cfg, s) : dispatch_a<MODE_LIN>(a, cfg, s);
}

cudaError_t launch_pass_b_csr(const PassBArgs &b, int mode, const LaunchCfg &cfg, cudaStream_t s) {
    if (b.nrows <= 0) return cudaSuccess;
    return mode == MODE_SOLVE ? dispatch_b<MODE_SOLVE>(b, cfg, s) : dispatch_b<MODE_LIN>(b, cfg, s);
}

cudaError_t launch_rebase(int32_t *dst, const int32_t *src, int64_t count, int32_t sub, int32_t add,
                          cudaStream_t s) {
    if (count <= 0) return cudaSuccess;
    k_rebase<<<nblk(count, 256), 256, 0, s>>>(dst, src, count, sub, add);
    return cudaGetLastError();
}

cudaError_t launch_check_csr(const int32_t *rp, const int32_t *ci, const double *va, int64_t rows,
                             int64_t cols, int64_t nnz, int32_t *flag, cudaStream_t s) {
    k_check_csr<<<592, 256, 0, s>>>(rp, ci, va, rows, cols, nnz, flag);
    return cudaGetLastError();
}

cudaError_t launch_csr_sym_cmp(const int32_t *rp, const int32_t *ci, const double *va, const int32_t *trp,
                               const int32_t *tci, const double *tva, int64_t rows, int64_t nnz, int32_t *flag,
                               cudaStream_t s) {
    k_csr_sym_cmp<<<592, 256, 0, s>>>(rp, ci, va, trp, tci, tva, rows, nnz, flag);
    return cudaGetLastError();
}

cudaError_t csr_transpose_rows(const int32_t *rp, const int32_t *ci, const double *va, int64_t rows,
                               int64_t cols, int64_t nnz, int64_t c0, int64_t nc, int32_t **rp_t,
                               int32_t **ci_t, double **va_t, int64_t *nnz_t, cudaStream_t s) {
    (void)cols;
    cudaError_t e;
    *rp_t = nullptr;
    *ci_t = nullptr;
    *va_t = nullptr;
    *nnz_t = 0;
    if ((e = cudaMalloc(rp_t, (nc + 1) * sizeof(int32_t)))) return e;
    if (nnz == 0 || nc == 0) {
        cudaMemsetAsync(*rp_t, 0, (nc + 1) * sizeof(int32_t), s);
        if ((e = cudaMalloc(ci_t, 8))) return e;
        return cudaMalloc(va_t, 8);
    }
    int64_t *keys = nullptr, *bounds = nullptr;
    double *vals = nullptr;
    if ((e = cudaMalloc(&keys, nnz * sizeof(int64_t)))) return e;
    if ((e = cudaMalloc(&vals, nnz * sizeof(double)))) return e;
    if ((e = cudaMalloc(&bounds, (nc + 1) * sizeof(int64_t)))) return e;
    k_expand_rows<<<nblk(rows, 256), 256, 0, s>>>(rp, rows, keys, ci);
    cudaMemcpyAsync(vals, va, nnz * sizeof(double), cudaMemcpyDeviceToDevice, s);
    thrust::device_ptr<int64_t> kp(keys);
    thrust::device_ptr<double> vp(vals);
    thrust::sort_by_key(thrust::cuda::par.on(s), kp, kp + nnz, vp);   // keys unique: deterministic
    auto search = thrust::make_transform_iterator(thrust::counting_iterator<int64_t>(0), TimesRows{rows, c0});
    thrust::device_ptr<int64_t> bp(bounds);
    thrust::lower_bound(thrust::cuda::par.on(s), kp, kp + nnz, search, search + (nc + 1), bp);
    int64_t lo = 0, hi = 0;
    cudaMemcpyAsync(&lo, bounds, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(&hi, bounds + nc, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
    if ((e = cudaStreamSynchronize(s))) return e;
    const int64_t cnt = hi - lo;
    k_sub_i64_to_i32<<<nblk(nc + 1, 256), 256, 0, s>>>(bounds, nc + 1, lo, *rp_t);
    if ((e = cudaMalloc(ci_t, std::max<int64_t>(cnt, 1) * sizeof(int32_t)))) return e;
    if ((e = cudaMalloc(va_t, std::max<int64_t>(cnt, 1) * sizeof(double)))) return e;
    if (cnt > 0) {
        k_split_keys<<<nblk(cnt, 256), 256, 0, s>>>(keys + lo, rows, cnt, *ci_t);
        cudaMemcpyAsync(*va_t, vals + lo, cnt * sizeof(double), cudaMemcpyDeviceToDevice, s);
    }
    e = cudaStreamSynchronize(s);
    cudaFree(keys);
    cudaFree(vals);
    cudaFree(bounds);
    *nnz_t = cnt;
    if (e) return e;
    return cudaGetLastError();
}

}  // namespace dq
