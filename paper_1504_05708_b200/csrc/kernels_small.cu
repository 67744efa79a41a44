// Whole-solve persistent kernel for small dense QPs (BASELINE.json configs[0]).
//
// When [Q;G], G' and every vector fit in one SM's shared memory (config 0: 40 KB), the entire
// DFOM solve -- (K_out + 1) x K_in inner steps, each a pass A and a pass B -- runs in ONE CTA:
// the matrices are read from HBM once, every pass is a shared-memory GEMV, and a __syncthreads
// replaces each kernel boundary (≈0.5 µs per inner step instead of two launches).  The row dot
// product has the same summation order as the streaming dense kernels (kernels_dense.cu) and the
// epilogues are the shared ones (epilogue.cuh), so the result is bit-identical to the
// multi-launch dense path.
#include <cuda_runtime.h>
#include <stdint.h>

#include "duquad_internal.h"
#include "epilogue.cuh"

namespace dq {

namespace {

constexpr int kSmallThreads = 1024;
constexpr int kUnrollS = 8;   // must match kUnroll of kernels_dense.cu (summation order)

// identical arithmetic to row_dot() of kernels_dense.cu, operands in shared memory
__device__ __forceinline__ double row_dot_smem(const double2 *row, const double2 *sv, int nv2, int lane) {
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
    int c = lane;
    for (; c + 32 * (kUnrollS - 1) < nv2; c += 32 * kUnrollS) {
#pragma unroll
        for (int u = 0; u < kUnrollS; u += 2) {
            const double2 v0 = row[c + 32 * u], v1 = row[c + 32 * (u + 1)];
            const double2 y0 = sv[c + 32 * u], y1 = sv[c + 32 * (u + 1)];
            acc0 = fma(v0.x, y0.x, acc0);
            acc1 = fma(v0.y, y0.y, acc1);
            acc2 = fma(v1.x, y1.x, acc2);
            acc3 = fma(v1.y, y1.y, acc3);
        }
    }
    for (; c < nv2; c += 32) {
        const double2 v = row[c], y0 = sv[c];
        acc0 = fma(v.x, y0.x, acc0);
        acc1 = fma(v.y, y0.y, acc1);
    }
    return warp_sum((acc0 + acc1) + (acc2 + acc3));
}

__device__ __forceinline__ void copy_in(double *dst, const double *src, int64_t count) {
    for (int64_t i = threadIdx.x; i < count; i += blockDim.x) dst[i] = src[i];
}

__global__ void __launch_bounds__(kSmallThreads, 1) k_small_solve(const SmallArgs sa) {
    extern __shared__ __align__(16) double sm[];
    const int64_t n = sa.n, p = sa.p, ld = sa.ld, ldp = sa.ldp, rows = n + p;
    // shared-memory carve-up (all offsets multiples of 2 doubles)
    double *A = sm;                       // rows x ld
    double *GT = A + rows * ld;           // n x ldp
    double *y = GT + n * ldp;             // ld
    double *w = y + ld;                   // max(ldp, 2)
    double *x = w + (ldp > 2 ? ldp : 2);  // n (rounded to even)
    const int64_t n2 = (n + 1) & ~1LL, p2 = (p + 1) & ~1LL;
    double *xh = x + n2;
    double *qy = xh + n2;
    double *q = qy + n2;
    double *lb = q + n2;
    double *ub = lb + n2;
    double *g = ub + n2;
    double *mu = g + p2;
    double *lp = mu + p2;
    uint8_t *cone = reinterpret_cast<uint8_t *>(lp + p2);
    __shared__ int32_t jj;

    copy_in(A, sa.A, rows * ld);
    copy_in(GT, sa.GT, n * ldp);
    for (int64_t i = threadIdx.x; i < ld; i += blockDim.x) y[i] = 0.0;
    for (int64_t i = threadIdx.x; i < (ldp > 2 ? ldp : 2); i += blockDim.x) w[i] = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double x0 = fmin(fmax(0.0, sa.lb[i]), sa.ub[i]);   // u_bar^0 = [0]_U (reading c7)
        x[i] = x0;
        y[i] = x0;
        xh[i] = 0.0;
        q[i] = sa.q[i];
        lb[i] = sa.lb[i];
        ub[i] = sa.ub[i];
    }
    for (int64_t k = threadIdx.x; k < p; k += blockDim.x) {
        g[k] = sa.g[k];
        mu[k] = 0.0;   // mu^1 = lambda^0 = 0
        lp[k] = 0.0;
        cone[k] = sa.cone[k];
    }
    if (threadIdx.x == 0) jj = 1;
    __syncthreads();

    PassAArgs a = sa.a;   // scalars from the host; pointers re-aimed at shared memory
    a.A = A;
    a.y = y;
    a.qy = qy;
    a.w = w;
    a.g = g;
    a.mu = mu;
    a.lam_prev = lp;
    a.cone = cone;
    a.d_j = &jj;
    PassBArgs b = sa.b;
    b.w = w;
    b.qy = qy;
    b.q = q;
    b.lb = lb;
    b.ub = ub;
    b.x = x;
    b.y = y;
    b.xhat = xh;
    b.d_j = &jj;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int nw = kSmallThreads / 32;
    const int nv2a = (int)(ld >> 1), nv2b = (int)(ldp >> 1);
    for (int j = 1; j <= sa.K + 1; ++j) {
        for (int k = 1; k <= sa.Kin; ++k) {
            a.first_inner = (k == 1);
            const OuterA o = outer_a(a, MODE_SOLVE);
            for (int64_t row = warp; row < rows; row += nw) {
                const EpiA e = epi_a_load(a, MODE_SOLVE, row, o);
                const double s = row_dot_smem(reinterpret_cast<const double2 *>(A + row * ld),
                                              reinterpret_cast<const double2 *>(y), nv2a, lane);
                if (lane == 0) epi_a_store(a, MODE_SOLVE, row, s, e, o);
            }
            __syncthreads();
            if (k == 1 && j >= 2 && sa.trace_lam && j - 2 < sa.trace_max)
                for (int64_t i = threadIdx.x; i < p; i += blockDim.x) sa.trace_lam[(j - 2) * p + i] = lp[i];
            b.beta_in = sa.beta_in[k];
            b.last_inner = (k == sa.Kin);
            const double avg_w = avg_weight(b, MODE_SOLVE);
            for (int64_t r = warp; r < n; r += nw) {
                const EpiB e = epi_b_load(b, MODE_SOLVE, r, avg_w);
                const double t = nv2b > 0 ? row_dot_smem(reinterpret_cast<const double2 *>(GT + r * ldp),
                                                         reinterpret_cast<const double2 *>(w), nv2b, lane)
                                          : 0.0;
                if (lane == 0) epi_b_store(b, MODE_SOLVE, r, t, e, avg_w);
            }
            __syncthreads();
        }
        if (sa.trace_u && j <= sa.K && j - 1 < sa.trace_max)
            for (int64_t i = threadIdx.x; i < n; i += blockDim.x) sa.trace_u[(j - 1) * n + i] = x[i];
        if (threadIdx.x == 0) jj = j + 1;
        __syncthreads();
    }
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        sa.x_out[i] = x[i];
        sa.xhat_out[i] = xh[i];
        sa.y_out[i] = y[i];
    }
    for (int64_t k = threadIdx.x; k < p; k += blockDim.x) {
        sa.lam_out[k] = lp[k];
        sa.mu_out[k] = mu[k];
    }
}

}  // namespace

size_t small_smem_bytes(int64_t n, int64_t p, int64_t ld, int64_t ldp) {
    const int64_t n2 = (n + 1) & ~1LL, p2 = (p + 1) & ~1LL;
    const int64_t doubles = (n + p) * ld + n * ldp + ld + (ldp > 2 ? ldp : 2) + 6 * n2 + 3 * p2;
    return (size_t)doubles * 8 + (size_t)p + 16;
}

cudaError_t configure_small_kernel(size_t smem) {
    return cudaFuncSetAttribute(k_small_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

cudaError_t launch_small_solve(const SmallArgs &sa, size_t smem, cudaStream_t s) {
    k_small_solve<<<1, kSmallThreads, smem, s>>>(sa);
    return cudaGetLastError();
}

}  // namespace dq
