// Whole-solve persistent kernel for small dense QPs (BASELINE.json configs[0]).
//
// When [Q;G], G' and every vector fit in one SM's shared memory (config 0: 40 KB), the entire
// DFOM solve -- (K_out + 1) x K_in inner steps, each a pass A and a pass B -- runs in ONE CTA:
// the matrices are read from HBM once, every pass is a shared-memory GEMV, and a __syncthreads
// replaces each kernel boundary.  Eight threads per row (a 3-level shuffle instead of a warp-wide
// one, so every pass is spread over up to 32 warps): row r of pass A reads column r of the
// symmetric Q (Q_cr = Q_rc) or column r-n of G', pass B column j of G; the 8 threads of a
// row take every 8th column.  Shared-memory rows are padded by 4 doubles, so the 8 column groups
// of a warp fall on different banks.  The epilogues are the shared ones (epilogue.cuh); the
// summation order differs from the streaming kernels (agreement ~1e-15).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "duquad_internal.h"
#include "epilogue.cuh"

namespace dq {

namespace {

constexpr int kSmallThreads = 1024;

constexpr int kTpr = 8;   // threads per row
constexpr int kPad = 4;   // doubles of padding per shared-memory row

// this thread's part of sum_c M[c * ldm + col] v[c], c < len: every kTpr-th c from `sub`, two
// interleaved accumulators
__device__ __forceinline__ double col_part(const double *M, int ldm, int col, const double *v, int len, int sub) {
    double a0 = 0.0, a1 = 0.0;
    int c = sub;
    for (; c + kTpr < len; c += 2 * kTpr) {
        a0 = fma(M[c * ldm + col], v[c], a0);
        a1 = fma(M[(c + kTpr) * ldm + col], v[c + kTpr], a1);
    }
    if (c < len) a0 = fma(M[c * ldm + col], v[c], a0);
    return a0 + a1;
}

// sum over the kTpr threads of a row (fixed xor tree); every lane of the warp must call it
__device__ __forceinline__ double row_sum8(double s) {
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    return s;
}

__device__ __forceinline__ void copy_rows(double *dst, int ldd, const double *src, int64_t lds, int64_t rows,
                                          int64_t cols) {
    for (int64_t t = threadIdx.x; t < rows * cols; t += blockDim.x) {
        const int64_t r = t / cols, c = t - r * cols;
        dst[r * ldd + c] = src[r * lds + c];
    }
}

__global__ void __launch_bounds__(kSmallThreads, 1) k_small_solve(const SmallArgs sa) {
    extern __shared__ __align__(16) double sm[];
    const int64_t n = sa.n, p = sa.p, ld = sa.ld, ldp = sa.ldp, rows = n + p;
    // shared-memory carve-up (all offsets multiples of 2 doubles)
    const int lda = (int)ld + kPad, ldg = (int)ldp + kPad;   // padded shared-memory strides
    double *A = sm;                       // rows x lda
    double *GT = A + rows * lda;          // n x ldg
    double *y = GT + n * ldg;             // ld
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
    double *beta = lp + p2;               // Kin + 1 (rounded to even): inner momentum table
    const int64_t kb2 = (sa.Kin + 2) & ~1LL;
    OuterParam *ops = reinterpret_cast<OuterParam *>(beta + kb2);   // K + 2 per-outer scalars
    uint8_t *cone = reinterpret_cast<uint8_t *>(ops + sa.K + 2);
    __shared__ int32_t jj;

    copy_rows(A, lda, sa.A, ld, rows, n);
    if (p > 0) copy_rows(GT, ldg, sa.GT, ldp, n, p);
    for (int64_t i = threadIdx.x; i < ld; i += blockDim.x) y[i] = 0.0;
    for (int64_t i = threadIdx.x; i < (ldp > 2 ? ldp : 2); i += blockDim.x) w[i] = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double x0 = fmin(fmax(sa.x_init ? sa.x_init[i] : 0.0, sa.lb[i]), sa.ub[i]);   // [0]_U (c7) or warm start
        x[i] = x0;
        y[i] = x0;
        xh[i] = 0.0;
        q[i] = sa.q[i];
        lb[i] = sa.lb[i];
        ub[i] = sa.ub[i];
    }
    for (int64_t k = threadIdx.x; k < p; k += blockDim.x) {
        g[k] = sa.g[k];
        mu[k] = sa.lam_init ? sa.lam_init[k] : 0.0;   // mu^1 = lambda^0 = 0, or the warm start
        lp[k] = mu[k];
        cone[k] = sa.cone[k];
    }
    for (int i = threadIdx.x; i <= sa.Kin; i += blockDim.x) beta[i] = sa.beta_in[i];
    for (int i = threadIdx.x; i < sa.K + 2; i += blockDim.x) ops[i] = sa.a.ops[i];
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
    a.ops = ops;
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
    b.ops = ops;

    const double *Gm = A + n * lda;   // G rows of the packed [Q;G]
    const int sub = threadIdx.x % kTpr, unit0 = threadIdx.x / kTpr, nunit = blockDim.x / kTpr;
    const int ni = (int)n, pi = (int)p, rowsi = (int)rows;
    for (int j = 1; j <= sa.K + 1; ++j) {
        for (int k = 1; k <= sa.Kin; ++k) {
            a.first_inner = (k == 1);
            const OuterA o = outer_a(a, MODE_SOLVE);
            // pass A: kTpr threads per row (the loop bound is uniform over a row's threads)
            for (int base = 0; base < rowsi; base += nunit) {
                const int row = base + unit0;
                double s = 0.0;
                if (row < ni) s = col_part(A, lda, row, y, ni, sub);                      // (Q y)_row, Q symmetric
                else if (row < rowsi) s = col_part(GT, ldg, row - ni, y, ni, sub);         // (G y)_{row-n} via G'
                s = row_sum8(s);   // all lanes (converged)
                if (sub == 0 && row < rowsi) {
                    const EpiA e = epi_a_load(a, MODE_SOLVE, row, o);
                    epi_a_store(a, MODE_SOLVE, row, s, e, o);
                }
            }
            __syncthreads();
            if (k == 1 && j >= 2 && sa.trace_lam && j - 2 < sa.trace_max)
                for (int64_t i = threadIdx.x; i < p; i += blockDim.x) sa.trace_lam[(j - 2) * p + i] = lp[i];
            b.beta_in = beta[k];
            b.last_inner = (k == sa.Kin);
            const double avg_w = avg_weight(b, MODE_SOLVE);
            for (int base = 0; base < ni; base += nunit) {                                  // pass B
                const int r = base + unit0;
                const double t = row_sum8((r < ni && pi > 0) ? col_part(Gm, lda, r, w, pi, sub) : 0.0);
                if (sub == 0 && r < ni) {
                    const EpiB e = epi_b_load(b, MODE_SOLVE, r, avg_w);
                    epi_b_store(b, MODE_SOLVE, r, t, e, avg_w);
                }
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

size_t small_smem_bytes(int64_t n, int64_t p, int64_t ld, int64_t ldp, int K, int Kin) {
    const int64_t n2 = (n + 1) & ~1LL, p2 = (p + 1) & ~1LL, kb2 = ((int64_t)Kin + 2) & ~1LL;
    const int64_t doubles = (n + p) * (ld + kPad) + n * (ldp + kPad) + ld + (ldp > 2 ? ldp : 2) + 6 * n2 + 3 * p2 + kb2;
    return (size_t)doubles * 8 + (size_t)(K + 2) * sizeof(OuterParam) + (size_t)p + 16;
}

cudaError_t configure_small_kernel(size_t smem) {
    return cudaFuncSetAttribute(k_small_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

cudaError_t launch_small_solve(const SmallArgs &sa, size_t smem, cudaStream_t s) {
    // kTpr threads per row of the larger pass ([Q;G]: n + p rows), whole warps, at most 1024: warps
    // that would own no row of either pass only add issue slots and barrier arrivals (config 0:
    // 600 of 1024 threads busy in pass A); the per-row arithmetic does not depend on the block size
    const int64_t need = ((sa.n + sa.p) * kTpr + 31) / 32 * 32;
    const int threads = (int)std::min<int64_t>(kSmallThreads, std::max<int64_t>(32, need));
    k_small_solve<<<1, threads, smem, s>>>(sa);
    return cudaGetLastError();
}

}  // namespace dq
