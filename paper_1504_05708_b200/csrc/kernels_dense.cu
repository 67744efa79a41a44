// Dense sm_100a kernels of the DuQuad hot path.
//
// Pass A (K1): one streaming pass over the row-stacked [Q;G] (HBM-bound GEMV)
//   Q rows -> Qy;  G rows -> w = [mu + rho (G y + g)]_{K polar}  (grad of (auglag1),
//   PAPER.md:243-251), and on the first inner step of an outer iteration the
//   fused DFOM dual step lambda = [mu + step (r - s)]_{K_d}, mu <- lambda + beta (lambda - lambda_prev)
//    -- all row-local, so no extra matrix pass.
// Pass B (K2): one streaming pass over the stored G' (n x p)
//   t = G'w; grad = Qy + q + t; x+ = [y - grad/L]_U;
//   y+ = x+ + beta (x+ - x); running primal average on the last inner step.
//
// Design: persistent grid of one CTA per SM; the dense vector
// (y for pass A, w for pass B) is staged once into shared memory; each warp
// owns whole rows and streams them with 128-bit L1-bypassing loads, U loads in
// flight per lane; row reduction by a fixed xor-shuffle tree, so every row's
// value is independent of the grid and of the sharding (bitwise reproducible).

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>

#include "duquad_internal.h"
#include "epilogue.cuh"

namespace dq {

namespace {

constexpr int kThreads = 512;  // threads per CTA of the pass kernels
constexpr int kUnroll = 16;    // 16-byte loads in flight per lane per row chunk

__device__ __forceinline__ double2 ldg_stream(const double2 *p) {
    double2 r;
    asm("ld.global.nc.L1::no_allocate.L2::256B.v2.f64 {%0, %1}, [%2];"
        : "=d"(r.x), "=d"(r.y)
        : "l"(p));
    return r;
}

// Dot product of one matrix row (nv2 double2 entries, 16-byte aligned) with a
// shared-memory vector; fixed summation order for a given nv2.  Every chunk, the ragged last one
// included, issues its kUnroll loads together (predicated, zeros past the row end: fma(0, 0, acc)
// = acc exactly), so a row costs ceil(nv2 / (32 kUnroll)) memory round trips.
__device__ __forceinline__ double row_dot(const double2 *__restrict__ row,
                                          const double2 *__restrict__ sv, int nv2, int lane) {
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
    for (int c = lane; c - lane < nv2; c += 32 * kUnroll) {
        double2 v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
            v[u] = c + 32 * u < nv2 ? ldg_stream(row + c + 32 * u) : make_double2(0.0, 0.0);
#pragma unroll
        for (int u = 0; u < kUnroll; u += 2) {
            const double2 y0 = c + 32 * u < nv2 ? sv[c + 32 * u] : make_double2(0.0, 0.0);
            const double2 y1 = c + 32 * (u + 1) < nv2 ? sv[c + 32 * (u + 1)] : make_double2(0.0, 0.0);
            acc0 = fma(v[u].x, y0.x, acc0);
            acc1 = fma(v[u].y, y0.y, acc1);
            acc2 = fma(v[u + 1].x, y1.x, acc2);
            acc3 = fma(v[u + 1].y, y1.y, acc3);
        }
    }
    return warp_sum((acc0 + acc1) + (acc2 + acc3));
}

// The same row dot with its first chunk already in registers (v, loaded by chunk_load), and the
// next row's first chunk loaded into v after the last FMA of this row (next != nullptr): the
// matrix stream of a warp's next row, or of its first row before griddepcontrol.wait (the stored
// matrices are written by no kernel of a solve, epilogue.cuh), is in flight while this row's
// butterfly, epilogue and the y / w staging run.  Same loads, FMAs and order as row_dot: bitwise
// the same row value.
__device__ __forceinline__ void chunk_load(const double2 *__restrict__ row, int c, int nv2, double2 (&v)[kUnroll]) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
        v[u] = c + 32 * u < nv2 ? ldg_stream(row + c + 32 * u) : make_double2(0.0, 0.0);
}

__device__ __forceinline__ double row_dot_pre(const double2 *__restrict__ row, const double2 *__restrict__ sv,
                                              int nv2, int lane, double2 (&v)[kUnroll],
                                              const double2 *__restrict__ next) {
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
    for (int c = lane; c - lane < nv2; c += 32 * kUnroll) {
        if (c != lane) chunk_load(row, c, nv2, v);
#pragma unroll
        for (int u = 0; u < kUnroll; u += 2) {
            const double2 y0 = c + 32 * u < nv2 ? sv[c + 32 * u] : make_double2(0.0, 0.0);
            const double2 y1 = c + 32 * (u + 1) < nv2 ? sv[c + 32 * (u + 1)] : make_double2(0.0, 0.0);
            acc0 = fma(v[u].x, y0.x, acc0);
            acc1 = fma(v[u].y, y0.y, acc1);
            acc2 = fma(v[u + 1].x, y1.x, acc2);
            acc3 = fma(v[u + 1].y, y1.y, acc3);
        }
    }
    if (next) chunk_load(next, lane, nv2, v);
    return warp_sum((acc0 + acc1) + (acc2 + acc3));
}

// Four loads per thread in flight before the first shared-memory store, so a vector of up to
// 4 x blockDim double2 (config 1's y: 1000 double2 over 512 threads) costs one L2 round trip
// (the plain loop was compiled as a one-trip-at-a-time remainder loop: load, store, load, ...).
__device__ __forceinline__ void stage(double *s, const double *g, int64_t len) {
    const double2 *g2 = reinterpret_cast<const double2 *>(g);
    double2 *s2 = reinterpret_cast<double2 *>(s);
    const int64_t n2 = len >> 1;
    for (int64_t i0 = threadIdx.x; i0 < n2; i0 += 4 * (int64_t)blockDim.x) {
        double2 t[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t i = i0 + k * (int64_t)blockDim.x;
            if (i < n2) t[k] = g2[i];
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t i = i0 + k * (int64_t)blockDim.x;
            if (i < n2) s2[i] = t[k];
        }
    }
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) k_pass_a(const PassAArgs a) {
    extern __shared__ __align__(16) double smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int nw = kThreads / 32;
    const int64_t rows = a.row_end - a.row_begin;
    const int64_t r0 = a.row_begin + rows * blockIdx.x / gridDim.x;
    const int64_t r1 = a.row_begin + rows * (blockIdx.x + 1) / gridDim.x;
    const int nv2 = (int)(a.ld >> 1);
    const double2 *A2 = reinterpret_cast<const double2 *>(a.A);
    const int64_t ld2 = a.ld >> 1;
    double2 v[kUnroll];
    if (r0 + warp < r1) chunk_load(A2 + (r0 + warp) * ld2, lane, nv2, v);   // matrix only: before the wait
    pdl_wait();   // PDL (epilogue.cuh): the launch overlaps the previous kernel's tail
    pdl_trigger();
    if (a.skip && *a.skip) return;
    stage(smem, a.y, a.ld);
    __syncthreads();
    const double2 *sv = reinterpret_cast<const double2 *>(smem);
    const OuterA o = outer_a(a, MODE);
    for (int64_t row = r0 + warp; row < r1; row += nw) {
        // epilogue operands are fetched before the stream so their latency overlaps it
        EpiA e{};
        if (lane == 0) e = epi_a_load(a, MODE, row, o);
        const double s = row_dot_pre(A2 + row * ld2, sv, nv2, lane, v, row + nw < r1 ? A2 + (row + nw) * ld2 : nullptr);
        if (lane == 0) epi_a_store(a, MODE, row, s, e, o);
    }
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) k_pass_b(const PassBArgs b) {
    extern __shared__ __align__(16) double smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int nw = kThreads / 32;
    const int64_t r0 = b.nrows * blockIdx.x / gridDim.x;
    const int64_t r1 = b.nrows * (blockIdx.x + 1) / gridDim.x;
    const int nv2 = (int)(b.ldp >> 1);
    const double2 *G2 = reinterpret_cast<const double2 *>(b.GT);
    const int64_t ld2 = b.ldp >> 1;
    double2 v[kUnroll];
    if (nv2 > 0 && r0 + warp < r1) chunk_load(G2 + (r0 + warp) * ld2, lane, nv2, v);   // before the wait
    pdl_wait();   // PDL (epilogue.cuh): the launch overlaps the previous kernel's tail
    pdl_trigger();
    if (b.skip && *b.skip) return;
    stage(smem, b.w, b.ldp);
    __syncthreads();
    const double2 *sv = reinterpret_cast<const double2 *>(smem);
    const double avg_w = avg_weight(b, MODE);
    for (int64_t j = r0 + warp; j < r1; j += nw) {
        EpiB e{};
        if (lane == 0) e = epi_b_load(b, MODE, j, avg_w);
        const double t = nv2 > 0 ? row_dot_pre(G2 + j * ld2, sv, nv2, lane, v, j + nw < r1 ? G2 + (j + nw) * ld2 : nullptr)
                                 : 0.0;
        if (lane == 0) epi_b_store(b, MODE, j, t, e, avg_w);
    }
}

// ------------------------------------------------------------------ persistent two-pass solve
// For dense single-GPU QPs whose matrices sit in L2 (config 1: 64 MB), kernel launches dominate
// a two-kernel inner step.  k_persist runs the whole solve in ONE cooperative launch: per inner
// step, pass A (y staged from L2), a grid barrier, pass B (w staged), a grid barrier.  Q rows and
// G rows are partitioned separately and pass B uses pass A's Q-row partition with the same warp
// mapping, so qy[j] is written and read by the same thread; the vectors every CTA reads (y, w)
// are staged with L1-bypassing loads (L1 is not coherent across SMs).  Same row sums and epilogues
// as k_pass_a / k_pass_b: bitwise the multi-launch result.
__device__ __forceinline__ void stage_cg(double *s, const double *g, int64_t len) {
    const double2 *g2 = reinterpret_cast<const double2 *>(g);
    double2 *s2 = reinterpret_cast<double2 *>(s);
    for (int64_t i = threadIdx.x; i < (len >> 1); i += blockDim.x) s2[i] = __ldcg(g2 + i);
}

__device__ __forceinline__ void grid_barrier(uint32_t *bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile uint32_t *gen = bar + 1;
        const uint32_t g = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            bar[0] = 0;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kThreads, 1) k_persist(const PassAArgs a0, const PassBArgs b0,
                                                        const double *beta_in, int K, int Kin, uint32_t *bar) {
    extern __shared__ __align__(16) double smem[];
    __shared__ int32_t jj;
    PassAArgs a = a0;
    PassBArgs b = b0;
    a.d_j = &jj;
    b.d_j = &jj;
    const double2 *sv = reinterpret_cast<const double2 *>(smem);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int nw = kThreads / 32;
    const int64_t n = a.nq, p = a.row_end - a.nq;
    const int64_t q0 = n * blockIdx.x / gridDim.x, q1 = n * (blockIdx.x + 1) / gridDim.x;       // Q rows
    const int64_t g0 = n + p * blockIdx.x / gridDim.x, g1 = n + p * (blockIdx.x + 1) / gridDim.x;   // G rows
    const int nva = (int)(a.ld >> 1), nvb = (int)(b.ldp >> 1);
    for (int j = 1; j <= K + 1; ++j) {
        if (threadIdx.x == 0) jj = j;
        for (int k = 1; k <= Kin; ++k) {
            a.first_inner = (k == 1);
            stage_cg(smem, a.y, a.ld);
            __syncthreads();
            const OuterA o = outer_a(a, MODE_SOLVE);
            for (int h = 0; h < 2; ++h) {   // pass A: this CTA's Q rows, then its G rows
                const int64_t r0 = h ? g0 : q0, r1 = h ? g1 : q1;
                for (int64_t row = r0 + warp; row < r1; row += nw) {
                    EpiA e{};
                    if (lane == 0) e = epi_a_load(a, MODE_SOLVE, row, o);
                    const double s = row_dot(reinterpret_cast<const double2 *>(a.A + row * a.ld), sv, nva, lane);
                    if (lane == 0) epi_a_store(a, MODE_SOLVE, row, s, e, o);
                }
            }
            grid_barrier(bar);   // w complete
            b.beta_in = beta_in[k];
            b.last_inner = (k == Kin);
            stage_cg(smem, b.w, b.ldp);
            __syncthreads();
            const double avg_w = avg_weight(b, MODE_SOLVE);
            for (int64_t r = q0 + warp; r < q1; r += nw) {   // pass B on pass A's Q-row partition
                EpiB e{};
                if (lane == 0) e = epi_b_load(b, MODE_SOLVE, r, avg_w);
                const double t = nvb > 0 ? row_dot(reinterpret_cast<const double2 *>(b.GT + r * b.ldp), sv, nvb, lane)
                                         : 0.0;
                if (lane == 0) epi_b_store(b, MODE_SOLVE, r, t, e, avg_w);
            }
            grid_barrier(bar);   // y complete
        }
    }
}

// K3, the rho = 0 inner step (SURVEY §8(a) row a1'): with rho = 0 the multiplier term of the
// gradient is G'mu, constant over an inner solve ("only G'mu is computed at each
// outer iteration"), so c = q + G'mu is formed once per outer iteration and each inner step
// streams Q only: grad = Qy + c, x+ = [y - grad/L]_U, y+ = x+ + beta (x+ - x).
// y is read (staged) from yin and written to yout (ping-pong: every CTA stages all of y).
__global__ void __launch_bounds__(kThreads, 1) k_rho0_step(const PassAArgs a, const PassBArgs bl,
                                                          const PassBArgs bs) {
    extern __shared__ __align__(16) double smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int nw = kThreads / 32;
    const int64_t r0 = a.nq * blockIdx.x / gridDim.x;
    const int64_t r1 = a.nq * (blockIdx.x + 1) / gridDim.x;
    const int nv2 = (int)(a.ld >> 1);
    const double2 *A2 = reinterpret_cast<const double2 *>(a.A);
    const int64_t ld2 = a.ld >> 1;
    double2 v[kUnroll];
    if (r0 + warp < r1) chunk_load(A2 + (r0 + warp) * ld2, lane, nv2, v);   // matrix only: before the wait
    pdl_wait();   // PDL (epilogue.cuh): the launch overlaps the previous kernel's tail
    pdl_trigger();
    if (a.skip && *a.skip) return;
    stage(smem, a.y, a.ld);
    __syncthreads();
    const double2 *sv = reinterpret_cast<const double2 *>(smem);
    const double avg_w = avg_weight(bl, MODE_SOLVE);
    for (int64_t j = r0 + warp; j < r1; j += nw) {
        EpiB e{};
        if (lane == 0) e = epi_b_load(bl, MODE_SOLVE, j, avg_w);     // bl.q = c, bl.y = yin slice
        const double s = row_dot_pre(A2 + j * ld2, sv, nv2, lane, v, j + nw < r1 ? A2 + (j + nw) * ld2 : nullptr);
        if (lane == 0) {
            e.qy = s;                                                  // grad = (Qy + c) + 0
            epi_b_store(bs, MODE_SOLVE, j, 0.0, e, avg_w);             // bs.y = yout slice
        }
    }
}

__global__ void k_init_state(double *x, double *y, double *xhat, const double *lb, const double *ub,
                             int64_t n, double *mu, double *lam_prev, int64_t p, int32_t *d_j,
                             int32_t *flag) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        const double x0 = fmin(fmax(0.0, lb[i]), ub[i]);   // u_bar^0 = [0]_U (reading c7)
        x[i] = x0;
        y[i] = x0;
        xhat[i] = 0.0;
    }
    if (i < p) {
        mu[i] = 0.0;        // mu^1 = lambda^0 = 0
        lam_prev[i] = 0.0;
    }
    if (i == 0) {
        *d_j = 1;
        *flag = 0;
    }
}

__global__ void k_advance(int32_t *d_j) { *d_j += 1; }

// H_ji := H_ij for i < j (row-major, leading dim ld): an exactly symmetric H for the equality path
__global__ void k_mirror_upper(double *H, int64_t n, int64_t ld) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n * n) return;
    const int64_t i = t / n, j = t % n;
    if (i < j) H[j * ld + i] = H[i * ld + j];
}

// warm start (duquad_set_initial): u_bar^0 = [x0]_U, lambda^0 = mu^1 = lam0, for B QPs with
// strides sn / sp (B = 1: plain slices); runs after k_init_state / k_init_batched
__global__ void k_apply_initial(double *x, double *y, const double *lb, const double *ub, int64_t n, int64_t sn,
                                const double *x0, double *mu, double *lam_prev, int64_t p, int64_t sp,
                                const double *lam0, int64_t B) {
    const int64_t m = n > p ? n : p;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < B * m;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = t / m, i = t - b * m;
        if (x0 && i < n) {
            const double v = fmin(fmax(x0[b * sn + i], lb[i]), ub[i]);
            x[b * sn + i] = v;
            y[b * sn + i] = v;
        }
        if (lam0 && i < p) {
            mu[b * sp + i] = lam0[b * sp + i];
            lam_prev[b * sp + i] = lam0[b * sp + i];
        }
    }
}

// eps_in mode: gradient-map test after an inner step (fixed-order sum: block partials over
// contiguous ranges, then the last block to finish adds them in block order)
// out_sum (row-sharded): write this rank's fixed-order sum there and leave the decision to
// k_inner_decide after the all-reduce
__global__ void k_inner_check(const double *gm_sq, int64_t n, double *partials, uint32_t *counter, int32_t *done,
                              double thresh2, int32_t *counts, const int32_t *d_j, double *out_sum) {
    if (*done) return;
    __shared__ double red[32];
    __shared__ bool last;
    const int64_t lo = n * blockIdx.x / gridDim.x, hi = n * (blockIdx.x + 1) / gridDim.x;
    double s = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) s += gm_sq[i];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b += red[w];
        partials[blockIdx.x] = b;
        __threadfence();
        last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        double t = 0.0;
        for (int c = 0; c < (int)gridDim.x; ++c) t += partials[c];
        *counter = 0;
        if (out_sum) {
            *out_sum = t;
            return;
        }
        counts[*d_j - 1] += 1;
        if (t <= thresh2) *done = 1;
    }
}

// the decision of k_inner_check on the all-reduced sum (identical on every rank)
__global__ void k_inner_decide(const double *sum, int32_t *done, double thresh2, int32_t *counts, const int32_t *d_j) {
    if (*done) return;
    counts[*d_j - 1] += 1;
    if (*sum <= thresh2) *done = 1;
}

__global__ void k_inner_finish(const double *x, double *y_dst, double *xhat, int64_t n, const OuterParam *ops,
                               const int32_t *d_j, int32_t *done, int32_t *conv) {
    const double w = ops[*d_j].avg_w;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double xi = x[i];
        y_dst[i] = xi;                                         // y = u_bar^j for the next outer iteration
        if (w != 0.0) xhat[i] = xhat[i] + w * (xi - xhat[i]);  // P:700-706 (running form)
    }
}

__global__ void k_inner_reset(const int32_t *d_j, int32_t *done, int32_t *conv) {
    conv[*d_j - 1] = *done;
    *done = 0;
}

// out[j - col0][i] = G[i][j] for j in [col0, col0 + ncols), i in [0, p)
__global__ void k_transpose(const double *__restrict__ G, int64_t ldG, int64_t p, int64_t col0,
                            int64_t ncols, double *__restrict__ GT, int64_t ldp) {
    __shared__ double tile[32][33];
    const int64_t i0 = (int64_t)blockIdx.y * 32, j0 = (int64_t)blockIdx.x * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t i = i0 + r, j = j0 + threadIdx.x;
        tile[r][threadIdx.x] = (i < p && j < ncols) ? G[i * ldG + col0 + j] : 0.0;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t j = j0 + r, i = i0 + threadIdx.x;
        if (j < ncols && i < p) GT[j * ldp + i] = tile[threadIdx.x][r];
    }
}

__global__ void k_check(const double *v, int64_t rows, int64_t cols, int64_t ld, int32_t *flag) {
    const int64_t total = rows * cols;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = t / cols, c = t - r * cols;
        if (!isfinite(v[r * ld + c])) *flag = 1;
    }
}

// flag = 2 if the n x n block at A (leading dimension ld) is not symmetric to 1e-12 relative:
// 32 x 32 tiles (i0 <= j0) and their mirrors through shared memory, both read coalesced
__global__ void k_check_sym(const double *__restrict__ A, int64_t n, int64_t ld, int32_t *flag) {
    __shared__ double tile[32][33];
    const int64_t bi = blockIdx.y, bj = blockIdx.x;
    if (bj < bi) return;
    const int64_t i0 = bi * 32, j0 = bj * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {   // mirror tile: rows j0.., columns i0..
        const int64_t i = j0 + r, j = i0 + threadIdx.x;
        tile[r][threadIdx.x] = (i < n && j < n) ? A[i * ld + j] : 0.0;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t i = i0 + r, j = j0 + threadIdx.x;
        if (i < n && j < n) {
            const double a = A[i * ld + j], b = tile[threadIdx.x][r];   // Q_ij and Q_ji
            if (fabs(a - b) > 1e-12 * (fabs(a) + fabs(b))) *flag = 2;
        }
    }
}

__global__ void k_check_box(const double *lb, const double *ub, int64_t n, int32_t *flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (isnan(lb[i]) || isnan(ub[i]) || lb[i] > ub[i] || lb[i] == INFINITY || ub[i] == -INFINITY)
            *flag = 1;
    }
}

// ----------------------------------------------------------- reductions
__device__ __forceinline__ double block_sum(double v, double *red) {
    v = warp_sum(v);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    }
    return s;   // valid in thread 0
}

__global__ void k_dot_partial(const double *a, const double *b, int64_t n, double *partials) {
    __shared__ double red[32];
    const int64_t lo = n * blockIdx.x / gridDim.x, hi = n * (blockIdx.x + 1) / gridDim.x;
    double s = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) s = fma(a[i], b[i], s);
    s = block_sum(s, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// out[v] = sum_{c < nparts} partials[c * nvals + v]   (fixed order)
__global__ void k_reduce_final(const double *partials, int nparts, int nvals, double *out) {
    const int v = threadIdx.x;
    if (v >= nvals) return;
    double s = 0.0;
    for (int c = 0; c < nparts; ++c) s += partials[c * nvals + v];
    out[v] = s;
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__global__ void k_fill_hash(double *v, int64_t n, int64_t offset) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) v[i] = 0.5 + (double)(splitmix64((uint64_t)(i + offset)) >> 11) * 0x1.0p-53;
}

__global__ void k_scale_by_rsqrt(double *v, int64_t n, const double *sumsq, double *beta_out) {
    const double nrm = sqrt(*sumsq);
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) v[i] = v[i] / nrm;
    if (i == 0 && beta_out) *beta_out = nrm;
}

__global__ void k_lanczos_update(double *w, const double *v, const double *vprev, int64_t n,
                                 const double *alpha, const double *beta_prev, double *partials) {
    __shared__ double red[32];
    const double al = *alpha, be = *beta_prev;
    const int64_t lo = n * blockIdx.x / gridDim.x, hi = n * (blockIdx.x + 1) / gridDim.x;
    double s = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const double wi = w[i] - al * v[i] - be * vprev[i];
        w[i] = wi;
        s = fma(wi, wi, s);
    }
    s = block_sum(s, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void k_lanczos_next(double *v, double *vprev, const double *w, int64_t n,
                               const double *sumsq, double *beta) {
    const double nrm = sqrt(*sumsq);
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        vprev[i] = v[i];
        v[i] = nrm > 0.0 ? w[i] / nrm : 0.0;
    }
    if (i == 0) *beta = nrm;
}

__global__ void k_residual_partial(const double *x, const double *qy, const double *q, int64_t n,
                                   const double *Gx, const double *g, const double *lam,
                                   const uint8_t *cone, int64_t p, double rho, double *partials) {
    __shared__ double red[32];
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    {
        const int64_t lo = n * blockIdx.x / gridDim.x, hi = n * (blockIdx.x + 1) / gridDim.x;
        for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x)
            acc[0] += 0.5 * x[i] * qy[i] + q[i] * x[i];
    }
    {
        const int64_t lo = p * blockIdx.x / gridDim.x, hi = p * (blockIdx.x + 1) / gridDim.x;
        for (int64_t k = lo + threadIdx.x; k < hi; k += blockDim.x) {
            const double r = Gx[k] + g[k];
            const double d = r - proj_K(r, cone[k]);
            acc[1] += d * d;
            if (rho > 0.0) {
                const double wv = r + lam[k] / rho;
                const double dw = wv - proj_K(wv, cone[k]);
                acc[2] += dw * dw;
            }
            acc[3] += lam[k] * lam[k];
            acc[4] += lam[k] * r;
        }
    }
#pragma unroll
    for (int v = 0; v < 5; ++v) {
        const double s = block_sum(acc[v], red);
        if (threadIdx.x == 0) partials[blockIdx.x * 5 + v] = s;
    }
}

inline int blocks_for(int64_t n, int t) { return (int)((n + t - 1) / t); }

}  // namespace

int pass_threads() { return kThreads; }

cudaError_t configure_pass_kernels(size_t smem_a, size_t smem_b) {
    cudaError_t e;
    const size_t sm_a = smem_a < 48 * 1024 ? 48 * 1024 : smem_a;
    const size_t sm_b = smem_b < 48 * 1024 ? 48 * 1024 : smem_b;
    if ((e = cudaFuncSetAttribute(k_pass_a<MODE_SOLVE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_a)))
        return e;
    if ((e = cudaFuncSetAttribute(k_pass_a<MODE_LIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_a)))
        return e;
    if ((e = cudaFuncSetAttribute(k_pass_b<MODE_SOLVE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_b)))
        return e;
    if ((e = cudaFuncSetAttribute(k_rho0_step, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_a))) return e;
    return cudaFuncSetAttribute(k_pass_b<MODE_LIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_b);
}

cudaError_t launch_pass_a(const PassAArgs &a, int mode, const LaunchCfg &cfg, cudaStream_t s) {
    if (a.row_end <= a.row_begin) return cudaSuccess;
    if (a.fmt == DUQUAD_CSR) return a.sp_kind != SPK_CSR ? launch_pass_a_lane(a, mode, cfg, s) : launch_pass_a_csr(a, mode, cfg, s);
    if (mode == MODE_SOLVE)
        return launch_ex(k_pass_a<MODE_SOLVE>, cfg.grid, kThreads, cfg.smem, s, cfg.pdl, 0, a);
    else
        return launch_ex(k_pass_a<MODE_LIN>, cfg.grid, kThreads, cfg.smem, s, cfg.pdl, 0, a);
}

cudaError_t launch_pass_b(const PassBArgs &b, int mode, const LaunchCfg &cfg, cudaStream_t s) {
    if (b.nrows <= 0) return cudaSuccess;
    if (b.fmt == DUQUAD_CSR) return b.sp_kind != SPK_CSR ? launch_pass_b_lane(b, mode, cfg, s) : launch_pass_b_csr(b, mode, cfg, s);
    if (mode == MODE_SOLVE)
        return launch_ex(k_pass_b<MODE_SOLVE>, cfg.grid, kThreads, cfg.smem, s, cfg.pdl, 0, b);
    else
        return launch_ex(k_pass_b<MODE_LIN>, cfg.grid, kThreads, cfg.smem, s, cfg.pdl, 0, b);
}

cudaError_t launch_rho0_step(const PassAArgs &a, const PassBArgs &bl, const PassBArgs &bs, const LaunchCfg &cfg,
                             cudaStream_t s) {
    if (a.nq <= 0) return cudaSuccess;
    return launch_ex(k_rho0_step, cfg.grid, kThreads, cfg.smem, s, cfg.pdl, 0, a, bl, bs);
}

cudaError_t launch_init_state(double *x, double *y, double *xhat, const double *lb, const double *ub,
                              int64_t n, double *mu, double *lam_prev, int64_t p, int32_t *d_j,
                              int32_t *flag, cudaStream_t s) {
    const int64_t m = n > p ? n : p;
    k_init_state<<<blocks_for(m > 0 ? m : 1, 256), 256, 0, s>>>(x, y, xhat, lb, ub, n, mu, lam_prev, p,
                                                               d_j, flag);
    return cudaGetLastError();
}

cudaError_t launch_inner_check(const double *gm_sq, int64_t n, double *partials, uint32_t *counter, int32_t *done,
                               double thresh2, int32_t *counts, const int32_t *d_j, double *out_sum, cudaStream_t s) {
    k_inner_check<<<kRedGrid, kRedThreads, 0, s>>>(gm_sq, n, partials, counter, done, thresh2, counts, d_j,
                                                   out_sum);
    return cudaGetLastError();
}

cudaError_t launch_inner_decide(const double *sum, int32_t *done, double thresh2, int32_t *counts,
                                const int32_t *d_j, cudaStream_t s) {
    k_inner_decide<<<1, 1, 0, s>>>(sum, done, thresh2, counts, d_j);
    return cudaGetLastError();
}

cudaError_t launch_inner_finish(const double *x, double *y_dst, double *xhat, int64_t n, const OuterParam *ops,
                                const int32_t *d_j, int32_t *done, int32_t *conv, cudaStream_t s) {
    const int grid = (int)std::min<int64_t>(1184, std::max<int64_t>(1, (n + 255) / 256));
    k_inner_finish<<<grid, 256, 0, s>>>(x, y_dst, xhat, n, ops, d_j, done, conv);
    k_inner_reset<<<1, 1, 0, s>>>(d_j, done, conv);
    return cudaGetLastError();
}

cudaError_t launch_apply_initial(double *x, double *y, const double *lb, const double *ub, int64_t n, int64_t sn,
                                 const double *x0, double *mu, double *lam_prev, int64_t p, int64_t sp,
                                 const double *lam0, int64_t B, cudaStream_t s) {
    const int64_t m = B * std::max<int64_t>(std::max<int64_t>(n, p), 1);
    k_apply_initial<<<(unsigned)std::min<int64_t>(1184, (m + 255) / 256), 256, 0, s>>>(x, y, lb, ub, n, sn, x0, mu,
                                                                                     lam_prev, p, sp, lam0, B);
    return cudaGetLastError();
}

cudaError_t launch_persist(const PassAArgs &a, const PassBArgs &b, const double *beta_in, int K, int Kin,
                           uint32_t *bar, int grid, size_t smem, cudaStream_t s) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_persist, a, b, beta_in, K, Kin, bar);
}

cudaError_t configure_persist(size_t smem) {
    return cudaFuncSetAttribute(k_persist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

cudaError_t launch_advance(int32_t *d_j, cudaStream_t s) {
    k_advance<<<1, 1, 0, s>>>(d_j);
    return cudaGetLastError();
}

cudaError_t launch_transpose(const double *G, int64_t ldG, int64_t p, int64_t col0, int64_t ncols,
                             double *GT, int64_t ldp, cudaStream_t s) {
    if (p <= 0 || ncols <= 0) return cudaSuccess;
    dim3 grid((unsigned)((ncols + 31) / 32), (unsigned)((p + 31) / 32));
    k_transpose<<<grid, dim3(32, 8), 0, s>>>(G, ldG, p, col0, ncols, GT, ldp);
    return cudaGetLastError();
}

cudaError_t launch_check(const double *v, int64_t rows, int64_t cols, int64_t ld, int32_t *flag,
                         cudaStream_t s) {
    if (rows <= 0 || cols <= 0) return cudaSuccess;
    k_check<<<1184, 256, 0, s>>>(v, rows, cols, ld, flag);
    return cudaGetLastError();
}

cudaError_t launch_check_sym(const double *A, int64_t n, int64_t ld, int32_t *flag, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const unsigned nb = (unsigned)((n + 31) / 32);
    k_check_sym<<<dim3(nb, nb), dim3(32, 8), 0, s>>>(A, n, ld, flag);
    return cudaGetLastError();
}

cudaError_t launch_check_box(const double *lb, const double *ub, int64_t n, int32_t *flag,
                             cudaStream_t s) {
    k_check_box<<<148, 256, 0, s>>>(lb, ub, n, flag);
    return cudaGetLastError();
}

cudaError_t launch_dot_partial(const double *a, const double *b, int64_t n, double *partials,
                               cudaStream_t s) {
    k_dot_partial<<<kRedGrid, kRedThreads, 0, s>>>(a, b, n, partials);
    return cudaGetLastError();
}

cudaError_t launch_reduce_final(const double *partials, int nparts, int nvals, double *out,
                                cudaStream_t s) {
    k_reduce_final<<<1, 32, 0, s>>>(partials, nparts, nvals, out);
    return cudaGetLastError();
}

cudaError_t launch_fill_hash(double *v, int64_t n, int64_t offset, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    k_fill_hash<<<blocks_for(n, 256), 256, 0, s>>>(v, n, offset);
    return cudaGetLastError();
}

cudaError_t launch_mirror_upper(double *H, int64_t n, int64_t ld, cudaStream_t s) {
    if (n <= 1) return cudaSuccess;
    const int64_t m = n * n;
    k_mirror_upper<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(H, n, ld);
    return cudaGetLastError();
}

cudaError_t launch_scale_by_rsqrt(double *v, int64_t n, const double *sumsq, double *beta_out,
                                  cudaStream_t s) {
    k_scale_by_rsqrt<<<blocks_for(n > 0 ? n : 1, 256), 256, 0, s>>>(v, n, sumsq, beta_out);
    return cudaGetLastError();
}

cudaError_t launch_lanczos_update(double *w, const double *v, const double *vprev, int64_t n,
                                  const double *alpha, const double *beta_prev, double *partials,
                                  cudaStream_t s) {
    k_lanczos_update<<<kRedGrid, kRedThreads, 0, s>>>(w, v, vprev, n, alpha, beta_prev, partials);
    return cudaGetLastError();
}

cudaError_t launch_lanczos_next(double *v, double *vprev, const double *w, int64_t n,
                                const double *sumsq, double *beta, cudaStream_t s) {
    k_lanczos_next<<<blocks_for(n > 0 ? n : 1, 256), 256, 0, s>>>(v, vprev, w, n, sumsq, beta);
    return cudaGetLastError();
}

cudaError_t launch_residual_partial(const double *x, const double *qy, const double *q, int64_t n,
                                    const double *Gx, const double *g, const double *lam,
                                    const uint8_t *cone, int64_t p, double rho, double *partials,
                                    cudaStream_t s) {
    k_residual_partial<<<kRedGrid, kRedThreads, 0, s>>>(x, qy, q, n, Gx, g, lam, cone, p, rho, partials);
    return cudaGetLastError();
}

}  // namespace dq
