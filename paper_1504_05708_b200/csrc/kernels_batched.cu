// Batched (MPC-shaped) sm_100a kernels: B QPs sharing Q and G (SURVEY.md §8(a) row a9,
// BASELINE.json configs[3], north_star (c)).
//
// With B right-hand sides the two passes of an inner step are real dense contractions:
//   pass A:  [Q;G] (n+p x n) . Y (n x B)   -> QY, and per (row, QP) the w / DFOM epilogue
//   pass B:  G'    (n x p)   . W (p x B)   -> per (row, QP) the clamp / momentum / average epilogue
// run on the FP64 tensor pipe with DMMA (`mma.sync.aligned.m8n8k4.row.col.f64`, SASS DMMA.8x8x4;
// tcgen05.mma has no f64 kind).  Per-QP vectors are stored QP-major (B x ld, zero-padded to a
// multiple of 32), which is exactly the "col" B-operand layout, so no transposes are needed.
// Tiles: a CTA computes BM = 8*MT rows x BN = NW*WN QPs; the K dimension is streamed in
// BK = 32 chunks through a cp.async double buffer; shared-memory rows are padded by 4 doubles
// so the 8x4 fragment loads of a half-warp hit 32 distinct banks.  The epilogue (epilogue.cuh)
// is the single-QP one applied to a per-QP view, so every QP follows the identical arithmetic.
#include <cuda_runtime.h>
#include <stdint.h>

#include "duquad_internal.h"
#include "epilogue.cuh"

namespace dq {

namespace {

constexpr int BK = 32;
constexpr int PADK = BK + 4;

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool pred) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int bytes = pred ? 16 : 0;   // src-size 0 -> zero fill
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// C[m][b] = sum_k A[m][k] * Bop[b][k];  A: M x K row-major (lda), Bop: N x K (ldb), K padded to BK.
template <int MT, int WN, int NW, int PASS, int MODE>
__global__ void __launch_bounds__(NW * 32) k_batched(const BatchedArgs args) {
    constexpr int BM = 8 * MT, BN = NW * WN, NT = WN / 8;
    extern __shared__ __align__(16) double smem[];
    double *As = smem;                    // [2][BM][PADK]
    double *Bs = smem + 2 * BM * PADK;    // [2][BN][PADK]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
    const int nchunks = (int)(args.K / BK);

    auto load_chunk = [&](int kc, int buf) {
        double *as = As + buf * BM * PADK;
        double *bs = Bs + buf * BN * PADK;
        const int64_t k0 = (int64_t)kc * BK;
        for (int c = tid; c < BM * (BK / 2); c += NW * 32) {
            const int r = c / (BK / 2), kk = (c % (BK / 2)) * 2;
            const bool ok = m0 + r < args.M;
            cp_async16(as + r * PADK + kk, args.Aop + (ok ? (m0 + r) * args.lda + k0 + kk : 0), ok);
        }
        for (int c = tid; c < BN * (BK / 2); c += NW * 32) {
            const int r = c / (BK / 2), kk = (c % (BK / 2)) * 2;
            const bool ok = n0 + r < args.N;
            cp_async16(bs + r * PADK + kk, args.Bop + (ok ? (n0 + r) * args.ldb + k0 + kk : 0), ok);
        }
    };

    double acc[MT][NT][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    const int fr = lane >> 2, fk = lane & 3;   // fragment row / k index of this lane
    load_chunk(0, 0);
    cp_async_commit();
    for (int kc = 0; kc < nchunks; ++kc) {
        const int buf = kc & 1;
        if (kc + 1 < nchunks) {
            load_chunk(kc + 1, buf ^ 1);
            cp_async_commit();
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const double *as = As + buf * BM * PADK;
        const double *bs = Bs + buf * BN * PADK + (warp * WN) * PADK;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double bf[NT];
#pragma unroll
            for (int j = 0; j < NT; ++j) bf[j] = bs[(j * 8 + fr) * PADK + kk + fk];
#pragma unroll
            for (int i = 0; i < MT; ++i) {
                const double af = as[(i * 8 + fr) * PADK + kk + fk];
#pragma unroll
                for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], af, bf[j]);
            }
        }
        __syncthreads();
    }

    // epilogue, stage 1: the C tile goes to shared memory QP-major, Cs[col][row]
    // (fragment element: row fr, cols 2*fk, 2*fk+1 of each 8x8 tile); the operand buffers are free.
    constexpr int LDC = BM + 1;
    double *Cs = smem;
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) Cs[(warp * WN + j * 8 + 2 * fk + h) * LDC + i * 8 + fr] = acc[i][j][h];
    __syncthreads();
    // stage 2: a warp owns QP columns, lanes own rows, so the per-QP vectors (QP-major) are
    // accessed coalesced; the operands of 2 columns x RPL rows are loaded before any store.
    constexpr int RPL = (BM + 31) / 32;
    if (PASS == 0) {
        const OuterA o = outer_a(args.a, MODE);
        for (int cb = warp; cb < BN; cb += 2 * NW) {
            PassAArgs v[2];
            bool vb[2];
            EpiA e[2][RPL];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int col = cb + c * NW;
                const int64_t b = n0 + col;
                vb[c] = col < BN && b < args.N;
                v[c] = args.a;                   // per-QP view
                v[c].qy += b * args.sn;
                v[c].w += b * args.sp;
                v[c].g += b * args.sp;
                v[c].mu += b * args.sp;
                v[c].lam_prev += b * args.sp;
#pragma unroll
                for (int t = 0; t < RPL; ++t) {
                    const int r = lane + 32 * t;
                    if (vb[c] && r < BM && m0 + r < args.M) e[c][t] = epi_a_load(v[c], MODE, m0 + r, o);
                }
            }
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
                for (int t = 0; t < RPL; ++t) {
                    const int r = lane + 32 * t;
                    if (vb[c] && r < BM && m0 + r < args.M)
                        epi_a_store(v[c], MODE, m0 + r, Cs[(cb + c * NW) * LDC + r], e[c][t], o);
                }
        }
    } else {
        const double avg_w = avg_weight(args.b, MODE);
        for (int cb = warp; cb < BN; cb += 2 * NW) {
            PassBArgs v[2];
            bool vb[2];
            EpiB e[2][RPL];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int col = cb + c * NW;
                const int64_t b = n0 + col;
                vb[c] = col < BN && b < args.N;
                v[c] = args.b;
                v[c].qy += b * args.sn;
                v[c].q += b * args.sn;
                v[c].x += b * args.sn;
                v[c].y += b * args.sn;
                v[c].xhat += b * args.sn;
                if (MODE == MODE_LIN) v[c].out += b * args.sn;
#pragma unroll
                for (int t = 0; t < RPL; ++t) {
                    const int r = lane + 32 * t;
                    if (vb[c] && r < BM && m0 + r < args.M) e[c][t] = epi_b_load(v[c], MODE, m0 + r, avg_w);
                }
            }
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
                for (int t = 0; t < RPL; ++t) {
                    const int r = lane + 32 * t;
                    if (vb[c] && r < BM && m0 + r < args.M)
                        epi_b_store(v[c], MODE, m0 + r, Cs[(cb + c * NW) * LDC + r], e[c][t], avg_w);
                }
        }
    }
}

template <int MT, int WN, int NW, int PASS>
cudaError_t launch_t(const BatchedArgs &a, int mode, cudaStream_t s) {
    constexpr int BM = 8 * MT, BN = NW * WN;
    const size_t smem = (size_t)2 * (BM + BN) * PADK * sizeof(double);
    dim3 grid((unsigned)((a.N + BN - 1) / BN), (unsigned)((a.M + BM - 1) / BM));
    if (mode == MODE_SOLVE)
        k_batched<MT, WN, NW, PASS, MODE_SOLVE><<<grid, NW * 32, smem, s>>>(a);
    else
        k_batched<MT, WN, NW, PASS, MODE_LIN><<<grid, NW * 32, smem, s>>>(a);
    return cudaGetLastError();
}

template <int MT, int WN, int NW, int PASS>
cudaError_t configure_t() {
    constexpr int BM = 8 * MT, BN = NW * WN;
    const int smem = 2 * (BM + BN) * PADK * (int)sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(k_batched<MT, WN, NW, PASS, MODE_SOLVE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e) return e;
    return cudaFuncSetAttribute(k_batched<MT, WN, NW, PASS, MODE_LIN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                smem);
}

}  // namespace

cudaError_t configure_batched_kernels() {
    cudaError_t e;
    if ((e = configure_t<15, 16, 4, 0>())) return e;
    if ((e = configure_t<16, 16, 4, 0>())) return e;
    if ((e = configure_t<15, 8, 4, 1>())) return e;
    return configure_t<16, 8, 4, 1>();
}

// Row-tile height: 8*15 = 120 (configs[3]: n = 120, n + p = 840 = 7 x 120) unless 128 pads less.
int batched_mt(int64_t M) {
    const int64_t pad15 = (M + 119) / 120 * 120 - M, pad16 = (M + 127) / 128 * 128 - M;
    return pad15 <= pad16 ? 15 : 16;
}

cudaError_t launch_batched(const BatchedArgs &a, int pass, int mode, cudaStream_t s) {
    if (a.N <= 0 || a.M <= 0) return cudaSuccess;
    const int mt = batched_mt(a.M);
    if (pass == 0)
        return mt == 15 ? launch_t<15, 16, 4, 0>(a, mode, s) : launch_t<16, 16, 4, 0>(a, mode, s);
    return mt == 15 ? launch_t<15, 8, 4, 1>(a, mode, s) : launch_t<16, 8, 4, 1>(a, mode, s);
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
