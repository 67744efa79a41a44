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
// One persistent, warp-specialised CTA per SM.  The QPs are cut into groups of <= NT octets
// (8 QPs); a CTA owns whole groups, so there is no inter-CTA traffic.  For each group it walks
// the rows in blocks of 128 (16 m8 tiles) and the reduction dimension in BK = 32 chunks:
//   - 2 producer warps stream the A chunk (128 x 32) and the B chunk (8*NT x 32) of every step
//     into a STAGES-deep shared-memory ring with cp.async; each thread's copies arrive on the
//     stage's "full" mbarrier (cp.async.mbarrier.arrive.noinc);
//   - 8 math warps (two per SM sub-partition; warp w owns m8 tiles w and w + 8 of the block,
//     all NT n8 tiles) issue the DMMAs and release the stage on its "empty" mbarrier;
//   - at the end of a block the math warps park the C tile in shared memory (QP-major) and
//     6 epilogue warps apply the DFOM epilogue (epilogue.cuh, the single-QP arithmetic on a
//     per-QP view) while the math warps already run the next block.
// The DMMA pipe is the bound (1 DMMA.8x8x4 per 16 cycles per sub-partition on this part); the
// old 2-CTA/SM tile kernel ran it at 30 % (pass A) because its epilogue and the 3.03-wave
// tail were serialised with the math.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "duquad_internal.h"
#include "epilogue.cuh"

namespace dq {

namespace {

constexpr int BK = 32;
constexpr int PADK = BK + 4;    // smem row pitch (doubles): the 8x4 fragment loads of a half-warp hit 32 banks
constexpr int kMathW = 8, kProdW = 2, kEpiW = 6;
constexpr int kWarpsB = kMathW + kProdW + kEpiW;
constexpr int kThreadsB = 32 * kWarpsB;
constexpr int kBlkM = 128;      // rows per block: 16 m8 tiles
constexpr int LDC = kBlkM + 4;  // C tile: Cs[qp][row]
constexpr int kSmemCap = 225 * 1024;

template <int NT>
struct Geo {
    static constexpr int BN = 8 * NT;
    static constexpr int SA = kBlkM * PADK, SB = BN * PADK;   // doubles per stage
    static constexpr int CS = BN * LDC;
    static constexpr int STAGES = (kSmemCap - 8 * CS - 128) / (8 * (SA + SB));
    static constexpr size_t SMEM = 8 * ((size_t)STAGES * (SA + SB) + CS) + 128;
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

struct Group {
    int64_t q0;   // first QP
    int nq, nc;   // valid QPs, octets
};
__device__ __forceinline__ Group group_of(const BatchedArgs &a, int64_t g) {
    const int64_t c0 = g * a.ncol8 / a.ngroups, c1 = (g + 1) * a.ncol8 / a.ngroups;
    Group r;
    r.q0 = 8 * c0;
    r.nc = (int)(c1 - c0);
    const int64_t nq = a.N - r.q0 < 8 * (c1 - c0) ? a.N - r.q0 : 8 * (c1 - c0);
    r.nq = nq > 0 ? (int)nq : 0;
    return r;
}

// ---------------------------------------------------------------- epilogues (one block of one group)
// Pass A: 3 QP columns x 4 rows per lane per round, operands loaded before any store.
__device__ __forceinline__ void epi_block_a(const BatchedArgs &args, const double *Cs, int64_t m0, const Group &gr,
                                            int wid, int nwk, int lane, const OuterA &o) {
    constexpr int NCOL = 2, RPL = kBlkM / 32;
    for (int cb = wid; cb < gr.nq; cb += NCOL * nwk) {
        EpiA e[NCOL][RPL];
#pragma unroll
        for (int c = 0; c < NCOL; ++c) {
            const int col = cb + c * nwk;
            PassAArgs v = args.a;
            const int64_t b = gr.q0 + col;
            v.g += b * args.sp;
            v.mu += b * args.sp;
            v.lam_prev += b * args.sp;
#pragma unroll
            for (int t = 0; t < RPL; ++t) {
                const int64_t row = m0 + lane + 32 * t;
                if (col < gr.nq && row < args.M) e[c][t] = epi_a_load(v, MODE_SOLVE, row, o);
            }
        }
#pragma unroll
        for (int c = 0; c < NCOL; ++c) {
            const int col = cb + c * nwk;
            PassAArgs v = args.a;
            const int64_t b = gr.q0 + col;
            v.qy += b * args.sn;
            v.w += b * args.sp;
            v.mu += b * args.sp;
            v.lam_prev += b * args.sp;
#pragma unroll
            for (int t = 0; t < RPL; ++t) {
                const int r = lane + 32 * t;
                if (col < gr.nq && m0 + r < args.M)
                    epi_a_store(v, MODE_SOLVE, m0 + r, Cs[col * LDC + r], e[c][t], o);
            }
        }
    }
}

// Pass B: 1 QP column x 4 rows per lane per round (seven operands each).
__device__ __forceinline__ void epi_block_b(const BatchedArgs &args, const double *Cs, int64_t m0, const Group &gr,
                                            int wid, int nwk, int lane, double avg_w) {
    constexpr int RPL = kBlkM / 32;
    for (int col = wid; col < gr.nq; col += nwk) {
        PassBArgs v = args.b;
        const int64_t b = gr.q0 + col;
        v.qy += b * args.sn;
        v.q += b * args.sn;
        v.x += b * args.sn;
        v.y += b * args.sn;
        v.xhat += b * args.sn;
        EpiB e[RPL];
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
            const int64_t row = m0 + lane + 32 * t;
            if (row < args.M) e[t] = epi_b_load(v, MODE_SOLVE, row, avg_w);
        }
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
            const int r = lane + 32 * t;
            if (m0 + r < args.M) epi_b_store(v, MODE_SOLVE, m0 + r, Cs[col * LDC + r], e[t], avg_w);
        }
    }
}

// C[m][b] = sum_k A[m][k] * Bop[b][k];  A: M x K row-major (lda), Bop: N x K (ldb), K padded to BK.
template <int PASS, int NT>
__global__ void __launch_bounds__(kThreadsB, 1) k_batched(const BatchedArgs args) {
    using GE = Geo<NT>;
    constexpr int ST = GE::STAGES;
    extern __shared__ __align__(16) double smem[];
    double *As = smem;
    double *Bs = As + ST * GE::SA;
    double *Cs = Bs + ST * GE::SB;
    uint64_t *bars = reinterpret_cast<uint64_t *>(Cs + GE::CS);
    uint64_t *full = bars, *empty = bars + ST, *cs_full = bars + 2 * ST, *cs_empty = cs_full + 1;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(full + s, kProdW * 32);
            mbar_init(empty + s, kMathW * 32);
        }
        mbar_init(cs_full, kMathW * 32);
        mbar_init(cs_empty, kEpiW * 32);
    }
    __syncthreads();
    const int nmb = (int)((args.M + kBlkM - 1) / kBlkM), nkc = (int)(args.K / BK);

    if (warp < kMathW) {   // ------------------------------------------------ math warps
        const int fr = lane >> 2, fk = lane & 3;
        uint32_t s = 0, blk = 0;
        for (int64_t g = blockIdx.x; g < args.ngroups; g += gridDim.x) {
            const Group gr = group_of(args, g);
            if (gr.nq == 0) continue;
            for (int mb = 0; mb < nmb; ++mb) {
                const int64_t m0 = (int64_t)mb * kBlkM;
                const bool v0 = m0 + 8 * warp < args.M, v1 = m0 + 8 * (warp + 8) < args.M;
                double acc[2][NT][2];
#pragma unroll
                for (int j = 0; j < NT; ++j) acc[0][j][0] = acc[0][j][1] = acc[1][j][0] = acc[1][j][1] = 0.0;
                for (int kc = 0; kc < nkc; ++kc, ++s) {
                    const int slot = (int)(s % ST);
                    mbar_wait(full + slot, (s / ST) & 1);
                    const double *as = As + slot * GE::SA + (8 * warp + fr) * PADK + fk;
                    const double *bs = Bs + slot * GE::SB + fr * PADK + fk;
#pragma unroll
                    for (int kk = 0; kk < BK; kk += 4) {
                        double bf[NT];
#pragma unroll
                        for (int j = 0; j < NT; ++j) bf[j] = bs[j * 8 * PADK + kk];
                        const double a0 = as[kk], a1 = as[64 * PADK + kk];
#pragma unroll
                        for (int j = 0; j < NT; ++j)
                            if (j < gr.nc) {
                                if (v0) dmma(acc[0][j][0], acc[0][j][1], a0, bf[j]);
                                if (v1) dmma(acc[1][j][0], acc[1][j][1], a1, bf[j]);
                            }
                    }
                    mbar_arrive(empty + slot);
                }
                // park the C tile QP-major (fragment: row fr, cols 2fk, 2fk+1 of each 8x8 tile)
                mbar_wait(cs_empty, (blk & 1) ^ 1);
#pragma unroll
                for (int j = 0; j < NT; ++j)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (j < gr.nc) {
                            Cs[(8 * j + 2 * fk + h) * LDC + 8 * warp + fr] = acc[0][j][h];
                            Cs[(8 * j + 2 * fk + h) * LDC + 8 * (warp + 8) + fr] = acc[1][j][h];
                        }
                    }
                mbar_arrive(cs_full);
                ++blk;
            }
        }
    } else if (warp < kMathW + kProdW) {   // ----------------------------------- producer warps
        const int pt = tid - 32 * kMathW;
        uint32_t s = 0;
        for (int64_t g = blockIdx.x; g < args.ngroups; g += gridDim.x) {
            const Group gr = group_of(args, g);
            if (gr.nq == 0) continue;
            for (int mb = 0; mb < nmb; ++mb) {
                const int64_t m0 = (int64_t)mb * kBlkM;
                const int rows = (int)(args.M - m0 < kBlkM ? args.M - m0 : kBlkM);
                for (int kc = 0; kc < nkc; ++kc, ++s) {
                    const int slot = (int)(s % ST);
                    mbar_wait(empty + slot, ((s / ST) & 1) ^ 1);
                    double *as = As + slot * GE::SA;
                    const double *ag = args.Aop + m0 * args.lda + (int64_t)kc * BK;
                    for (int i = pt; i < rows * (BK / 2); i += 32 * kProdW) {
                        const int r = i / (BK / 2), c = (i % (BK / 2)) * 2;
                        cp16(as + r * PADK + c, ag + r * args.lda + c);
                    }
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
    } else {   // -------------------------------------------------------------- epilogue warps
        const int wid = warp - kMathW - kProdW;
        const OuterA o = PASS == 0 ? outer_a(args.a, MODE_SOLVE) : OuterA{0, 0.0};
        const double avg_w = PASS == 1 ? avg_weight(args.b, MODE_SOLVE) : 0.0;
        uint32_t blk = 0;
        for (int64_t g = blockIdx.x; g < args.ngroups; g += gridDim.x) {
            const Group gr = group_of(args, g);
            if (gr.nq == 0) continue;
            for (int mb = 0; mb < nmb; ++mb) {
                mbar_wait(cs_full, blk & 1);
                const int64_t m0 = (int64_t)mb * kBlkM;
                if (PASS == 0)
                    epi_block_a(args, Cs, m0, gr, wid, kEpiW, lane, o);
                else
                    epi_block_b(args, Cs, m0, gr, wid, kEpiW, lane, avg_w);
                mbar_arrive(cs_empty);
                ++blk;
            }
        }
    }
}

// Pass A reads a (128 x 32) A chunk per (block, chunk) and reuses it over 7 octets (56 QPs);
// pass B has a single row block (n <= 128 typical) and 4-octet groups, two per CTA, so the
// epilogue of a CTA's first group overlaps the math of its second.
constexpr int kNTA = 7, kNTB = 4;

int g_num_sms = 0;   // grid cap: the SM count, or DUQUAD_BATCHED_CTAS (tests: several groups per CTA)

template <int PASS, int NT>
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
    const int64_t base = (a.ncol8 + NT - 1) / NT;
    const int64_t nctas = base < g_num_sms ? base : g_num_sms;
    a.ngroups = (base + nctas - 1) / nctas * nctas;
    k_batched<PASS, NT><<<(unsigned)nctas, kThreadsB, Geo<NT>::SMEM, s>>>(a);
    return cudaGetLastError();
}

template <int PASS, int NT>
cudaError_t configure_t() {
    return cudaFuncSetAttribute(k_batched<PASS, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)Geo<NT>::SMEM);
}

}  // namespace

cudaError_t configure_batched_kernels() {
    cudaError_t e;
    if ((e = configure_t<0, kNTA>())) return e;
    return configure_t<1, kNTB>();
}

cudaError_t launch_batched(const BatchedArgs &a, int pass, int mode, cudaStream_t s) {
    if (a.N <= 0 || a.M <= 0) return cudaSuccess;
    if (mode != MODE_SOLVE) return cudaErrorInvalidValue;   // the batched path runs solve passes only
    return pass == 0 ? launch_t<0, kNTA>(a, s) : launch_t<1, kNTB>(a, s);
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
