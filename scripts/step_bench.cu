// Microbenchmark: what in the byte-floor Q-role step loop costs time on B200.  Each variant
// streams 2 GiB through a per-thread cp.async ring (6 x 32 KB per CTA, 148 CTAs x 512 threads),
// adding one ingredient of the real loop at a time:
//   V0 plain stream (sum)            V1 + row dot and column sums (16 DFMA, 8+8 registers)
//   V2 + warp_sum of the row dot and a lane-0 store per step
//   V3 + rows of 16384 doubles (32 KB of a 128 KB row per step) instead of contiguous chunks
//   V4 + two rows per step, interleaved (ILP 2)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o step_bench step_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void waitg() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ double wsum(double s) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

constexpr int S = 6, V = 4, T = 512;

template <int VAR>
__global__ void __launch_bounds__(T, 1) k_step(const double *__restrict__ src, int64_t steps, const double *y,
                                               double *out) {
    extern __shared__ __align__(128) uint8_t sm[];
    const int tid = threadIdx.x, lane = tid & 31;
    const double2 *ring = (const double2 *)sm + tid;
    const uint32_t ru = su32(ring);
    // step s reads 4096 doubles: contiguous (VAR < 3) or the first/second 4096 of row s of a
    // 16384-wide matrix block owned by this CTA
    const int64_t ld = 16384;
    const double *base = src + (int64_t)blockIdx.x * steps * 4096;
    auto addr = [&](int64_t st) -> const double * {
        if (VAR < 3) return base + st * 4096;
        return src + ((int64_t)blockIdx.x * steps + st) * (ld / 2);   // first 32 KB of 64 KB rows
    };
    int64_t is = 0;
    int ps = 0;
    auto issue = [&]() {
        if (is < steps) {
            const double *p = addr(is);
#pragma unroll
            for (int k = 0; k < V; ++k) cp16(ru + (uint32_t)((ps * V + k) * T) * 16, p + 2 * tid + 1024 * k);
        }
        commit();
        ++is;
        if (++ps == S) ps = 0;
    };
    for (int t = 0; t < S; ++t) issue();
    double yv[8], acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        yv[e] = y[e * 512 + tid];
        acc[e] = 0.0;
    }
    double tot = 0.0;
    int cs = 0;
    if (VAR < 4) {
        for (int64_t st = 0; st < steps; ++st) {
            const double yr = y[(st & 4095)];
            waitg<S - 1>();
            double q[8];
#pragma unroll
            for (int k = 0; k < V; ++k) {
                const double2 v = ring[(cs * V + k) * T];
                q[2 * k] = v.x;
                q[2 * k + 1] = v.y;
            }
            issue();
            if (++cs == S) cs = 0;
            if (VAR == 0) {
#pragma unroll
                for (int e = 0; e < 8; ++e) tot += q[e];
            } else {
                double ra = 0.0, rb = 0.0;
#pragma unroll
                for (int e = 0; e < 8; e += 2) {
                    ra = fma(q[e], yv[e], ra);
                    rb = fma(q[e + 1], yv[e + 1], rb);
                    acc[e] = fma(q[e], yr, acc[e]);
                    acc[e + 1] = fma(q[e + 1], yr, acc[e + 1]);
                }
                if (VAR >= 2) {
                    const double r = wsum(ra + rb);
                    if (lane == 0) out[blockIdx.x * steps + st] = r;
                } else {
                    tot += ra + rb;
                }
            }
        }
    } else {
        for (int64_t st = 0; st < steps; st += 2) {
            const double yr0 = y[(st & 4095)], yr1 = y[((st + 1) & 4095)];
            waitg<S - 2>();
            double q0[8], q1[8];
            const int c1 = cs + 1 == S ? 0 : cs + 1;
#pragma unroll
            for (int k = 0; k < V; ++k) {
                const double2 v = ring[(cs * V + k) * T], w = ring[(c1 * V + k) * T];
                q0[2 * k] = v.x;
                q0[2 * k + 1] = v.y;
                q1[2 * k] = w.x;
                q1[2 * k + 1] = w.y;
            }
            issue();
            issue();
            cs = c1 + 1 == S ? 0 : c1 + 1;
            double ra = 0.0, rb = 0.0;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                ra = fma(q0[e], yv[e], ra);
                rb = fma(q1[e], yv[e], rb);
                acc[e] = fma(q0[e], yr0, acc[e]);
                acc[e] = fma(q1[e], yr1, acc[e]);
            }
            // two row sums with one 5-level butterfly + 1 exchange
            double mine = (lane & 16) ? rb : ra, other = (lane & 16) ? ra : rb;
            mine += __shfl_xor_sync(0xffffffffu, other, 16);
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
            if (lane == 0) out[blockIdx.x * steps + st] = mine;
            if (lane == 16) out[blockIdx.x * steps + st + 1] = mine;
        }
    }
    waitg<0>();
#pragma unroll
    for (int e = 0; e < 8; ++e) tot += acc[e];
    if (tot == 123.456) out[0] = tot;
}

int main() {
    const int nsm = 148;
    const size_t total = (size_t)2 << 30;
    double *buf, *out, *y;
    cudaMalloc(&buf, total);
    cudaMemset(buf, 0, total);
    cudaMalloc(&y, 16384 * 8);
    cudaMemset(y, 0, 16384 * 8);
    const int64_t steps = (int64_t)(total / 8 / 4096 / nsm) & ~1LL;
    cudaMalloc(&out, (size_t)nsm * steps * 8 + 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const size_t smem = (size_t)S * V * T * 16;
    auto run = [&](auto kern, const char *name, int64_t steps) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<nsm, T, smem>>>(buf, steps, y, out);
        cudaDeviceSynchronize();
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            kern<<<nsm, T, smem>>>(buf, steps, y, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        const double bytes = (double)nsm * steps * 4096 * 8;
        printf("{\"variant\":\"%s\",\"gbs\":%.1f,\"us_per_step\":%.3f,\"err\":\"%s\"}\n", name, bytes / best / 1e6,
               best * 1e3 / steps, cudaGetErrorString(cudaGetLastError()));
    };
    run(k_step<0>, "V0 plain stream", steps);
    run(k_step<1>, "V1 +16 DFMA", steps);
    run(k_step<2>, "V2 +warp_sum+store", steps);
    run(k_step<3>, "V3 +row-strided", steps / 2);
    run(k_step<4>, "V4 2 rows/step", steps / 2);
    return 0;
}
