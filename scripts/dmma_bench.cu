// DMMA.8x8x4 issue-model microbenchmark: W warps per SM sub-partition, A independent accumulators
// per warp, registers only.  Prints DMMA/cycle/SMSP.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int A>
__global__ void kb(double *out, int iters, double a, double b) {
    double c[A][2];
#pragma unroll
    for (int i = 0; i < A; ++i) c[i][0] = c[i][1] = threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < A; ++i) dmma(c[i][0], c[i][1], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < A; ++i) s += c[i][0] + c[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int A>
void run(int wps) {
    double *o;
    cudaMalloc(&o, 148 * 1024 * 8);
    int iters = 20000 / A * 4;
    kb<A><<<148, 128 * wps>>>(o, 10, 1.0, 1.0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kb<A><<<148, 128 * wps>>>(o, iters, 1.0, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double dm = (double)iters * A * wps;            // per SMSP
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("warps/SMSP %d acc/warp %2d: %.3f ms, %.2f cycles/DMMA/SMSP (at %.0f MHz), %.1f TFLOP/s\n", wps, A, ms,
           ms * 1e-3 * clk * 1e3 / dm, clk / 1e3, dm * 4 * 148 * 512 / (ms * 1e-3) / 1e12);
    cudaFree(o);
}
int main() {
    for (int w : {1, 2, 3, 4, 6, 8}) { run<4>(w); run<8>(w); run<14>(w); run<28>(w); }
    return 0;
}
