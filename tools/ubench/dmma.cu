// Microbenchmark: FP64 tensor-core MMA (mma.sync m8n8k4 f64) throughput on one
// SM / whole GPU, alone and concurrently with DFMA-bound warps.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a dmma.cu
#include <cstdio>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
// role: 0 = DMMA warp, 1 = DFMA warp
__global__ void mix(double* out, int iters, int dmma_warps_per_block) {
    const int warp = threadIdx.x >> 5;
    double a = 1.0 + threadIdx.x * 1e-3, b = 0.999;
    if (warp < dmma_warps_per_block) {
        double c[8][2] = {};
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int k = 0; k < 8; ++k) dmma(c[k][0], c[k][1], a, b);
        }
        double s = 0; for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
        out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    } else {
        double x[8];
        for (int k = 0; k < 8; ++k) x[k] = a + k;
        for (int i = 0; i < iters * 4; ++i) {
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = fma(x[k], b, a);
        }
        double s = 0; for (int k = 0; k < 8; ++k) s += x[k];
        out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    }
}
int main() {
    double* out; cudaMalloc(&out, 148 * 1024 * 8 * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 4000;
    struct Cfg { int threads, dmma_warps; } cfgs[] = {{256, 8}, {512, 16}, {256, 0}, {512, 0}, {512, 8}, {1024, 8}, {1024, 16}};
    for (auto c : cfgs) {
        mix<<<148, c.threads>>>(out, 10, c.dmma_warps);
        cudaEventRecord(e0);
        mix<<<148, c.threads>>>(out, iters, c.dmma_warps);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const int nw = c.threads / 32;
        const double dmma_flop = 148.0 * c.dmma_warps * iters * 8 * 2.0 * 8 * 8 * 4;
        const double dfma_flop = 148.0 * (nw - c.dmma_warps) * 32 * iters * 4 * 8 * 2.0;
        printf("threads %4d dmma warps %2d dfma warps %2d: %.3f ms  DMMA %.1f TF/s  DFMA %.1f TF/s\n", c.threads,
               c.dmma_warps, nw - c.dmma_warps, ms, dmma_flop / ms / 1e9, dfma_flop / ms / 1e9);
    }
    return 0;
}
