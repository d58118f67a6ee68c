// Microbenchmark: dependent-chain latency of DFMA / DMUL / DADD / MUFU.RCP64H / SHFL(f64)
// and FP64 throughput vs warps per SM, on one SM.  nvcc -arch=sm_100a fp64_lat.cu
#include <cstdio>
__global__ void lat(double* out, long long* cyc, double a, double b, int iters) {
    double x = a + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) x = fma(x, b, a);
    }
    long long t1 = clock64();
    double y = x;
    long long t2 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) y = __shfl_sync(0xffffffffu, y, (threadIdx.x + 1) & 31);
    }
    long long t3 = clock64();
    double z = y;
    long long t4 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            double r;
            asm volatile("{.reg .b32 hi, lo; mov.b64 {lo,hi}, %1; rcp.approx.ftz.f64 %0, %1;}" : "=d"(r) : "d"(z));
            z = r + 1.0;
        }
    }
    long long t5 = clock64();
    if (threadIdx.x == 0) {
        cyc[0] = (t1 - t0) / (iters * 16);
        cyc[1] = (t3 - t2) / (iters * 16);
        cyc[2] = (t5 - t4) / (iters * 16);
    }
    out[threadIdx.x] = x + y + z;
}
__global__ void thr(double* out, long long* cyc, double a, double b, int iters) {
    double x0 = a + threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        x0 = fma(x0, b, a); x1 = fma(x1, b, a); x2 = fma(x2, b, a); x3 = fma(x3, b, a);
        x4 = fma(x4, b, a); x5 = fma(x5, b, a); x6 = fma(x6, b, a); x7 = fma(x7, b, a);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[3 + blockDim.x / 32] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 1 << 20); cudaMallocManaged(&cyc, 64 * 8);
    lat<<<1, 32>>>(out, cyc, 1e-3, 0.999, 1000);
    cudaDeviceSynchronize();
    printf("dependent DFMA latency: %lld cycles\nSHFL f64 (2x SHFL) chain: %lld cycles\nrcp.approx f64 + DADD chain: %lld cycles\n", cyc[0], cyc[1], cyc[2]);
    for (int w = 1; w <= 16; w *= 2) {
        thr<<<1, 32 * w>>>(out, cyc, 1e-3, 0.999, 10000);
        cudaDeviceSynchronize();
        long long c = cyc[3 + w];
        printf("warps/SM %2d, 8 indep chains/warp: %.2f DFMA warp-instr per cycle per SM\n", w, (double)w * 8 * 10000 / c);
    }
    return 0;
}
