// Microbenchmark: FP64 pipe throughput of DFMA, DMUL, DADD and of DFMA mixed
// with MUFU.RCP64H (1 per K FP64 ops), 16 warps/SM, 8 independent chains.
#include <cstdio>
template <int MODE>
__global__ void k(double* out, int iters, double a, double b) {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = a + threadIdx.x + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) x[i] = fma(x[i], b, a);
            if (MODE == 1) x[i] = x[i] * b;
            if (MODE == 2) x[i] = x[i] + b;
            if (MODE == 3) {  // 11 DFMA + 1 rcp.approx per element-step
#pragma unroll
                for (int j = 0; j < 11; ++j) x[i] = fma(x[i], b, a);
                double r;
                asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x[i]));
                x[i] = r + x[i];
            }
        }
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    double* out; cudaMalloc(&out, 148 * 512 * 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char* names[4] = {"DFMA", "DMUL", "DADD", "11 DFMA + 1 RCP64H + 1 DADD"};
    for (int mode = 0; mode < 4; ++mode) {
        const int iters = mode == 3 ? 400 : 4000;
        auto run = [&] {
            if (mode == 0) k<0><<<148 * 2, 256>>>(out, iters, 1e-3, 0.999);
            if (mode == 1) k<1><<<148 * 2, 256>>>(out, iters, 1e-3, 0.999);
            if (mode == 2) k<2><<<148 * 2, 256>>>(out, iters, 1e-3, 0.999);
            if (mode == 3) k<3><<<148 * 2, 256>>>(out, iters, 1e-3, 0.999);
        };
        run();
        cudaEventRecord(e0); run(); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double ops = 148.0 * 2 * 256 * iters * 8 * (mode == 3 ? 13 : 1);
        printf("%-30s %.2f G FP64-class instr/s per SM-cycle-equiv: %.1f T ops/s\n", names[mode],
               ops / ms / 1e6, ops / ms / 1e9);
    }
    return 0;
}
