// Microbenchmark: the symmetric near-field ring step (k_p2p_sym's rotate_ring4)
// in isolation -- registers only, no item bookkeeping -- to see what FP64-pipe
// fraction the instruction mix itself reaches, and variants of it.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o ring4 ring4.cu
// Prints, per variant, ns per launch and the FP64 pipe fraction implied by
// 22 FP64 instructions per unordered pair at 64 lanes/clk/SM and the SM clock.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>

constexpr int kTabN = 60 * 128 + 1;
__constant__ double c_p[4] = {5.415212348123814e-03, 1.4662262387636998e-05,
                              2.6466433582090788e-08, 3.5830355923967645e-11};

__device__ __forceinline__ double rcp_fast(double x) {
    const unsigned hi = max((unsigned)__double2hiint(x), 0x05D00000u);
    x = __hiloint2double((int)hi, __double2loint(x));
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    e = fma(e, e, e);
    return fma(y, e, y);
}

struct SymExp {
    double q;
    unsigned hi;
};

// TAB: 0 = 60 KB table 2^(n/128); 1 = 1 KB table 2^(j/128), exponent added as an integer
// ABL (ablations, wrong numerics, cost probes only): 1 no shuffles, 2 no table
// load, 4 no MUFU (seed from an FMA), 8 no integer clamps
template <int N, int TAB, int ABL = 0, int ORD = 0>
__device__ __forceinline__ void pair_kernels(const double (&dx)[N], const double (&dy)[N], double (&K)[N],
                                             SymExp q2, const double* __restrict__ tab) {
    double r2[N];
#pragma unroll
    for (int k = 0; k < N; ++k) r2[k] = fma(dy[k], dy[k], dx[k] * dx[k]);
    const double kShift0 = 6755399441055744.0;
    double sr0[N];
    int ti0[N];
    if (ORD == 1) {  // exp range reduction before the reciprocal
#pragma unroll
        for (int k = 0; k < N; ++k) {
            const unsigned hi = min((unsigned)__double2hiint(r2[k]), q2.hi);
            const double r2c = __hiloint2double((int)hi, __double2loint(r2[k]));
            const double t = fma(r2c, q2.q, kShift0);
            ti0[k] = __double2loint(t);
            sr0[k] = fma(r2c, q2.q, kShift0 - t);
        }
    }
#pragma unroll
    for (int k = 0; k < N; ++k) {
        if (ABL & 4) {
            const double y = fma(r2[k], -1e-3, 2.0);
            double e = fma(-r2[k], y, 1.0);
            e = fma(e, e, e);
            K[k] = fma(y, e, y);
        } else if (ABL & 8) {
            double y;
            asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2[k]));
            double e = fma(-r2[k], y, 1.0);
            e = fma(e, e, e);
            K[k] = fma(y, e, y);
        } else {
            K[k] = rcp_fast(r2[k]);
        }
    }
    const double kShift = 6755399441055744.0;
    double sr[N], pp[N];
    int ti[N];
    if (ORD == 1) {
#pragma unroll
        for (int k = 0; k < N; ++k) {
            sr[k] = sr0[k];
            ti[k] = ti0[k];
        }
    } else {
#pragma unroll
        for (int k = 0; k < N; ++k) {
            const unsigned hi = (ABL & 8) ? 0u : min((unsigned)__double2hiint(r2[k]), q2.hi);
            const double r2c = (ABL & 8) ? r2[k] : __hiloint2double((int)hi, __double2loint(r2[k]));
            const double t = fma(r2c, q2.q, kShift);
            ti[k] = __double2loint(t);
            sr[k] = fma(r2c, q2.q, kShift - t);
        }
    }
#pragma unroll
    for (int k = 0; k < N; ++k) pp[k] = fma(c_p[3], sr[k], c_p[2]);
#pragma unroll
    for (int k = 0; k < N; ++k) pp[k] = fma(pp[k], sr[k], c_p[1]);
#pragma unroll
    for (int k = 0; k < N; ++k) pp[k] = fma(pp[k], sr[k], c_p[0]);
#pragma unroll
    for (int k = 0; k < N; ++k) {
        double T;
        if (ABL & 2) {
            T = __hiloint2double(ti[k] | 0x3ff00000, 0);
        } else if (TAB == 0) {
            T = tab[ti[k]];
        } else {
            const double b = tab[ti[k] & 127];
            T = __hiloint2double(__double2hiint(b) + ((ti[k] >> 7) << 20), __double2loint(b));
        }
        const double e = fma(T, sr[k] * pp[k], T);
        K[k] = fma(-K[k], e, K[k]);
    }
}

// V: 0 = ring4 as in k_p2p_sym; 1 = eight residents (two ring4 halves share one rotating source)
template <int TAB, int V, int MINB, int ABL = 0, int BT = 256, int UNR = 2, int ORD = 0>
__global__ void __launch_bounds__(BT, MINB) k_ring(const double* __restrict__ pos, const double* __restrict__ gtab,
                                                    double* out, int reps, double q2v) {
    extern __shared__ double tab_s[];
    const int ntab = TAB == 0 ? kTabN : 128;
    for (int i = threadIdx.x; i < ntab; i += blockDim.x) tab_s[i] = gtab[TAB == 0 ? i : kTabN - 128 + i];
    __syncthreads();
    const double* tab = TAB == 0 ? tab_s + (kTabN - 1) : tab_s;
    SymExp q2;
    q2.q = 128.0 * q2v;
    q2.hi = (unsigned)__double2hiint(7680.0 / -q2.q);
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    constexpr int NR = V == 1 ? 8 : (V == 2 ? 6 : (V == 3 ? 2 : 4));
    __shared__ double4 rot[8][32];  // V == 4: the rotating chunk's (x, y, g) per warp
    if (V == 4) {
        rot[threadIdx.x >> 5][lane] = make_double4(pos[(gw * 64 + 200 + lane) % 4096 * 2],
                                                   pos[(gw * 64 + 200 + lane) % 4096 * 2 + 1], 0.5, 0.0);
        __syncwarp();
    }
    const double4* rw = rot[threadIdx.x >> 5];
    double ax[NR], ay[NR], ag[NR], u[NR], v[NR];
#pragma unroll
    for (int k = 0; k < NR; ++k) {
        ax[k] = pos[(gw * 64 + k * 8 + lane) % 4096 * 2];
        ay[k] = pos[(gw * 64 + k * 8 + lane) % 4096 * 2 + 1];
        ag[k] = 1.0 + 1e-3 * k;
        u[k] = v[k] = 0.0;
    }
    double bx = pos[(gw * 64 + 200 + lane) % 4096 * 2], by = pos[(gw * 64 + 200 + lane) % 4096 * 2 + 1];
    double bg = 0.5, ub = 0.0, vb = 0.0;
    const int from = (lane + 1) & 31;
    for (int r = 0; r < reps; ++r) {
#pragma unroll(UNR)
        for (int st = 0; st < 32; ++st) {
            if (V == 3) {  // two residents
                double dx[2], dy[2], K[2];
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    dx[k] = ax[k] - bx;
                    dy[k] = ay[k] - by;
                }
                pair_kernels<2, TAB, ABL>(dx, dy, K, q2, tab);
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const double ca = bg * K[k], cb = ag[k] * K[k];
                    u[k] = fma(-ca, dy[k], u[k]);
                    v[k] = fma(ca, dx[k], v[k]);
                    ub = fma(cb, dy[k], ub);
                    vb = fma(-cb, dx[k], vb);
                }
            } else if (V == 2) {  // six residents: chains of 4 + 2
                {
                    double dx[4], dy[4], K[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        dx[k] = ax[k] - bx;
                        dy[k] = ay[k] - by;
                    }
                    pair_kernels<4, TAB, ABL, ORD>(dx, dy, K, q2, tab);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const double ca = bg * K[k], cb = ag[k] * K[k];
                        u[k] = fma(-ca, dy[k], u[k]);
                        v[k] = fma(ca, dx[k], v[k]);
                        ub = fma(cb, dy[k], ub);
                        vb = fma(-cb, dx[k], vb);
                    }
                }
                {
                    double dx[2], dy[2], K[2];
#pragma unroll
                    for (int k = 0; k < 2; ++k) {
                        dx[k] = ax[4 + k] - bx;
                        dy[k] = ay[4 + k] - by;
                    }
                    pair_kernels<2, TAB, ABL>(dx, dy, K, q2, tab);
#pragma unroll
                    for (int k = 0; k < 2; ++k) {
                        const double ca = bg * K[k], cb = ag[4 + k] * K[k];
                        u[4 + k] = fma(-ca, dy[k], u[4 + k]);
                        v[4 + k] = fma(ca, dx[k], v[4 + k]);
                        ub = fma(cb, dy[k], ub);
                        vb = fma(-cb, dx[k], vb);
                    }
                }
            } else if (V == 4) {
                const double4 b = rw[(lane + st) & 31];
                double dx[4], dy[4], K[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    dx[k] = ax[k] - b.x;
                    dy[k] = ay[k] - b.y;
                }
                pair_kernels<4, TAB, ABL, ORD>(dx, dy, K, q2, tab);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const double ca = b.z * K[k], cb = ag[k] * K[k];
                    u[k] = fma(-ca, dy[k], u[k]);
                    v[k] = fma(ca, dx[k], v[k]);
                    ub = fma(cb, dy[k], ub);
                    vb = fma(-cb, dx[k], vb);
                }
            } else if (V == 0) {
                double dx[4], dy[4], K[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    dx[k] = ax[k] - bx;
                    dy[k] = ay[k] - by;
                }
                pair_kernels<4, TAB, ABL, ORD>(dx, dy, K, q2, tab);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const double ca = bg * K[k], cb = ag[k] * K[k];
                    u[k] = fma(-ca, dy[k], u[k]);
                    v[k] = fma(ca, dx[k], v[k]);
                    ub = fma(cb, dy[k], ub);
                    vb = fma(-cb, dx[k], vb);
                }
            } else {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    double dx[4], dy[4], K[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        dx[k] = ax[4 * h + k] - bx;
                        dy[k] = ay[4 * h + k] - by;
                    }
                    pair_kernels<4, TAB, ABL, ORD>(dx, dy, K, q2, tab);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const double ca = bg * K[k], cb = ag[4 * h + k] * K[k];
                        u[4 * h + k] = fma(-ca, dy[k], u[4 * h + k]);
                        v[4 * h + k] = fma(ca, dx[k], v[4 * h + k]);
                        ub = fma(cb, dy[k], ub);
                        vb = fma(-cb, dx[k], vb);
                    }
                }
            }
            if (V == 4) {
                ub = __shfl_sync(0xffffffffu, ub, from);
                vb = __shfl_sync(0xffffffffu, vb, from);
            } else if (ABL & 1) {
                bx += 1e-9;
                by -= 1e-9;
            } else {
                bx = __shfl_sync(0xffffffffu, bx, from);
                by = __shfl_sync(0xffffffffu, by, from);
                bg = __shfl_sync(0xffffffffu, bg, from);
                ub = __shfl_sync(0xffffffffu, ub, from);
                vb = __shfl_sync(0xffffffffu, vb, from);
            }
        }
    }
    double s = ub + vb;
#pragma unroll
    for (int k = 0; k < NR; ++k) s += u[k] + v[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main(int argc, char** argv) {
    const int reps = argc > 1 ? atoi(argv[1]) : 200;
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    std::vector<double> hp(8192), ht(kTabN);
    srand(1);
    const double h = 2.0 / 1024;
    for (int i = 0; i < 4096; ++i) {  // a 64 x 64 lattice patch
        hp[2 * i] = (i % 64) * h;
        hp[2 * i + 1] = (i / 64) * h;
    }
    for (int i = 0; i < kTabN; ++i) ht[i] = std::exp2((double)(i - (kTabN - 1)) / 128.0);
    double *dp, *dt, *out;
    cudaMalloc(&dp, 8 * 8192);
    cudaMalloc(&dt, 8 * kTabN);
    cudaMalloc(&out, 8 * 148 * 4 * 512);
    cudaMemcpy(dp, hp.data(), 8 * 8192, cudaMemcpyHostToDevice);
    cudaMemcpy(dt, ht.data(), 8 * kTabN, cudaMemcpyHostToDevice);
    const double sigma = h / 0.8, q2 = -1.4426950408889634 / (2 * sigma * sigma);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, auto kern, int smem, int minb, int npairs_per_step, int bt = 256) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int grid = 148 * minb;
        kern<<<grid, bt, smem>>>(dp, dt, out, 2, q2);
        cudaEventRecord(e0);
        kern<<<grid, bt, smem>>>(dp, dt, out, reps, q2);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double pairs = (double)grid * bt * reps * 32 * npairs_per_step;  // lane-pairs
        const double fp64 = pairs * 22;
        const double peak = 64.0 * 148 * clk_khz * 1e3;  // FP64 lanes/s at the rated clock
        printf("%-34s %8.3f ms  %.3f Gpair/s  fp64 frac %.3f  (%s)\n", name, ms, pairs / ms / 1e6,
               fp64 / (ms * 1e-3) / peak, cudaGetErrorString(cudaGetLastError()));
    };
    run("ring4 60KB table MINB2", k_ring<0, 0, 2>, kTabN * 8, 2, 4);
    run("ring4 1KB table MINB2", k_ring<1, 0, 2>, 128 * 8, 2, 4);
    run("ring8 60KB table MINB1", k_ring<0, 1, 1>, kTabN * 8, 1, 8);
    run("ring8 1KB table MINB1", k_ring<1, 1, 1>, 128 * 8, 1, 8);
    run("ring8 1KB table MINB2", k_ring<1, 1, 2>, 128 * 8, 2, 8);
    run("ring4 1KB table MINB3", k_ring<1, 0, 3>, 128 * 8, 3, 4);
    run("ring4 abl no-shfl", k_ring<0, 0, 2, 1>, kTabN * 8, 2, 4);
    run("ring4 abl no-lds", k_ring<0, 0, 2, 2>, kTabN * 8, 2, 4);
    run("ring4 abl no-mufu", k_ring<0, 0, 2, 4>, kTabN * 8, 2, 4);
    run("ring4 abl no-shfl,lds,mufu", k_ring<0, 0, 2, 7>, kTabN * 8, 2, 4);
    run("ring8 384thr MINB1", k_ring<0, 1, 1, 0, 384>, kTabN * 8, 1, 8, 384);
    run("ring6 384thr MINB1", k_ring<0, 2, 1, 0, 384>, kTabN * 8, 1, 6, 384);
    run("ring6 256thr MINB1", k_ring<0, 2, 1, 0, 256>, kTabN * 8, 1, 6, 256);
    run("ring4 256thr MINB1", k_ring<0, 0, 1, 0, 256>, kTabN * 8, 1, 4, 256);
    run("ring4 smem-positions MINB2", k_ring<0, 4, 2, 0, 256>, kTabN * 8, 2, 4, 256);
    run("ring4 MINB2 unroll1", k_ring<0, 0, 2, 0, 256, 1>, kTabN * 8, 2, 4, 256);
    run("ring4 MINB2 unroll4", k_ring<0, 0, 2, 0, 256, 4>, kTabN * 8, 2, 4, 256);
    run("ring4 MINB2 exp-first", k_ring<0, 0, 2, 0, 256, 2, 1>, kTabN * 8, 2, 4, 256);
    run("ring4 MINB2 exp-first unroll1", k_ring<0, 0, 2, 0, 256, 1, 1>, kTabN * 8, 2, 4, 256);
    run("ring2 256thr MINB2", k_ring<0, 3, 2, 0, 256>, kTabN * 8, 2, 2, 256);
    run("ring2 256thr MINB1", k_ring<0, 3, 1, 0, 256>, kTabN * 8, 1, 2, 256);
    run("ring8 abl no-shfl,lds,mufu", k_ring<0, 1, 1, 7>, kTabN * 8, 1, 8);
    return 0;
}
