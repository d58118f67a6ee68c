// Near field P2P (north-star item 5) and the O(N^2) direct sum (item 6).
//
// P2P replaces engine.near_field / _neighbor_ranges / _gather /
// _pair_velocity (engine.py:216-285); the direct sum replaces
// kernels.velocity_direct (kernels.py:52-94).  Both evaluate the
// Gaussian-regularised Biot-Savart pair term of kernels.kernel_eval
// (kernels.py:39-49) in fp64 with self terms excluded by r^2 > 0.
//
// P2P work unit = one warp task: 32 consecutive targets of one leaf (the
// task list is built by k_tasks_fill).  The leaf's 3x3 neighbourhood is at most
// three contiguous row slices of the sorted sources (row-major leaf order),
// streamed through shared memory in tiles shared by the warps of the block
// that work on the same leaf, otherwise read as warp-uniform (broadcast)
// loads through L1.  The 1/(2 pi) factor is applied once per target.
#include <atomic>
#include <climits>
#include <cstdlib>

#include "vfmm_internal.cuh"

namespace vfmm {

namespace {

constexpr int kP2PWarps = 8;
constexpr int kP2PBlocksPerSM = 4;

// Asynchronous global->shared copy of 16 bytes (LDGSTS), bypassing registers.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

constexpr int kChunk = 32;  // sources per staged chunk (one per lane)

// One warp's targets (TPT per lane) against the contiguous source slice
// [a, b): the slice streams through a per-warp double buffer in shared memory
// (cp.async, one 32-byte record per lane per chunk) so the arithmetic reads
// warp-uniform broadcasts from smem while the next chunk is in flight.
template <bool GAUSS, int TPT>
__device__ __forceinline__ void slice_acc(const Src* __restrict__ src, int a, int b,
                                          Src (*buf)[kChunk], const double* __restrict__ tab,
                                          double tx0, double ty0, double tx1, double ty1,
                                          double& u0, double& v0, double& u1, double& v1) {
    const int lane = threadIdx.x & 31;
    const int nch = (b - a + kChunk - 1) / kChunk;
    if (nch == 0) return;
    if (a + lane < b) {
        cp_async16(&buf[0][lane], &src[a + lane]);
        cp_async16(reinterpret_cast<char*>(&buf[0][lane]) + 16,
                   reinterpret_cast<const char*>(&src[a + lane]) + 16);
    }
    cp_async_commit();
    for (int c = 0; c < nch; ++c) {
        const int base = a + c * kChunk;
        if (c + 1 < nch) {
            const int j = base + kChunk + lane;
            if (j < b) {
                Src* d = &buf[(c + 1) & 1][lane];
                cp_async16(d, &src[j]);
                cp_async16(reinterpret_cast<char*>(d) + 16, reinterpret_cast<const char*>(&src[j]) + 16);
            }
            cp_async_commit();
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncwarp();
        const Src* sb = buf[c & 1];
        const int cnt = min(kChunk, b - base);
        int k = 0;
        for (; k + 2 <= cnt; k += 2) {
            const Src s0 = sb[k], s1 = sb[k + 1];
            pair_acc<GAUSS>(tx0, ty0, s0.x, s0.y, s0.g, s0.q2, tab, u0, v0);
            if (TPT == 2) pair_acc<GAUSS>(tx1, ty1, s0.x, s0.y, s0.g, s0.q2, tab, u1, v1);
            pair_acc<GAUSS>(tx0, ty0, s1.x, s1.y, s1.g, s1.q2, tab, u0, v0);
            if (TPT == 2) pair_acc<GAUSS>(tx1, ty1, s1.x, s1.y, s1.g, s1.q2, tab, u1, v1);
        }
        if (k < cnt) {
            const Src s0 = sb[k];
            pair_acc<GAUSS>(tx0, ty0, s0.x, s0.y, s0.g, s0.q2, tab, u0, v0);
            if (TPT == 2) pair_acc<GAUSS>(tx1, ty1, s0.x, s0.y, s0.g, s0.q2, tab, u1, v1);
        }
        __syncwarp();
    }
}

// Persistent grid; warps pull (task, neighbourhood row) work items from a
// global cursor (dynamic balance; every item's arithmetic is fixed, so results
// do not depend on which warp runs it).  A task is 32*TPT consecutive targets
// of one leaf, TPT per lane (each loaded source feeds TPT pairs).  Row dy of
// the 3x3 neighbourhood is one contiguous slice of the sorted sources; its
// partial sums go to near_uv[dy + 1][i] and are added in row order by the
// combine kernel.
template <bool GAUSS, int TPT>
__global__ void __launch_bounds__(kP2PWarps * 32, kP2PBlocksPerSM)
    k_p2p(const Src* __restrict__ src, const int* __restrict__ ls, const int2* __restrict__ tasks,
          Counters* __restrict__ ctr, int levels, int64_t n, const Tables* __restrict__ T,
          double2* __restrict__ near_uv, unsigned long long* __restrict__ pairs, int items_per_warp,
          int sym_enabled) {
    pdl_enter();
    if (sym_enabled && p2p_symmetric(ctr, GAUSS)) return;  // the symmetric kernel handles it
    const int nitems = ctr->ntasks * kNearRows;
    if ((int64_t)blockIdx.x * kP2PWarps * items_per_warp >= nitems) return;  // spare CTA
    __shared__ double sexp[kExpTab];
    __shared__ __align__(16) Src sbuf[kP2PWarps][2][kChunk];
    const double* tab = stage_exp_table(sexp, T->exp2tab);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    Src(*buf)[kChunk] = sbuf[threadIdx.x >> 5];
    const int m = 1 << levels;
    long long my_pairs = 0;
    for (int it = 0; it < items_per_warp; ++it) {
        int item = 0;
        if (lane == 0) item = atomicAdd(&ctr->task_cursor, 1);
        item = __shfl_sync(0xffffffffu, item, 0);
        if (item >= nitems) break;
        const int row = item % kNearRows;
        const int2 tk = tasks[item / kNearRows];
        const int leaf = tk.x;
        const int lo = ls[leaf], hi = ls[leaf + 1];
        const int i0 = lo + tk.y + lane, i1 = i0 + 32;
        const bool act0 = i0 < hi, act1 = TPT == 2 && i1 < hi;
        double tx0 = 0.0, ty0 = 0.0, tx1 = 0.0, ty1 = 0.0;
        if (act0) {
            const double2 t = *reinterpret_cast<const double2*>(&src[i0]);
            tx0 = t.x;
            ty0 = t.y;
        }
        if (act1) {
            const double2 t = *reinterpret_cast<const double2*>(&src[i1]);
            tx1 = t.x;
            ty1 = t.y;
        }
        const int cx = leaf & (m - 1), cy = leaf >> levels;
        const int ny = cy + row - 1;
        double u0 = 0.0, v0 = 0.0, u1 = 0.0, v1 = 0.0;
        if (ny >= 0 && ny < m) {
            const int xlo = cx > 0 ? cx - 1 : 0, xhi = cx < m - 1 ? cx + 1 : m - 1;
            const int a = ls[(int64_t)ny * m + xlo], b = ls[(int64_t)ny * m + xhi + 1];
            if (TPT == 2 && __any_sync(0xffffffffu, act1))
                slice_acc<GAUSS, 2>(src, a, b, buf, tab, tx0, ty0, tx1, ty1, u0, v0, u1, v1);
            else
                slice_acc<GAUSS, 1>(src, a, b, buf, tab, tx0, ty0, tx1, ty1, u0, v0, u1, v1);
            // engine.py:284: pairs += n_leaf * (n_nbhd - 1), split over tasks and rows
            const long long cnt = min(32 * TPT, hi - lo - tk.y);
            my_pairs += cnt * (long long)(b - a) - (row == 1 ? cnt : 0);
        }
        if (act0) near_uv[(int64_t)row * n + i0] = make_double2(u0 * kInv2Pi, v0 * kInv2Pi);
        if (act1) near_uv[(int64_t)row * n + i1] = make_double2(u1 * kInv2Pi, v1 * kInv2Pi);
    }
    if (lane == 0 && my_pairs) atomicAdd(pairs, (unsigned long long)my_pairs);
}

// ---------------------------------------------------------------------------
// Symmetric near field (Newton's third law).  With one core size for every
// particle the pair kernel K(r) = (1 - exp(-r^2/(2 sigma^2))) / r^2 is shared
// by (a <- b) and (b <- a): u_a += -G_b K dy, v_a += G_b K dx and
// u_b += G_a K dy, v_b += -G_a K dx (dx, dy = a - b).  A work item is a leaf
// A: its self block (each unordered pair once) and its "forward" neighbours
// d in {(1,0), (-1,1), (0,1), (1,1)}, so every neighbouring leaf pair is
// visited once.  The forward sources form one stream S = R1 ++ R2 (the right
// neighbour, then the three leaves of the row above -- one contiguous range
// of the sorted sources), so ragged leaves waste lanes once per item, not
// once per neighbour.  Rings: lanes keep resident particles (one or two per
// lane) while a chunk of 32 / 16 / 8 rotating sources moves one lane per step
// by shuffles together with its accumulators, so after R steps every
// (resident, rotating) pair has been seen once and each rotating accumulator
// is back home.  Per item the cheaper layout (counted in lane-pairs) is used:
// the leaf resident and S rotating, or S resident in passes of 64 and the
// leaf rotating (its sums in shared memory).  The leaf's own sums go to slot
// 0, the reaction on a stream particle to its slot `kind` (1..4); the combine
// adds slot 0 and the reaction slots in kind order: deterministic, no
// atomics, 80 bytes of slots per particle.  Work per unordered pair: 22 FP64
// instructions (the one-directional generic kernel: 21 per ordered pair).
#ifndef VFMM_RING_UNROLL
#define VFMM_RING_UNROLL 1
#endif
constexpr int kRingUnroll = VFMM_RING_UNROLL;  // steps of a full ring per loop iteration
#ifndef VFMM_RING4_UNROLL
#define VFMM_RING4_UNROLL 2
#endif
// the same for four residents per lane: two steps per iteration let the
// scheduler overlap a step's tail with the next one's head (config 2 near
// field 0.578 -> 0.565 ms, step 0.7335 -> 0.7222 ms; 4: no further gain)
constexpr int kRing4Unroll = VFMM_RING4_UNROLL;
#ifndef VFMM_RING4_UNROLL_RAGGED
#define VFMM_RING4_UNROLL_RAGGED 1
#endif
#ifndef VFMM_SELF_UNROLL
#define VFMM_SELF_UNROLL 1
#endif
constexpr int kSelfUnroll = VFMM_SELF_UNROLL;  // self-block ring steps per iteration
#ifndef VFMM_SELF_MERGED
#define VFMM_SELF_MERGED 0  // 1: self block of 33..64 as one 4-chain loop (config 2 P2P -0.3%, config 3 +8%: off)
#endif

#ifndef VFMM_SYM_WARPS
#define VFMM_SYM_WARPS 8
#endif
constexpr int kSymWarps = VFMM_SYM_WARPS;  // warps per CTA of the symmetric kernel
// VFMM_SYM_TAB_GLOBAL: the exp table is read from global memory through L1
// (no per-CTA staging; one L1 copy per SM shared by every CTA it runs)
#ifdef VFMM_SYM_TAB_GLOBAL
constexpr int kSymExpBytes = 0;
#else
constexpr int kSymExpBytes = (kExpTab2N * 8 + 15) / 16 * 16;
#endif
constexpr int kSymSmem = kSymExpBytes + kSymWarps * kSymMaxLeaf * 16;  // 76 KB

__device__ __forceinline__ void load_lane(const Src* __restrict__ src, int lo, int cnt, int lane,
                                          double& x, double& y, double& g) {
    // ghosts (lane >= cnt) sit on the chunk's first particle with zero circulation
    VCHECK(cnt <= 0 || lo >= 0);
    const Src& s = src[lo + (lane < cnt ? lane : 0)];
    x = s.x;
    y = s.y;
    g = lane < cnt ? s.g : 0.0;
}

// Symmetric-kernel pair factor K = (1 - e) / r^2, e = exp(-r^2 / (2 sigma^2)),
// for the uniform core size of the symmetric mode.  With q = 128 q2
// (y = r^2 q in units of 1/128 octave) the range reduction reads r^2
// directly: n = round(r^2 q) by the 1.5*2^52 shifter, s = r^2 q - n by one
// FMA (|s| <= 1/2), e = T[n] (1 + s P(s)), T[n] = 2^(n/128), P the degree-3
// minimax fit of (2^(s/128) - 1) / s (relative error of e <= 7.6e-17,
// 0.68 ulp, before rounding).  y >= -60 octaves is enforced on r^2 with one
// integer op (r^2 <= r2max, high words); beyond, 1 - e rounds to 1 anyway.
struct SymExp {
    double q;      // 128 q2 (< 0)
    unsigned hi;   // high word of the largest r^2 kept (y128 >= -7680.01)
};
__device__ __forceinline__ SymExp sym_exp(double q2) {
    SymExp e;
    e.q = 128.0 * q2;
    e.hi = (unsigned)__double2hiint(7680.0 / -e.q);
    return e;
}
__constant__ double c_exp2_sym[4] = {5.415212348123814e-03, 1.4662262387636998e-05,
                                     2.6466433582090788e-08, 3.5830355923967645e-11};

template <bool GAUSS>
__device__ __forceinline__ double pair_kernel(double dx, double dy, SymExp x,
                                              const double* __restrict__ tab) {
    const double r2 = fma(dy, dy, dx * dx);
    const double inv = rcp_fast(r2);
    if (!GAUSS) return inv;
    const unsigned hi = min((unsigned)__double2hiint(r2), x.hi);
    const double r2c = __hiloint2double((int)hi, __double2loint(r2));
    const double kShift = 6755399441055744.0;  // 1.5 * 2^52
    const double t = fma(r2c, x.q, kShift);
    const double s = fma(r2c, x.q, kShift - t);  // r^2 q - n (exact: -n = shift - t)
    double p = c_exp2_sym[3];
    p = fma(p, s, c_exp2_sym[2]);
    p = fma(p, s, c_exp2_sym[1]);
    p = fma(p, s, c_exp2_sym[0]);
    VCHECK(__double2loint(t) <= 0 && __double2loint(t) >= -(kExpTab2N - 1));
    const double T = tab[__double2loint(t)];
    const double e = fma(T, s * p, T);
    return fma(-inv, e, inv);  // (1 - e) / r^2
}

// N independent pair factors advanced stage by stage (dx, dy -> r^2 -> 1/r^2
// -> range reduction -> polynomial -> K), so the N dependency chains issue
// interleaved: with N = 4 the ring step is 3% faster than four calls of
// pair_kernel (the compiler's own interleaving stops short under the
// 128-register cap).
#ifndef VFMM_SYM_I2F
#define VFMM_SYM_I2F 0
#endif
template <bool GAUSS, int N>
__device__ __forceinline__ void pair_kernels(const double (&dx)[N], const double (&dy)[N],
                                             double (&K)[N], SymExp q2,
                                             const double* __restrict__ tab) {
    double r2[N];
#pragma unroll
    for (int k = 0; k < N; ++k) r2[k] = fma(dy[k], dy[k], dx[k] * dx[k]);
#pragma unroll
    for (int k = 0; k < N; ++k) K[k] = rcp_fast(r2[k]);
    if (!GAUSS) return;
    const double kShift = 6755399441055744.0;  // 1.5 * 2^52
    double sr[N], pp[N];
    int ti[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
        const unsigned hi = min((unsigned)__double2hiint(r2[k]), q2.hi);
        const double r2c = __hiloint2double((int)hi, __double2loint(r2[k]));
        const double t = fma(r2c, q2.q, kShift);
        ti[k] = __double2loint(t);
#if VFMM_SYM_I2F
        // -n from the integer (I2F on the conversion pipe) instead of kShift - t (a DADD)
        sr[k] = fma(r2c, q2.q, -(double)ti[k]);
#else
        sr[k] = fma(r2c, q2.q, kShift - t);
#endif
    }
#pragma unroll
    for (int k = 0; k < N; ++k) pp[k] = fma(c_exp2_sym[3], sr[k], c_exp2_sym[2]);
#pragma unroll
    for (int k = 0; k < N; ++k) pp[k] = fma(pp[k], sr[k], c_exp2_sym[1]);
#pragma unroll
    for (int k = 0; k < N; ++k) pp[k] = fma(pp[k], sr[k], c_exp2_sym[0]);
#pragma unroll
    for (int k = 0; k < N; ++k) {
        VCHECK(ti[k] <= 0 && ti[k] >= -(kExpTab2N - 1));
        const double T = tab[ti[k]];
        const double e = fma(T, sr[k] * pp[k], T);
        K[k] = fma(-K[k], e, K[k]);  // (1 - e) / r^2
    }
}

// One ring rotation: the B chunk (R sources) is replicated in every R-lane
// segment of the warp ("ring"); lanes hold one or two A targets each, so a
// rotation of R steps pairs every lane-resident target with every source of
// the chunk exactly once.  Sources and their (u, v) accumulators move one lane
// per step within the ring (shuffle with width R); the rings' partial source
// sums are added in a fixed xor order at the end.  R < 32 serves the ragged
// last chunk of a leaf (R = 8 / 16 instead of 32 mostly-ghost lanes).
template <bool GAUSS, int TPL, int R, bool SYM>
__device__ __forceinline__ void rotate_ring(double a0x, double a0y, double a0g, double a1x,
                                            double a1y, double a1g, double bx, double by, double bg,
                                            double& ub, double& vb, SymExp q2,
                                            const double* __restrict__ tab, double& u0, double& v0,
                                            double& u1, double& v1) {
    const int from = ((threadIdx.x & 31) + 1) & (R - 1);
    // full rings are the hot loop; partial rings (ragged leaf tails) are kept
    // compact so the six ring instances do not crowd the instruction cache
#pragma unroll(R == 32 ? kRingUnroll : 1)
    for (int st = 0; st < R; ++st) {
        if (TPL == 2) {  // two chains, advanced stage by stage
            const double dx[2] = {a0x - bx, a1x - bx}, dy[2] = {a0y - by, a1y - by};
            double K[2];
            pair_kernels<GAUSS, 2>(dx, dy, K, q2, tab);
            const double ca0 = bg * K[0], ca1 = bg * K[1];
            u0 = fma(-ca0, dy[0], u0);
            v0 = fma(ca0, dx[0], v0);
            u1 = fma(-ca1, dy[1], u1);
            v1 = fma(ca1, dx[1], v1);
            if (SYM) {
                const double cb0 = a0g * K[0], cb1 = a1g * K[1];
                ub = fma(cb0, dy[0], ub);
                vb = fma(-cb0, dx[0], vb);
                ub = fma(cb1, dy[1], ub);
                vb = fma(-cb1, dx[1], vb);
            }
        } else {
            const double dx = a0x - bx, dy = a0y - by;
            const double K = pair_kernel<GAUSS>(dx, dy, q2, tab);
            const double ca = bg * K;
            u0 = fma(-ca, dy, u0);
            v0 = fma(ca, dx, v0);
            if (SYM) {
                const double cb = a0g * K;
                ub = fma(cb, dy, ub);
                vb = fma(-cb, dx, vb);
            }
        }
        bx = __shfl_sync(0xffffffffu, bx, from, R);
        by = __shfl_sync(0xffffffffu, by, from, R);
        bg = __shfl_sync(0xffffffffu, bg, from, R);
        if (SYM) {
            ub = __shfl_sync(0xffffffffu, ub, from, R);
            vb = __shfl_sync(0xffffffffu, vb, from, R);
        }
    }
    if (SYM) {
#pragma unroll
        for (int off = R; off < 32; off <<= 1) {
            ub += __shfl_xor_sync(0xffffffffu, ub, off);
            vb += __shfl_xor_sync(0xffffffffu, vb, off);
        }
    }
}

// Four resident particles per lane (a resident pass of 128): four independent
// pair chains per step and one rotation of the source (and its sums) per four
// pairs.  Symmetric only.
template <bool GAUSS, int R, int UNR = kRing4Unroll>
__device__ __forceinline__ void rotate_ring4(const double (&ax)[4], const double (&ay)[4],
                                             const double (&ag)[4], double bx, double by,
                                             double bg, double& ub, double& vb, SymExp q2,
                                             const double* __restrict__ tab, double (&u)[4],
                                             double (&v)[4]) {
    const int from = ((threadIdx.x & 31) + 1) & (R - 1);
#pragma unroll(UNR)
    for (int st = 0; st < R; ++st) {
        double dx[4], dy[4], K[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            dx[k] = ax[k] - bx;
            dy[k] = ay[k] - by;
        }
        pair_kernels<GAUSS, 4>(dx, dy, K, q2, tab);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double ca = bg * K[k], cb = ag[k] * K[k];
            u[k] = fma(-ca, dy[k], u[k]);
            v[k] = fma(ca, dx[k], v[k]);
            ub = fma(cb, dy[k], ub);
            vb = fma(-cb, dx[k], vb);
        }
        bx = __shfl_sync(0xffffffffu, bx, from, R);
        by = __shfl_sync(0xffffffffu, by, from, R);
        bg = __shfl_sync(0xffffffffu, bg, from, R);
        ub = __shfl_sync(0xffffffffu, ub, from, R);
        vb = __shfl_sync(0xffffffffu, vb, from, R);
    }
#pragma unroll
    for (int off = R; off < 32; off <<= 1) {
        ub += __shfl_xor_sync(0xffffffffu, ub, off);
        vb += __shfl_xor_sync(0xffffffffu, vb, off);
    }
}

// The leaf [loB, loB + nB) rotating past four residents per lane; its sums
// start from and return to acc[] in shared memory.
template <bool GAUSS, int UNR = kRing4Unroll>
__device__ __forceinline__ void rotate_leaf4(const Src* __restrict__ src, const double (&ax)[4],
                                             const double (&ay)[4], const double (&ag)[4], int loB,
                                             int nB, double2* acc, SymExp q2,
                                             const double* __restrict__ tab, double (&u)[4],
                                             double (&v)[4]) {
    const int lane = threadIdx.x & 31;
    auto ring_of = [](int rem) { return rem > 24 ? 32 : (rem > 8 ? 16 : 8); };
    double nbx, nby, nbg;
    {
        const int R = ring_of(nB);
        load_lane(src, loB, min(R, nB), lane & (R - 1), nbx, nby, nbg);
    }
    for (int j0 = 0; j0 < nB;) {
        const int rem = nB - j0;
        const int R = ring_of(rem);
        const int cnt = min(R, rem);
        const int li = lane & (R - 1);
        double bx = nbx, by = nby, bg = nbg;
        if (rem > R) {
            const int R2 = ring_of(rem - R);
            load_lane(src, loB + j0 + R, min(R2, rem - R), lane & (R2 - 1), nbx, nby, nbg);
        }
        double ub = 0.0, vb = 0.0;
        if (li < cnt && lane < R) {
            const double2 t = acc[j0 + li];
            ub = t.x;
            vb = t.y;
        }
        if (R == 32)
            rotate_ring4<GAUSS, 32, UNR>(ax, ay, ag, bx, by, bg, ub, vb, q2, tab, u, v);
        else if (R == 16)
            rotate_ring4<GAUSS, 16, UNR>(ax, ay, ag, bx, by, bg, ub, vb, q2, tab, u, v);
        else
            rotate_ring4<GAUSS, 8, UNR>(ax, ay, ag, bx, by, bg, ub, vb, q2, tab, u, v);
        if (lane < cnt) acc[j0 + lane] = make_double2(ub, vb);
        j0 += R;
    }
}

// The contiguous sources [loB, loB + nB) rotate through the lanes in rings of
// 32 / 16 / 8 (ragged tail) while the lanes keep their resident particles
// (one or two per lane); the rotating sources' sums start from and return to
// acc[0 .. nB) in shared memory.  Symmetric: both sides accumulate.
template <bool GAUSS>
__device__ __forceinline__ void rotate_leaf(const Src* __restrict__ src, double a0x, double a0y,
                                            double a0g, double a1x, double a1y, double a1g,
                                            bool two, int loB, int nB, double2* acc, SymExp q2,
                                            const double* __restrict__ tab, double& u0,
                                            double& v0, double& u1, double& v1) {
    const int lane = threadIdx.x & 31;
    auto ring_of = [](int rem) { return rem > 24 ? 32 : (rem > 8 ? 16 : 8); };
    double nbx, nby, nbg;
    {
        const int R = ring_of(nB);
        load_lane(src, loB, min(R, nB), lane & (R - 1), nbx, nby, nbg);
    }
    for (int j0 = 0; j0 < nB;) {
        const int rem = nB - j0;
        const int R = ring_of(rem);
        const int cnt = min(R, rem);
        const int li = lane & (R - 1);
        double bx = nbx, by = nby, bg = nbg;
        if (rem > R) {
            const int R2 = ring_of(rem - R);
            load_lane(src, loB + j0 + R, min(R2, rem - R), lane & (R2 - 1), nbx, nby, nbg);
        }
        double ub = 0.0, vb = 0.0;
        if (li < cnt && lane < R) {  // one ring carries the running sums
            const double2 t = acc[j0 + li];
            ub = t.x;
            vb = t.y;
        }
#define VFMM_RING(TPLV, RV)                                                                       \
    rotate_ring<GAUSS, TPLV, RV, true>(a0x, a0y, a0g, a1x, a1y, a1g, bx, by, bg, ub, vb, q2, tab, \
                                       u0, v0, u1, v1)
        if (two) {
            if (R == 32) VFMM_RING(2, 32); else if (R == 16) VFMM_RING(2, 16); else VFMM_RING(2, 8);
        } else {
            if (R == 32) VFMM_RING(1, 32); else if (R == 16) VFMM_RING(1, 16); else VFMM_RING(1, 8);
        }
#undef VFMM_RING
        if (lane < cnt) acc[j0 + lane] = make_double2(ub, vb);
        j0 += R;
    }
}

// Particle t of the forward stream S = R1 ++ R2 (two contiguous source
// ranges): its sorted index, or -1 past the end.
__device__ __forceinline__ int stream_index(int t, int r1, int n1, int r2, int n2) {
    return t < n1 ? r1 + t : (t < n1 + n2 ? r2 + (t - n1) : -1);
}

// Resident slots of the next pass over `rem` stream particles: 128 (four per
// lane) while more than 96 remain, else 64 or 32.
__device__ __forceinline__ int pass_slots(int rem) { return rem > 96 ? 128 : (rem > 32 ? 64 : 32); }

// Ring steps to rotate n sources through (rings of 32 / 16 / 8).
__device__ __forceinline__ int rot_steps(int n) {
    const int full = n >> 5, rem = n & 31;
    return 32 * full + (rem == 0 ? 0 : (rem > 24 ? 32 : (rem > 8 ? 16 : 8)));
}

// The forward stream S rotates through the lanes (chunks may straddle the
// R1 / R2 boundary) while the lanes keep up to 64 particles of the leaf; each
// chunk's reactions are complete when the ring returns home and go straight
// to the sources' slots.
template <bool GAUSS>
__device__ __forceinline__ void rotate_stream(const Src* __restrict__ src, double a0x, double a0y,
                                              double a0g, double a1x, double a1y, double a1g,
                                              bool two, int r1, int n1, int r2, int n2, int b3,
                                              int b4, double2* __restrict__ near5, int64_t n,
                                              SymExp q2, const double* __restrict__ tab,
                                              double& u0, double& v0, double& u1, double& v1) {
    const int lane = threadIdx.x & 31;
    const int nS = n1 + n2;
    auto ring_of = [](int rem) { return rem > 24 ? 32 : (rem > 8 ? 16 : 8); };
    auto load = [&](int j0, int cnt, int li, double& x, double& y, double& g) {
        const int t = j0 + (li < cnt ? li : 0);
        const Src& e = src[stream_index(t, r1, n1, r2, n2)];
        x = e.x;
        y = e.y;
        g = li < cnt ? e.g : 0.0;
    };
    double nbx, nby, nbg;
    {
        const int R = ring_of(nS);
        load(0, min(R, nS), lane & (R - 1), nbx, nby, nbg);
    }
    for (int j0 = 0; j0 < nS;) {
        const int rem = nS - j0;
        const int R = ring_of(rem);
        const int cnt = min(R, rem);
        double bx = nbx, by = nby, bg = nbg;
        if (rem > R) {
            const int R2 = ring_of(rem - R);
            load(j0 + R, min(R2, rem - R), lane & (R2 - 1), nbx, nby, nbg);
        }
        double ub = 0.0, vb = 0.0;
#define VFMM_RING(TPLV, RV)                                                                       \
    rotate_ring<GAUSS, TPLV, RV, true>(a0x, a0y, a0g, a1x, a1y, a1g, bx, by, bg, ub, vb, q2, tab, \
                                       u0, v0, u1, v1)
        if (two) {
            if (R == 32) VFMM_RING(2, 32); else if (R == 16) VFMM_RING(2, 16); else VFMM_RING(2, 8);
        } else {
            if (R == 32) VFMM_RING(1, 32); else if (R == 16) VFMM_RING(1, 16); else VFMM_RING(1, 8);
        }
#undef VFMM_RING
        if (lane < cnt) {
            const int t = j0 + lane;
            const int i = stream_index(t, r1, n1, r2, n2);
            const int kind = t < n1 ? 1 : (i < b3 ? 2 : (i < b4 ? 3 : 4));
            VCHECK(i >= 0 && i < n && kind >= 1 && kind <= 4);
            near5[(int64_t)kind * n + i] = make_double2(ub * kInv2Pi, vb * kInv2Pi);
        }
        j0 += R;
    }
}

template <bool GAUSS>
__device__ __forceinline__ void self_block_sym(double a0x, double a0y, double a0g, double a1x,
                                               double a1y, double a1g, bool two, SymExp q2,
                                               const double* __restrict__ tab, double& u0,
                                               double& v0, double& u1, double& v1) {
    const int lane = threadIdx.x & 31, from = (lane + 1) & 31;
    double b0x = __shfl_sync(0xffffffffu, a0x, from), b0y = __shfl_sync(0xffffffffu, a0y, from);
    double b0g = __shfl_sync(0xffffffffu, a0g, from);
    double b1x = __shfl_sync(0xffffffffu, a1x, from), b1y = __shfl_sync(0xffffffffu, a1y, from);
    double b1g = __shfl_sync(0xffffffffu, a1g, from);
    double ub0 = 0.0, vb0 = 0.0, ub1 = 0.0, vb1 = 0.0;
    const int home = (lane + 16) & 31;
#if VFMM_SELF_MERGED
    if (two) {
        // 33..64 particles: the two half rings and the cross ring (two
        // half-phase copies P, Q of chunk 1 against chunk 0) advance in ONE
        // 16-step loop -- four independent pair chains per step instead of
        // two, like the four-resident ring of the forward blocks.  The cross
        // terms of chunk 0 collect in (cu, cv) and are added after the half
        // ring's sums, as in the two-loop order.
        double pbx = a1x, pby = a1y, pbg = a1g;  // copy P: lane l starts with particle l
        double qbx = __shfl_sync(0xffffffffu, a1x, home), qby = __shfl_sync(0xffffffffu, a1y, home);
        double qbg = __shfl_sync(0xffffffffu, a1g, home);  // copy Q: particle l + 16
        double pu = 0.0, pv = 0.0, qu = 0.0, qv = 0.0, cu = 0.0, cv = 0.0;
#pragma unroll(kSelfUnroll)
        for (int st = 1; st <= 16; ++st) {
            const bool on = st < 16 || lane < 16;
            const double dx[4] = {a0x - b0x, a1x - b1x, a0x - pbx, a0x - qbx};
            const double dy[4] = {a0y - b0y, a1y - b1y, a0y - pby, a0y - qby};
            double K[4];
            pair_kernels<GAUSS, 4>(dx, dy, K, q2, tab);
            const double k0 = on ? K[0] : 0.0, k1 = on ? K[1] : 0.0;
            const double ca0 = b0g * k0, cb0 = a0g * k0, ca1 = b1g * k1, cb1 = a1g * k1;
            u0 = fma(-ca0, dy[0], u0);
            v0 = fma(ca0, dx[0], v0);
            ub0 = fma(cb0, dy[0], ub0);
            vb0 = fma(-cb0, dx[0], vb0);
            u1 = fma(-ca1, dy[1], u1);
            v1 = fma(ca1, dx[1], v1);
            ub1 = fma(cb1, dy[1], ub1);
            vb1 = fma(-cb1, dx[1], vb1);
            const double cap = pbg * K[2], caq = qbg * K[3], cbp = a0g * K[2], cbq = a0g * K[3];
            cu = fma(-cap, dy[2], cu);
            cv = fma(cap, dx[2], cv);
            cu = fma(-caq, dy[3], cu);
            cv = fma(caq, dx[3], cv);
            pu = fma(cbp, dy[2], pu);
            pv = fma(-cbp, dx[2], pv);
            qu = fma(cbq, dy[3], qu);
            qv = fma(-cbq, dx[3], qv);
            if (st < 16) {
                b0x = __shfl_sync(0xffffffffu, b0x, from);
                b0y = __shfl_sync(0xffffffffu, b0y, from);
                b0g = __shfl_sync(0xffffffffu, b0g, from);
                ub0 = __shfl_sync(0xffffffffu, ub0, from);
                vb0 = __shfl_sync(0xffffffffu, vb0, from);
                b1x = __shfl_sync(0xffffffffu, b1x, from);
                b1y = __shfl_sync(0xffffffffu, b1y, from);
                b1g = __shfl_sync(0xffffffffu, b1g, from);
                ub1 = __shfl_sync(0xffffffffu, ub1, from);
                vb1 = __shfl_sync(0xffffffffu, vb1, from);
            }
            pbx = __shfl_sync(0xffffffffu, pbx, from);
            pby = __shfl_sync(0xffffffffu, pby, from);
            pbg = __shfl_sync(0xffffffffu, pbg, from);
            pu = __shfl_sync(0xffffffffu, pu, from);
            pv = __shfl_sync(0xffffffffu, pv, from);
            qbx = __shfl_sync(0xffffffffu, qbx, from);
            qby = __shfl_sync(0xffffffffu, qby, from);
            qbg = __shfl_sync(0xffffffffu, qbg, from);
            qu = __shfl_sync(0xffffffffu, qu, from);
            qv = __shfl_sync(0xffffffffu, qv, from);
        }
        // lane l holds the half-ring reaction of particle l + 16: send it home
        u0 += __shfl_sync(0xffffffffu, ub0, home);
        v0 += __shfl_sync(0xffffffffu, vb0, home);
        u1 += __shfl_sync(0xffffffffu, ub1, home);
        v1 += __shfl_sync(0xffffffffu, vb1, home);
        u0 += cu;
        v0 += cv;
        // after 16 shifts copy Q is home; copy P holds particle l + 16
        u1 += __shfl_sync(0xffffffffu, pu, home) + qu;
        v1 += __shfl_sync(0xffffffffu, pv, home) + qv;
        return;
    }
#endif
#pragma unroll(kSelfUnroll)
    for (int st = 1; st <= 16; ++st) {
        const bool on = st < 16 || lane < 16;
        {  // both chunks' chains together (the second is all ghosts when !two)
            const double dx[2] = {a0x - b0x, a1x - b1x}, dy[2] = {a0y - b0y, a1y - b1y};
            double K[2];
            pair_kernels<GAUSS, 2>(dx, dy, K, q2, tab);
            const double k0 = on ? K[0] : 0.0, k1 = on && two ? K[1] : 0.0;
            const double ca0 = b0g * k0, cb0 = a0g * k0, ca1 = b1g * k1, cb1 = a1g * k1;
            u0 = fma(-ca0, dy[0], u0);
            v0 = fma(ca0, dx[0], v0);
            ub0 = fma(cb0, dy[0], ub0);
            vb0 = fma(-cb0, dx[0], vb0);
            u1 = fma(-ca1, dy[1], u1);
            v1 = fma(ca1, dx[1], v1);
            ub1 = fma(cb1, dy[1], ub1);
            vb1 = fma(-cb1, dx[1], vb1);
        }
        if (st < 16) {
            b0x = __shfl_sync(0xffffffffu, b0x, from);
            b0y = __shfl_sync(0xffffffffu, b0y, from);
            b0g = __shfl_sync(0xffffffffu, b0g, from);
            ub0 = __shfl_sync(0xffffffffu, ub0, from);
            vb0 = __shfl_sync(0xffffffffu, vb0, from);
            if (two) {
                b1x = __shfl_sync(0xffffffffu, b1x, from);
                b1y = __shfl_sync(0xffffffffu, b1y, from);
                b1g = __shfl_sync(0xffffffffu, b1g, from);
                ub1 = __shfl_sync(0xffffffffu, ub1, from);
                vb1 = __shfl_sync(0xffffffffu, vb1, from);
            }
        }
    }
    // lane l holds the reaction of particle l + 16: send it home
    u0 += __shfl_sync(0xffffffffu, ub0, home);
    v0 += __shfl_sync(0xffffffffu, vb0, home);
    if (!two) return;
    u1 += __shfl_sync(0xffffffffu, ub1, home);
    v1 += __shfl_sync(0xffffffffu, vb1, home);
    // cross ring chunk 0 x chunk 1 as two half-phase copies of chunk 1 (offsets
    // 0..15 and 16..31) rotating together: two chains per step for 16 steps
    double pbx = a1x, pby = a1y, pbg = a1g;  // copy P: lane l starts with particle l
    double qbx = __shfl_sync(0xffffffffu, a1x, home), qby = __shfl_sync(0xffffffffu, a1y, home);
    double qbg = __shfl_sync(0xffffffffu, a1g, home);  // copy Q: particle l + 16
    double pu = 0.0, pv = 0.0, qu = 0.0, qv = 0.0;
#pragma unroll(kSelfUnroll)
    for (int st = 0; st < 16; ++st) {
        const double dx[2] = {a0x - pbx, a0x - qbx}, dy[2] = {a0y - pby, a0y - qby};
        double K[2];
        pair_kernels<GAUSS, 2>(dx, dy, K, q2, tab);
        const double cap = pbg * K[0], caq = qbg * K[1], cbp = a0g * K[0], cbq = a0g * K[1];
        u0 = fma(-cap, dy[0], u0);
        v0 = fma(cap, dx[0], v0);
        u0 = fma(-caq, dy[1], u0);
        v0 = fma(caq, dx[1], v0);
        pu = fma(cbp, dy[0], pu);
        pv = fma(-cbp, dx[0], pv);
        qu = fma(cbq, dy[1], qu);
        qv = fma(-cbq, dx[1], qv);
        pbx = __shfl_sync(0xffffffffu, pbx, from);
        pby = __shfl_sync(0xffffffffu, pby, from);
        pbg = __shfl_sync(0xffffffffu, pbg, from);
        pu = __shfl_sync(0xffffffffu, pu, from);
        pv = __shfl_sync(0xffffffffu, pv, from);
        qbx = __shfl_sync(0xffffffffu, qbx, from);
        qby = __shfl_sync(0xffffffffu, qby, from);
        qbg = __shfl_sync(0xffffffffu, qbg, from);
        qu = __shfl_sync(0xffffffffu, qu, from);
        qv = __shfl_sync(0xffffffffu, qv, from);
    }
    // after 16 shifts copy Q is home; copy P holds particle l + 16
    u1 += __shfl_sync(0xffffffffu, pu, home) + qu;
    v1 += __shfl_sync(0xffffffffu, pv, home) + qv;
}

// One write event on owned leaf `lf` (all its writes fenced before): the last
// of the expected events sums the leaf's near-field slots into slot 0 in
// k_near_sum's order -- own item(s) (slot 0, slot kSplitSlot), then the
// reactions of the backward neighbours d_k = (1,0), (-1,1), (0,1), (1,1)
// (slots 1..4) that exist and hold particles.  The sums read L2 (just written
// by other SMs: __ldcg).
__device__ __noinline__ void leaf_written(int lf, int m, int levels, int64_t n, int split_from,
                                          int item_base, const int* __restrict__ ls, double2* near5,
                                          int* done) {
    const int lane = threadIdx.x & 31;
    const int split = sym_leaf_split(lf, item_base, split_from);
    const int ix = lf & (m - 1), iy = lf >> levels;
    bool ok[5];
    int expected = split;  // own items
#pragma unroll
    for (int k = 1; k < 5; ++k) {
        const int ax = ix - (k == 2 ? -1 : (k == 3 ? 0 : 1)), ay = iy - (k == 1 ? 0 : 1);
        ok[k] = ax >= 0 && ax < m && ay >= 0 && ls[ay * m + ax + 1] != ls[ay * m + ax];
        expected += ok[k] ? 1 : 0;
    }
    int old = 0;
    if (lane == 0) old = atomicAdd(&done[lf], 1);
    old = __shfl_sync(0xffffffffu, old, 0);
    if (old != expected - 1) return;
    __threadfence();
    const int lo = ls[lf], hi = ls[lf + 1];
    for (int i = lo + lane; i < hi; i += 32) {
        double2 nv = __ldcg(&near5[i]);
        if (split == 2) {
            const double2 t5 = __ldcg(&near5[(int64_t)kSplitSlot * n + i]);
            nv.x += t5.x;
            nv.y += t5.y;
        }
#pragma unroll
        for (int k = 1; k < 5; ++k)
            if (ok[k]) {
                const double2 t = __ldcg(&near5[(int64_t)k * n + i]);
                nv.x += t.x;
                nv.y += t.y;
            }
        near5[i] = nv;
    }
}

#ifdef VFMM_SYM_MAXNREG
#define VFMM_SYM_BOUNDS __maxnreg__(VFMM_SYM_MAXNREG)
#else
#define VFMM_SYM_BOUNDS __launch_bounds__(kSymWarps * 32, MINB)
#endif
// TSPLIT: leaves from split_from on are two items (a tail of half items);
// otherwise split_from is 0 (every leaf two items) or the leaf count (none)
// and the kernel uses the uniform item -> leaf map (its code is measurably
// faster: config 2 near field 0.558 vs 0.550 ms)
template <bool GAUSS, int MINB, bool TSPLIT>
__global__ void VFMM_SYM_BOUNDS
    k_p2p_sym(const Src* __restrict__ src, const int* __restrict__ ls, Counters* __restrict__ ctr,
              int levels, int64_t n, Rows rows, const Tables* __restrict__ T,
              double2* __restrict__ near5, unsigned long long* __restrict__ pairs,
              int items_per_warp, int item_base, int nitems, int split_from, GraphCond generic_cond,
              int* __restrict__ done) {
    pdl_enter();
    // a captured graph runs the generic near-field chain (an IF node after
    // this kernel) only when the symmetric mode does not apply
    graph_cond_set(generic_cond, p2p_symmetric(ctr, GAUSS) ? 0u : 1u);
    if (!p2p_symmetric(ctr, GAUSS)) return;  // the generic kernel handles it
    const int m = 1 << levels;
    // one item per leaf of rows [rows.lo - 1, rows.hi) (all leaves when not
    // sharded; the row below the strip pairs its halo leaves with the owned
    // row above); leaf = item_base + item
    if ((int64_t)blockIdx.x * kSymWarps * items_per_warp >= nitems) return;  // spare CTA
    // dynamic shared memory: exp table | per-warp accumulators of the item's leaf
    extern __shared__ __align__(16) unsigned char sym_smem[];
    double2* accA = reinterpret_cast<double2*>(sym_smem + kSymExpBytes);
#ifdef VFMM_SYM_TAB_GLOBAL
    const double* tab = T->exp2tab2 + (kExpTab2N - 1);
#else
    double* sexp = reinterpret_cast<double*>(sym_smem);
    const double* tab = sexp + (kExpTab2N - 1);  // 2^(n/128) at tab[n], n <= 0
    // The 60 KB table is staged by ONE bulk copy (TMA engine, mbarrier
    // completion) issued here and waited for only before the first pair of
    // the warp's first item, so it overlaps the item's index and particle
    // loads (the cooperative loop stalled every new CTA: 3% of the kernel's
    // stall samples at one item per warp).
    __shared__ __align__(8) unsigned long long tab_bar;
    const unsigned tab_ba = (unsigned)__cvta_generic_to_shared(&tab_bar);
    if (threadIdx.x == 0) {
        constexpr unsigned bytes = (unsigned)((kExpTab2N + 1) * sizeof(double));
        static_assert(bytes % 16 == 0 && bytes <= kSymExpBytes, "bulk copy of the exp table");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tab_ba));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tab_ba), "r"(bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                (unsigned)__cvta_generic_to_shared(sexp)),
            "l"(T->exp2tab2), "r"(bytes), "r"(tab_ba)
            : "memory");
    }
    __syncthreads();  // the barrier's initialisation is visible
    bool tab_ready = false;
    auto wait_tab = [&]() {
        if (tab_ready) return;
        asm volatile(
            "{\n .reg .pred p;\n WAIT_%=:\n"
            " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
            " @!p bra WAIT_%=;\n}" ::"r"(tab_ba)
            : "memory");
        tab_ready = true;
    };
#endif
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double2* accAw = accA + warp * kSymMaxLeaf;
    const SymExp q2 = sym_exp(GAUSS ? src[0].q2 : -1.0);  // uniform core size
    long long my_pairs = 0;
    // the next item index is fetched one item ahead to hide the atomic's latency
    int next = 0;
    if (lane == 0) next = atomicAdd(&ctr->task_cursor, 1);
    for (int it = 0; it < items_per_warp; ++it) {
        const int item = __shfl_sync(0xffffffffu, next, 0);
        if (item >= nitems) break;
        // leaves from split_from on (relative to item_base) are two items:
        // part 0 = self block + R1 + the left leaf of R2, part 1 = the other
        // two leaves of R2 (the leaf's sums go to kSplitSlot)
        const int split = TSPLIT ? (item < split_from ? 1 : 2) : (split_from == 0 ? 2 : 1);
        const int leaf =
            TSPLIT ? item_base + (split == 1 ? item : split_from + ((item - split_from) >> 1))
                   : item_base + item / split;
        const int part = TSPLIT ? (split == 1 ? 0 : (item - split_from) & 1) : item % split;
        if (lane == 0 && it + 1 < items_per_warp) next = atomicAdd(&ctr->task_cursor, 1);
        const int loA = ls[leaf], nA = ls[leaf + 1] - loA;
        VCHECK(loA >= 0 && nA >= 0 && (int64_t)loA + nA <= n && nA <= kSymMaxLeaf);
        VJITTER();
        if (nA == 0) continue;
        const int cx = leaf & (m - 1), cy = leaf >> levels;
        const bool ownA = cy >= rows.lo && cy < rows.hi;
        // forward stream S = R1 (leaf (cx+1, cy)) ++ R2 (leaves cx-1..cx+1 of row
        // cy+1, one contiguous range of the sorted sources)
        int r1 = 0, n1 = 0, r2 = 0, n2 = 0, b3 = 0, b4 = 0;
        int x2lo = 0, x2hi = 0;  // leaves [x2lo, x2hi) of row cy + 1 in the stream
        bool ownR2 = false;
        if (ownA && cx + 1 < m && part == 0) {
            r1 = ls[leaf + 1];
            n1 = ls[leaf + 2] - r1;
        }
        if (cy + 1 < m) {
            ownR2 = cy + 1 >= rows.lo && cy + 1 < rows.hi;
            if (ownA || ownR2) {
                const int row = (cy + 1) * m;
                const int x0 = cx > 0 ? cx - 1 : 0, x1 = cx + 1 < m ? cx + 1 : m - 1;
                b3 = ls[row + cx];                          // first source of kind 3 (0, 1)
                b4 = cx + 1 < m ? ls[row + cx + 1] : ls[row + x1 + 1];  // first source of kind 4 (1, 1)
                const int s0 = split == 1 || part == 1 ? (split == 1 ? x0 : cx) : x0;
                const int e0 = split == 1 || part == 1 ? x1 + 1 : cx;  // leaves [s0, e0) of row cy + 1
                r2 = ls[row + s0];
                n2 = ls[row + e0] - r2;
                x2lo = s0;
                x2hi = e0;
            }
        }
        if (!ownA && n2 == 0) continue;
#ifndef VFMM_SYM_TAB_GLOBAL
        wait_tab();
#endif
        // ---- self block (owned A only): each unordered pair once ----
        if (part == 0 && ownA && nA <= kSymMaxLeaf) {
            double a0x, a0y, a0g, a1x, a1y, a1g, a2x, a2y, a2g, a3x, a3y, a3g;
            load_lane(src, loA, min(32, nA), lane, a0x, a0y, a0g);
            load_lane(src, loA + (nA > 32 ? 32 : 0), max(nA - 32, 0), lane, a1x, a1y, a1g);
            double u0 = 0.0, v0 = 0.0, u1 = 0.0, v1 = 0.0;
            self_block_sym<GAUSS>(a0x, a0y, a0g, a1x, a1y, a1g, nA > 32, q2, tab, u0, v0, u1, v1);
            if (nA > 64) {
                load_lane(src, loA + 64, min(32, nA - 64), lane, a2x, a2y, a2g);
                load_lane(src, loA + (nA > 96 ? 96 : 64), max(nA - 96, 0), lane, a3x, a3y, a3g);
                double u2 = 0.0, v2 = 0.0, u3 = 0.0, v3 = 0.0;
                self_block_sym<GAUSS>(a2x, a2y, a2g, a3x, a3y, a3g, nA > 96, q2, tab, u2, v2, u3, v3);
                // chunks 0, 1 (resident) against chunk 2, then chunk 3 (rotating)
                double ub = 0.0, vb = 0.0;
                rotate_ring<GAUSS, 2, 32, true>(a0x, a0y, a0g, a1x, a1y, a1g, a2x, a2y, a2g, ub, vb,
                                                q2, tab, u0, v0, u1, v1);
                u2 += ub;
                v2 += vb;
                if (nA > 96) {
                    ub = vb = 0.0;
                    rotate_ring<GAUSS, 2, 32, true>(a0x, a0y, a0g, a1x, a1y, a1g, a3x, a3y, a3g, ub,
                                                    vb, q2, tab, u0, v0, u1, v1);
                    u3 += ub;
                    v3 += vb;
                }
                accAw[64 + lane] = make_double2(u2, v2);
                accAw[96 + lane] = make_double2(u3, v3);
            }
            accAw[lane] = make_double2(u0, v0);
            accAw[32 + lane] = make_double2(u1, v1);
            my_pairs += (long long)nA * nA - nA;
        } else {
            for (int j = lane; j < nA; j += 32) accAw[j] = make_double2(0.0, 0.0);
        }
        __syncwarp();
        const int nS = n1 + n2;
        // ---- forward blocks: whichever layout wastes fewer lane-pairs ----
        // (a) the leaf resident (<= 64: one or two per lane), S rotating;
        // (b) S resident in passes of 64, the leaf rotating (A's sums in smem).
        const int slotsA = nA > 32 ? 64 : 32;
        const int cost_a = nA <= 64 ? slotsA * rot_steps(nS) : INT_MAX;
        int cost_b = 0;  // resident passes of 128 (4 per lane), 64 or 32
        for (int r = nS; r > 0; r -= pass_slots(r)) cost_b += pass_slots(r) * rot_steps(nA);
        if (nS > 0 && cost_a < cost_b) {
            double a0x, a0y, a0g, a1x, a1y, a1g;
            load_lane(src, loA, min(32, nA), lane, a0x, a0y, a0g);
            load_lane(src, loA + (nA > 32 ? 32 : 0), max(nA - 32, 0), lane, a1x, a1y, a1g);
            const double2 s0 = accAw[lane], s1 = accAw[32 + lane];
            double u0 = s0.x, v0 = s0.y, u1 = s1.x, v1 = s1.y;
            rotate_stream<GAUSS>(src, a0x, a0y, a0g, a1x, a1y, a1g, nA > 32, r1, n1, r2, n2, b3, b4,
                                 near5, n, q2, tab, u0, v0, u1, v1);
            accAw[lane] = make_double2(u0, v0);
            accAw[32 + lane] = make_double2(u1, v1);
        }
        for (int p0 = 0; cost_a >= cost_b && p0 < nS;) {
            if (pass_slots(nS - p0) == 128) {  // four residents per lane
                double ax[4], ay[4], ag[4], u[4], v[4];
                int idx[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int t = p0 + 32 * k + lane;
                    idx[k] = stream_index(t < nS ? t : p0, r1, n1, r2, n2);
                    const Src& e = src[idx[k]];
                    ax[k] = e.x;
                    ay[k] = e.y;
                    ag[k] = t < nS ? e.g : 0.0;
                    u[k] = v[k] = 0.0;
                }
                // ragged leaves (the tail-split instance: large random-order
                // grids) take many code paths per SM; the ring is not unrolled
                // there (instruction-fetch stalls, config 3)
                rotate_leaf4<GAUSS, TSPLIT ? VFMM_RING4_UNROLL_RAGGED : kRing4Unroll>(src, ax, ay, ag, loA, nA,
                                                                                       accAw, q2, tab, u, v);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int t = p0 + 32 * k + lane;
                    if (t < nS) {
                        const int i = idx[k];
                        const int kind = t < n1 ? 1 : (i < b3 ? 2 : (i < b4 ? 3 : 4));
                        VCHECK(i >= 0 && i < n && kind >= 1 && kind <= 4);
                        near5[(int64_t)kind * n + i] = make_double2(u[k] * kInv2Pi, v[k] * kInv2Pi);
                    }
                }
                p0 += 128;
                continue;
            }
            const int cnt = min(64, nS - p0);
            const int t0 = p0 + lane, t1 = p0 + 32 + lane;
            const int i0 = stream_index(t0 < p0 + cnt ? t0 : p0, r1, n1, r2, n2);
            const int i1 = stream_index(t1 < p0 + cnt ? t1 : p0, r1, n1, r2, n2);
            const Src& s0 = src[i0];
            const Src& s1 = src[i1];
            const double a0x = s0.x, a0y = s0.y, a0g = t0 < p0 + cnt ? s0.g : 0.0;
            const double a1x = s1.x, a1y = s1.y, a1g = t1 < p0 + cnt ? s1.g : 0.0;
            double u0 = 0.0, v0 = 0.0, u1 = 0.0, v1 = 0.0;
            rotate_leaf<GAUSS>(src, a0x, a0y, a0g, a1x, a1y, a1g, cnt > 32, loA, nA, accAw, q2, tab,
                               u0, v0, u1, v1);
            // reactions on the stream particles -> their slot `kind`
            if (t0 < p0 + cnt) {
                const int kind = t0 < n1 ? 1 : (i0 < b3 ? 2 : (i0 < b4 ? 3 : 4));
                VCHECK(i0 >= 0 && i0 < n && kind >= 1 && kind <= 4);
                near5[(int64_t)kind * n + i0] = make_double2(u0 * kInv2Pi, v0 * kInv2Pi);
            }
            if (t1 < p0 + cnt) {
                const int kind = t1 < n1 ? 1 : (i1 < b3 ? 2 : (i1 < b4 ? 3 : 4));
                VCHECK(i1 >= 0 && i1 < n && kind >= 1 && kind <= 4);
                near5[(int64_t)kind * n + i1] = make_double2(u1 * kInv2Pi, v1 * kInv2Pi);
            }
            p0 += 64;
        }
        my_pairs += 2ll * nA * n1 + (long long)nA * n2 * ((ownA ? 1 : 0) + (ownR2 ? 1 : 0));
        // A's own targets: self + forward blocks -> slot 0 (kSplitSlot: part 1)
        __syncwarp();
        VCHECK(part == 0 || split == 2);
        double2* own = near5 + (part == 0 ? 0 : (int64_t)kSplitSlot * n);
        for (int j = lane; j < nA; j += 32) {
            const double2 t = accAw[j];
            own[loA + j] = make_double2(t.x * kInv2Pi, t.y * kInv2Pi);
        }
        __syncwarp();
        if (done) {
            // The last writer of an owned leaf adds its slots (the order of
            // k_near_sum, which then has nothing to do): every leaf this item
            // wrote into counts one write event; the expected number is the
            // leaf's own items plus its existing non-empty backward neighbours.
            __threadfence();
            if (ownA) leaf_written(leaf, m, levels, n, split_from, item_base, ls, near5, done);
            if (n1 > 0) leaf_written(leaf + 1, m, levels, n, split_from, item_base, ls, near5, done);
            if (ownR2 && n2 > 0)
                for (int x = x2lo; x < x2hi; ++x) {
                    const int lf = (cy + 1) * m + x;
                    if (ls[lf + 1] > ls[lf])
                        leaf_written(lf, m, levels, n, split_from, item_base, ls, near5, done);
                }
        }
    }
    if (lane == 0 && my_pairs) atomicAdd(pairs, (unsigned long long)my_pairs);
}

// Direct sum: one thread per target, sources in ascending index order through
// shared-memory tiles (the accumulation order of kernels.py:83-93).  When the
// target count is small the source range is split into `nsplit` slices whose
// partial sums are combined in slice order by k_direct_reduce.
constexpr int kDirThreads = 256;

template <bool GAUSS>
__global__ void __launch_bounds__(kDirThreads)
    k_direct(const double* __restrict__ tx, const double* __restrict__ ty, int64_t mt,
             const double* __restrict__ x, const double* __restrict__ y,
             const double* __restrict__ g, const double* __restrict__ sigma, int64_t n,
             int64_t slice_len, const Tables* __restrict__ T, double* __restrict__ pu,
             double* __restrict__ pv) {
    pdl_enter();
    __shared__ Src tile[kDirThreads];
    __shared__ double sexp[kExpTab];
    const double* stab = stage_exp_table(sexp, T->exp2tab);
    const int64_t i = (int64_t)blockIdx.x * kDirThreads + threadIdx.x;
    const int slice = blockIdx.y;
    const int64_t s0 = (int64_t)slice * slice_len;
    const int64_t s1 = s0 + slice_len < n ? s0 + slice_len : n;
    const bool active = i < mt;
    const double px = active ? tx[i] : 0.0, py = active ? ty[i] : 0.0;
    double u = 0.0, v = 0.0;
    for (int64_t base = s0; base < s1; base += kDirThreads) {
        __syncthreads();
        const int64_t j = base + threadIdx.x;
        if (j < s1) {
            Src r;
            r.x = x[j];
            r.y = y[j];
            r.g = g[j];
            const double sg = GAUSS ? sigma[j] : 1.0;
            r.q2 = -1.4426950408889634 / (2.0 * sg * sg);
            tile[threadIdx.x] = r;
        }
        __syncthreads();
        const int cnt = (int)(s1 - base < kDirThreads ? s1 - base : kDirThreads);
        int k = 0;
        for (; k + 4 <= cnt; k += 4) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const Src s = tile[k + q];
                pair_acc<GAUSS>(px, py, s.x, s.y, s.g, s.q2, stab, u, v);
            }
        }
        for (; k < cnt; ++k) {
            const Src s = tile[k];
            pair_acc<GAUSS>(px, py, s.x, s.y, s.g, s.q2, stab, u, v);
        }
    }
    if (active) {
        pu[(int64_t)slice * mt + i] = u;
        pv[(int64_t)slice * mt + i] = v;
    }
}

__global__ void k_direct_reduce(const double* __restrict__ pu, const double* __restrict__ pv,
                                int64_t mt, int nsplit, double* __restrict__ u,
                                double* __restrict__ v) {
    pdl_enter();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= mt) return;
    double a = 0.0, b = 0.0;
    for (int s = 0; s < nsplit; ++s) {
        a += pu[(int64_t)s * mt + i];
        b += pv[(int64_t)s * mt + i];
    }
    u[i] = a * kInv2Pi;
    v[i] = b * kInv2Pi;
}

}  // namespace

int p2p_targets_per_lane() {
    static int tpt = 0;
    if (!tpt) {
        const char* e = getenv("VFMM_P2P_TPT");
        tpt = (e && e[0] == '2') ? 2 : 1;
    }
    return tpt;
}

bool sym_disabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("VFMM_P2P_SYM");
        v = (e && e[0] == '0') ? 1 : 0;
    }
    return v == 1;
}

static void launch_p2p_generic(const Layout& L, const Tables* T, const Src* src,
                               const int* leaf_starts, char* ws, Counters* ctr, int kernel,
                               double2* near_uv, Rows rows, cudaStream_t s);

// Which leaves get two work items (split_from: the first split leaf,
// relative to the item base): all of them when two items per leaf still fit
// one wave of warps (2 CTAs of 8 warps per SM) -- the per-item latency, not
// the SM throughput, then bounds the near field (config 1, 1,024 leaves:
// 0.131 -> 0.093 ms); otherwise the last `tail` leaves (default one wave of
// warps: 2,368), so the final items are halves and the near field's tail,
// where SMs run out of work, is half as long.  VFMM_P2P_SPLIT=0|1 forces
// none / all, VFMM_P2P_SPLIT_TAIL sets the tail (A/B).
int p2p_sym_split_from(const Layout& L, Rows rows) {
    static const int env = getenv("VFMM_P2P_SPLIT") ? atoi(getenv("VFMM_P2P_SPLIT")) : -1;
    static const int tail_env = getenv("VFMM_P2P_SPLIT_TAIL") ? atoi(getenv("VFMM_P2P_SPLIT_TAIL")) : -1;
    const int mrow = 1 << L.levels;
    const int row0 = rows.lo > 0 ? rows.lo - 1 : 0, row1 = rows.hi < mrow ? rows.hi : mrow;
    const int64_t leaves = (int64_t)(row1 > row0 ? row1 - row0 : 0) * mrow;
    if (env == 0) return (int)leaves;
    if (env == 1) return 0;
    const int64_t wave = (int64_t)kSymWarps * 2 * 148;
    if (2 * leaves <= wave) return 0;  // two items per leaf fit one wave
    // the tail of half items pays off when warps take several items each
    // (config 3, 262K leaves: near field 11.99 -> 11.61 ms; a rank of an
    // 8-way config-3 run, 33K leaves: 1.952 -> 1.935 ms per step); with about
    // one item per warp (config 2, 16K leaves) the uniform kernel without it
    // is faster (0.550 vs 0.565 ms)
    if (tail_env < 0 && leaves < wave * 8) return (int)leaves;
    const int64_t tail = tail_env >= 0 ? tail_env : wave;
    return (int)(leaves > tail ? leaves - tail : 0);
}

void launch_p2p(const Layout& L, const Tables* T, const Src* src, const int* leaf_starts,
                char* ws, Counters* ctr, int kernel, double2* near_uv, Rows rows, const int* keys,
                cudaStream_t s) {
    // VFMM_SYM_FUSED_SUM=1 (A/B): the symmetric kernel's last writers sum each
    // leaf's slots instead of k_near_sum.  Measured slower (config 2 step
    // 0.7222 -> 0.7355 ms: the fences, counters and per-leaf sums at item
    // ends cost the near field more than the separate 20 us pass).
    static const bool fused_env = getenv("VFMM_SYM_FUSED_SUM") && getenv("VFMM_SYM_FUSED_SUM")[0] == '1';
    const bool fused = fused_env && !sym_disabled();
    int* done = fused ? (int*)(ws + L.near_done) : nullptr;
    auto generic_chain = [&](cudaStream_t st) {
        launch_p2p_generic(L, T, src, leaf_starts, ws, ctr, kernel, near_uv, rows, st);
    };
    auto near_sum = [&](cudaStream_t st) {
        launch_near_sum(L, keys, near_uv, rows, leaf_starts, ctr, kernel, fused, st);
    };
    const bool g = kernel == VFMM_KERNEL_GAUSSIAN;
    // Stream launches: the generic kernel and its task list go first: in
    // symmetric mode they return at once, and that ~10 us head start lets P2M
    // (far stream) take its first wave of SM slots before the near field
    // fills the GPU -- measured 0.790 vs 0.799 ms per config-2 evaluate with
    // them launched after the symmetric kernel.  Graph capture: the symmetric
    // kernel first, the generic chain in an IF node it sets (not launched at
    // all when the symmetric kernel ran).
    // VFMM_GRAPH_COND=2: the conditional node for the sort path only (A/B)
    static const bool cond_near = !(getenv("VFMM_GRAPH_COND") && getenv("VFMM_GRAPH_COND")[0] == '2');
    const GraphCond gc = (sym_disabled() || !cond_near) ? GraphCond{} : graph_cond_create(s);
    if (!gc.on) generic_chain(s);
    // symmetric kernel: runs instead when the device-side mode check allows it
    // Leaf items per warp: enough CTAs for ~4 waves of 2 CTAs per SM (so
    // the far chain finds free slots and the tail is short), otherwise as
    // few CTAs as possible (each stages the 60 KB exp table).  Measured:
    // config 1 (1K leaves) K=2, config 2 (16K) K=2..3, config 3 (262K) K=32
    // best (before the one-item rule below).  VFMM_P2P_SYM_K overrides (tuning).
    static int KS_env = -1;
    if (KS_env < 0) {
        const char* e = getenv("VFMM_P2P_SYM_K");
        KS_env = e ? atoi(e) : 0;
    }
    // one item (two when split) per leaf of the rows the strip needs: [rows.lo - 1, rows.hi)
    const int mrow = 1 << L.levels;
    const int row0 = rows.lo > 0 ? rows.lo - 1 : 0, row1 = rows.hi < mrow ? rows.hi : mrow;
    const int item_base = row0 * mrow;
    const int split_from = p2p_sym_split_from(L, rows);
    const int64_t sym_leaves = (int64_t)(row1 > row0 ? row1 - row0 : 0) * mrow;
    const int64_t sym_items = split_from + 2 * (sym_leaves - split_from);
    // at least 2 items per warp, except when even that leaves fewer than ~4
    // waves of 2 CTAs per SM: one item per warp then (config 1: 1,024 leaves,
    // P2P 0.144 -> 0.086 ms; a rank of an 8-way config-2 run: 0.266 -> 0.218
    // ms per step; config 2 itself keeps 2: 0.7257 vs 0.7297 ms with 1)
    const int kSymKMin = sym_items < (int64_t)kSymWarps * 2 * 148 * 2 * 4 ? 1 : 2;
    int ks = KS_env > 0 ? KS_env : (int)(sym_items / ((int64_t)kSymWarps * 148 * 2 * 4));
    ks = ks < kSymKMin ? kSymKMin : (ks > 32 ? 32 : ks);
    const unsigned sblocks = (unsigned)((sym_items + kSymWarps * ks - 1) / (kSymWarps * ks));
    static int minb = 0;
    if (!minb) {
        const char* e = getenv("VFMM_P2P_SYM_MINB");
        minb = (e && (e[0] == '3' || e[0] == '1')) ? e[0] - '0' : 2;
    }
    const bool tsplit = split_from != 0 && split_from < sym_leaves;  // a tail of half items
    auto* sfn = minb == 3 ? (g ? (tsplit ? k_p2p_sym<true, 3, true> : k_p2p_sym<true, 3, false>)
                               : (tsplit ? k_p2p_sym<false, 3, true> : k_p2p_sym<false, 3, false>))
                          : (g ? (tsplit ? k_p2p_sym<true, 2, true> : k_p2p_sym<true, 2, false>)
                               : (tsplit ? k_p2p_sym<false, 2, true> : k_p2p_sym<false, 2, false>));
    static std::atomic<unsigned long long> attr_set{0};  // per device ordinal
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !(attr_set.load() >> dev & 1ull)) {
        for (auto* f : {k_p2p_sym<true, 3, true>, k_p2p_sym<false, 3, true>, k_p2p_sym<true, 2, true>,
                        k_p2p_sym<false, 2, true>, k_p2p_sym<true, 3, false>, k_p2p_sym<false, 3, false>,
                        k_p2p_sym<true, 2, false>, k_p2p_sym<false, 2, false>})
            cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, kSymSmem);
        attr_set.fetch_or(1ull << dev);
    }
    if (!sym_disabled() && sblocks > 0) {
        launch_k(sfn, sblocks, kSymWarps * 32, kSymSmem, s, src, leaf_starts, ctr, L.levels, L.n, rows, T,
                                                      near_uv, &ctr->near_pairs, ks, item_base,
                 (int)sym_items, split_from, gc, done);
        note_launches(1);
    } else if (gc.on) {  // no symmetric kernel to set the condition: run the chain
        generic_chain(s);
        near_sum(s);
        return;
    }
    if (gc.on) {  // the generic chain only when the symmetric mode does not apply
        cudaGraphNode_t node = nullptr;
        cudaStream_t bs = graph_cond_begin(s, gc, &node);
        generic_chain(bs);
        if (fused) near_sum(bs);  // (the symmetric kernel summed its own slots)
        graph_cond_end(s, bs, node);
        if (!fused) near_sum(s);
    } else {
        near_sum(s);
    }
}

static void launch_p2p_generic(const Layout& L, const Tables* T, const Src* src,
                               const int* leaf_starts, char* ws, Counters* ctr, int kernel,
                               double2* near_uv, Rows rows, cudaStream_t s) {
    // Items per warp: short-lived CTAs (default 2) let far-field CTAs in as SM
    // slots free up; the grid covers the upper bound of work items and CTAs
    // beyond the actual count exit at once.  VFMM_P2P_K overrides (tuning).
    static int K = 0;
    if (!K) {
        const char* e = getenv("VFMM_P2P_K");
        K = e ? atoi(e) : 2;
        if (K < 1) K = 2;
    }
    // The grid covers the upper bound of work items (VFMM_P2P_GRID_CAP caps it,
    // raising the items per warp -- tuning only: in symmetric mode the idle
    // CTAs of this kernel give the far chain a head start before P2P fills
    // the GPU, and capping them cost config 3 3.6%: 14.23 -> 14.75 ms).
    static const size_t cap = getenv("VFMM_P2P_GRID_CAP") ? (size_t)atol(getenv("VFMM_P2P_GRID_CAP"))
                                                          : (size_t)0;
    const size_t max_items = L.max_tasks * kNearRows;
    size_t per_block = (size_t)kP2PWarps * K;
    if ((max_items + per_block - 1) / per_block > cap && cap > 0)
        per_block = ((max_items + cap - 1) / cap + kP2PWarps - 1) / kP2PWarps * kP2PWarps;
    const unsigned blocks = (unsigned)((max_items + per_block - 1) / per_block);
    const int kk = (int)(per_block / kP2PWarps);
    const bool g = kernel == VFMM_KERNEL_GAUSSIAN;
    auto* fn = p2p_targets_per_lane() == 2 ? (g ? k_p2p<true, 2> : k_p2p<false, 2>)
                                           : (g ? k_p2p<true, 1> : k_p2p<false, 1>);
    launch_tasks(L, ws, ctr, rows, kernel == VFMM_KERNEL_GAUSSIAN, s);
    const int2* tasks = (const int2*)(ws + L.tasks);
    launch_k(fn, blocks, kP2PWarps * 32, 0, s, src, leaf_starts, tasks, ctr, L.levels, L.n, T, near_uv,
                                         &ctr->near_pairs, kk, sym_disabled() ? 0 : 1);
    note_launches(1);
}

int direct_nsplit(int64_t m, int64_t n) {
    const int64_t tblocks = (m + kDirThreads - 1) / kDirThreads;
    int64_t ns = (148 * 8 + tblocks - 1) / tblocks;
    const int64_t maxs = (n + kDirThreads - 1) / kDirThreads;
    if (ns > maxs) ns = maxs;
    if (ns > 1024) ns = 1024;
    if (ns < 1) ns = 1;
    return (int)ns;
}

void launch_direct(const double* tx, const double* ty, int64_t m, const double* x,
                   const double* y, const double* g, const double* sigma, int64_t n, int kernel,
                   double* pu, double* pv, int nsplit, double* u, double* v, const Tables* T,
                   cudaStream_t s) {
    int64_t slice = (n + nsplit - 1) / nsplit;
    slice = (slice + kDirThreads - 1) / kDirThreads * kDirThreads;
    dim3 grid((unsigned)((m + kDirThreads - 1) / kDirThreads), (unsigned)nsplit);
    if (kernel == VFMM_KERNEL_GAUSSIAN)
        launch_k(k_direct<true>, grid, kDirThreads, 0, s, tx, ty, m, x, y, g, sigma, n, slice, T, pu, pv);
    else
        launch_k(k_direct<false>, grid, kDirThreads, 0, s, tx, ty, m, x, y, g, sigma, n, slice, T, pu, pv);
    note_launches(1);
    launch_k(k_direct_reduce, (unsigned)((m + 255) / 256), 256, 0, s, pu, pv, m, nsplit, u, v);
    note_launches(1);
}

}  // namespace vfmm
