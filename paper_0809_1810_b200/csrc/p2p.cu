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
#include "vfmm_internal.cuh"

namespace vfmm {

namespace {

constexpr int kP2PWarps = 8;

template <bool GAUSS>
__global__ void __launch_bounds__(kP2PWarps * 32)
    k_p2p(const Src* __restrict__ src, const int* __restrict__ ls, const int2* __restrict__ tasks,
          const Counters* __restrict__ ctr_in, int levels, const Tables* __restrict__ T,
          double2* __restrict__ near_uv, unsigned long long* __restrict__ pairs) {
    __shared__ double stab[32];
    if (threadIdx.x < 32) stab[threadIdx.x] = T->exp2tab[threadIdx.x];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int task = blockIdx.x * kP2PWarps + warp;
    if (task >= ctr_in->ntasks) return;
    const int2 tk = tasks[task];
    const int leaf = tk.x;
    const int m = 1 << levels;
    const int lo = ls[leaf], hi = ls[leaf + 1];
    const int i = lo + tk.y + lane;
    const bool active = i < hi;
    double tx = 0.0, ty = 0.0;
    if (active) {
        const Src t = src[i];
        tx = t.x;
        ty = t.y;
    }
    const int cx = leaf % m, cy = leaf / m;
    const int xlo = cx > 0 ? cx - 1 : 0, xhi = cx < m - 1 ? cx + 1 : m - 1;
    double u = 0.0, v = 0.0;
    int nsrc = 0;
    for (int ny = cy - 1; ny <= cy + 1; ++ny) {
        if (ny < 0 || ny >= m) continue;
        const int a = ls[(int64_t)ny * m + xlo], b = ls[(int64_t)ny * m + xhi + 1];
        nsrc += b - a;
        int j = a;
        for (; j + 4 <= b; j += 4) {
            const Src s0 = src[j], s1 = src[j + 1], s2 = src[j + 2], s3 = src[j + 3];
            pair_acc<GAUSS>(tx, ty, s0.x, s0.y, s0.g, s0.q2, stab, u, v);
            pair_acc<GAUSS>(tx, ty, s1.x, s1.y, s1.g, s1.q2, stab, u, v);
            pair_acc<GAUSS>(tx, ty, s2.x, s2.y, s2.g, s2.q2, stab, u, v);
            pair_acc<GAUSS>(tx, ty, s3.x, s3.y, s3.g, s3.q2, stab, u, v);
        }
        for (; j < b; ++j) {
            const Src s0 = src[j];
            pair_acc<GAUSS>(tx, ty, s0.x, s0.y, s0.g, s0.q2, stab, u, v);
        }
    }
    if (active) near_uv[i] = make_double2(u * kInv2Pi, v * kInv2Pi);
    if (lane == 0) {
        // engine.py:284: pairs += n_leaf * (n_nbhd - 1), split over the leaf's tasks
        const int cnt = min(32, hi - lo - tk.y);
        atomicAdd(pairs, (unsigned long long)cnt * (unsigned long long)(nsrc - 1));
    }
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
    __shared__ Src tile[kDirThreads];
    __shared__ double stab[32];
    if (threadIdx.x < 32) stab[threadIdx.x] = T->exp2tab[threadIdx.x];
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

void launch_p2p(const Layout& L, const Tables* T, const Src* src, const int* leaf_starts,
                const int2* tasks, Counters* ctr, int kernel, double2* near_uv, cudaStream_t s) {
    const unsigned blocks = (unsigned)((L.max_tasks + kP2PWarps - 1) / kP2PWarps);
    if (kernel == VFMM_KERNEL_GAUSSIAN)
        k_p2p<true><<<blocks, kP2PWarps * 32, 0, s>>>(src, leaf_starts, tasks, ctr, L.levels, T,
                                                      near_uv, &ctr->near_pairs);
    else
        k_p2p<false><<<blocks, kP2PWarps * 32, 0, s>>>(src, leaf_starts, tasks, ctr, L.levels, T,
                                                       near_uv, &ctr->near_pairs);
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
        k_direct<true><<<grid, kDirThreads, 0, s>>>(tx, ty, m, x, y, g, sigma, n, slice, T, pu, pv);
    else
        k_direct<false><<<grid, kDirThreads, 0, s>>>(tx, ty, m, x, y, g, sigma, n, slice, T, pu, pv);
    note_launches(1);
    k_direct_reduce<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(pu, pv, m, nsplit, u, v);
    note_launches(1);
}

}  // namespace vfmm
