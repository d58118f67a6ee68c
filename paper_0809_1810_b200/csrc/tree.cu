// Uniform-quadtree construction on the GPU (north-star item 1).
//
// Replaces quadtree.build_tree / grid_indices / Tree.__init__
// (quadtree.py:39-46, 116-134, 182-201) and the permutation in
// engine.evaluate (engine.py:355-358):
//   k_keys        floor-rule binning with max-edge clamp + domain check + max sigma
//   LSD radix     stable sort of the row-major leaf keys (== np.argsort(kind="stable"))
//   k_pack        gather x, y, gamma, sigma into the sorted Src records
//   k_leaf_starts leaf_starts[4^l + 1] (== concatenate([0], cumsum(bincount)))
//   k_counts      per-level occupancy pyramid (Tree.counts)
//   k_tasks_*     32-target warp tasks for the near-field kernel
#include <climits>

#include "vfmm_internal.cuh"

namespace vfmm {

namespace {

__device__ __forceinline__ unsigned long long ordered_bits(double d) {
    unsigned long long b = (unsigned long long)__double_as_longlong(d);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void k_keys(const double* __restrict__ x, const double* __restrict__ y,
                       const double* __restrict__ sigma, int64_t n, double xmin, double ymin,
                       double side, int levels, int* __restrict__ key, int* __restrict__ val,
                       Counters* ctr) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long sbits = 0ull;
    if (i < n) {
        const double xi = x[i], yi = y[i];
        const double xmax = xmin + side, ymax = ymin + side;  // Domain.xmax (model.py:51-57)
        const bool inside = (xi >= xmin) && (xi <= xmax) && (yi >= ymin) && (yi <= ymax);
        const int m = 1 << levels;
        int ix = 0, iy = 0;
        if (inside) {
            // quadtree.py:44-45: min(int((x - xmin) / side * m), m - 1)
            const double tx = (xi - xmin) / side * (double)m;
            const double ty = (yi - ymin) / side * (double)m;
            ix = (int)tx;
            iy = (int)ty;
            ix = ix < m - 1 ? ix : m - 1;
            iy = iy < m - 1 ? iy : m - 1;
        } else {
            atomicAdd(&ctr->bad_count, 1);
            atomicMin(&ctr->first_bad, (int)i);
        }
        key[i] = iy * m + ix;
        val[i] = (int)i;
        if (sigma) sbits = ordered_bits(sigma[i]);
    }
    // block max of the sigma bits, one atomic per block
    __shared__ unsigned long long wmax[32];
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long t = __shfl_xor_sync(0xffffffffu, sbits, o);
        sbits = t > sbits ? t : sbits;
    }
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = sbits;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) sbits = wmax[w] > sbits ? wmax[w] : sbits;
        if (sbits) atomicMax(&ctr->sigma_max_bits, sbits);
    }
}

constexpr int kWPB = 8;  // warps per block in the radix kernels

__global__ void k_radix_hist(const int* __restrict__ keys, int64_t n, int shift, int bits, int wc,
                             int nchunks, int* __restrict__ hist) {
    extern __shared__ int sh[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int B = 1 << bits;
    int* h = sh + warp * B;
    for (int d = lane; d < B; d += 32) h[d] = 0;
    __syncwarp();
    const int64_t chunk = (int64_t)blockIdx.x * kWPB + warp;
    if (chunk < nchunks) {
        const int64_t beg = chunk * wc;
        const int64_t end = beg + wc < n ? beg + wc : n;
        for (int64_t i = beg + lane; i < end; i += 32) atomicAdd(&h[(keys[i] >> shift) & (B - 1)], 1);
        __syncwarp();
        for (int d = lane; d < B; d += 32) hist[(int64_t)d * nchunks + chunk] = h[d];
    }
}

// Stable scatter: warp chunks are processed in index order, lanes in index
// order within a round, equal digits ranked by lane (match_any), so the
// relative order of equal keys is preserved (LSD radix => stable argsort).
__global__ void k_radix_scatter(const int* __restrict__ kin, const int* __restrict__ vin,
                                int* __restrict__ kout, int* __restrict__ vout, int64_t n, int shift,
                                int bits, int wc, int nchunks, const int* __restrict__ offs) {
    extern __shared__ int sh[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int B = 1 << bits;
    int* run = sh + warp * B;
    const int64_t chunk = (int64_t)blockIdx.x * kWPB + warp;
    if (chunk >= nchunks) return;
    for (int d = lane; d < B; d += 32) run[d] = offs[(int64_t)d * nchunks + chunk];
    __syncwarp();
    const unsigned lt = (1u << lane) - 1u;
    const int64_t beg = chunk * wc;
    const int64_t end = beg + wc < n ? beg + wc : n;
    for (int64_t base = beg; base < end; base += 32) {
        const int64_t i = base + lane;
        const bool valid = i < end;
        int k = 0, v = 0, d = B + lane;
        if (valid) {
            k = kin[i];
            v = vin[i];
            d = (k >> shift) & (B - 1);
        }
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const int rank = __popc(peers & lt);
        if (valid) {
            const int pos = run[d] + rank;
            kout[pos] = k;
            vout[pos] = v;
        }
        __syncwarp();
        if (valid && rank == __popc(peers) - 1) run[d] += __popc(peers);
        __syncwarp();
    }
}

// ---- exclusive scan (int32, in place): block scan + top scan + add ----
constexpr int kScanThreads = 512;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int block_exclusive_scan(int v, int* warp_sums, int* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = v;
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        int s = lane < nw ? warp_sums[lane] : 0;
        int si = s;
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(0xffffffffu, si, o);
            if (lane >= o) si += t;
        }
        if (lane < nw) warp_sums[lane] = si - s;
        if (lane == 31) *total = si;
    }
    __syncthreads();
    return warp_sums[warp] + incl - v;
}

__global__ void k_scan_local(int* __restrict__ data, int64_t n, int* __restrict__ block_sums) {
    __shared__ int warp_sums[32];
    __shared__ int total;
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    int vals[kScanItems];
    int s = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        vals[j] = (base + j < n) ? data[base + j] : 0;
        s += vals[j];
    }
    int run = block_exclusive_scan(s, warp_sums, &total);
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        if (base + j < n) data[base + j] = run;
        run += vals[j];
    }
    if (threadIdx.x == 0) block_sums[blockIdx.x] = total;
}

__global__ void k_scan_top(int* __restrict__ sums, int nb) {
    __shared__ int warp_sums[32];
    __shared__ int total;
    int carry = 0;
    for (int base = 0; base < nb; base += blockDim.x) {
        const int i = base + threadIdx.x;
        const int v = i < nb ? sums[i] : 0;
        const int ex = block_exclusive_scan(v, warp_sums, &total);
        if (i < nb) sums[i] = ex + carry;
        carry += total;
        __syncthreads();
    }
}

__global__ void k_scan_add(int* __restrict__ data, int64_t n, const int* __restrict__ block_sums) {
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    const int add = block_sums[blockIdx.x];
    for (int j = threadIdx.x; j < kScanTile; j += blockDim.x) {
        if (base + j < n) data[base + j] += add;
    }
}

__global__ void k_pack(const double* __restrict__ x, const double* __restrict__ y,
                       const double* __restrict__ g, const double* __restrict__ sigma,
                       const int* __restrict__ perm, int64_t n, Src* __restrict__ src) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int j = perm[i];
    const double s = sigma ? sigma[j] : 1.0;
    Src r;
    r.x = x[j];
    r.y = y[j];
    r.g = g[j];
    // -r^2 / (2 sigma^2) (engine.py:256) expressed in log2 units
    r.q2 = -1.4426950408889634 / (2.0 * s * s);
    src[i] = r;
}

__global__ void k_leaf_starts(const int* __restrict__ keys, int64_t n, int nleaves,
                              int* __restrict__ ls) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n) return;
    const int prev = i > 0 ? keys[i - 1] : -1;
    const int cur = i < n ? keys[i] : nleaves;
    for (int k = prev + 1; k <= cur; ++k) ls[k] = (int)i;
}

__global__ void k_counts(const int* __restrict__ ls, int levels, int64_t total_cells,
                         int* __restrict__ counts) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= total_cells) return;
    int k = 0;
    int64_t off = 0;
    while (off + (1ll << (2 * k)) <= t) {
        off += 1ll << (2 * k);
        ++k;
    }
    const int64_t cell = t - off;
    const int mk = 1 << k;
    const int ix = (int)(cell % mk), iy = (int)(cell / mk);
    const int m = 1 << levels;
    const int s = 1 << (levels - k);
    int c = 0;
    for (int r = iy * s; r < (iy + 1) * s; ++r) {
        const int64_t row = (int64_t)r * m;
        c += ls[row + (int64_t)(ix + 1) * s] - ls[row + (int64_t)ix * s];
    }
    counts[t] = c;
}

__global__ void k_tasks_count(const int* __restrict__ ls, int nleaves, int chunk,
                              int* __restrict__ nt) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nleaves) return;
    const int c = ls[i + 1] - ls[i];
    nt[i] = (c + chunk - 1) / chunk;
}

__global__ void k_tasks_fill(const int* __restrict__ ls, int nleaves, int chunk,
                             const int* __restrict__ off, int2* __restrict__ tasks, Counters* ctr) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nleaves) return;
    const int c = ls[i + 1] - ls[i];
    const int nt = (c + chunk - 1) / chunk;
    const int o = off[i];
    for (int t = 0; t < nt; ++t) tasks[o + t] = make_int2(i, chunk * t);
    if (i == nleaves - 1) ctr->ntasks = o + nt;
}

__global__ void k_init_counters(Counters* ctr) {
    ctr->m2l_count = 0ull;
    ctr->near_pairs = 0ull;
    ctr->sigma_max_bits = 0ull;
    ctr->bad_count = 0;
    ctr->first_bad = INT_MAX;
    ctr->ntasks = 0;
    ctr->task_cursor = 0;
}

inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }

}  // namespace

void launch_init_counters(Counters* ctr, cudaStream_t s) {
    k_init_counters<<<1, 1, 0, s>>>(ctr);
    note_launches(1);
}

void launch_keys(const double* x, const double* y, const double* sigma, int64_t n, double xmin,
                 double ymin, double side, int levels, int* key, int* val, Counters* ctr,
                 cudaStream_t s) {
    k_keys<<<grid_for(n, 256), 256, 0, s>>>(x, y, sigma, n, xmin, ymin, side, levels, key, val, ctr);
    note_launches(1);
}

void launch_scan_i32(int* data, int64_t n, int* aux, cudaStream_t s) {
    if (n <= 0) return;
    const int64_t nb = (n + kScanTile - 1) / kScanTile;
    k_scan_local<<<(unsigned)nb, kScanThreads, 0, s>>>(data, n, aux);
    note_launches(1);
    k_scan_top<<<1, 1024, 0, s>>>(aux, (int)nb);
    note_launches(1);
    if (nb > 1) k_scan_add<<<(unsigned)nb, 256, 0, s>>>(data, n, aux);
    note_launches(1);
}

size_t scan_aux_elems(int64_t n) { return (size_t)((n + kScanTile - 1) / kScanTile) + 1; }

void launch_sort(const Layout& L, char* ws, cudaStream_t s, int** keys_out, int** perm_out) {
    int* ka = (int*)(ws + L.key_a);
    int* kb = (int*)(ws + L.key_b);
    int* va = (int*)(ws + L.val_a);
    int* vb = (int*)(ws + L.val_b);
    int* hist = (int*)(ws + L.hist);
    int* aux = (int*)(ws + L.scan_aux);
    const int bits = L.digit_bits;
    const int B = 1 << bits;
    const unsigned blocks = (unsigned)((L.nchunks + kWPB - 1) / kWPB);
    const size_t shm = (size_t)kWPB * B * sizeof(int);
    for (int pass = 0; pass < L.passes; ++pass) {
        const int shift = pass * bits;
        k_radix_hist<<<blocks, kWPB * 32, shm, s>>>(ka, L.n, shift, bits, L.wc, L.nchunks, hist);
        note_launches(1);
        launch_scan_i32(hist, (int64_t)B * L.nchunks, aux, s);
        k_radix_scatter<<<blocks, kWPB * 32, shm, s>>>(ka, va, kb, vb, L.n, shift, bits, L.wc,
                                                      L.nchunks, hist);
        note_launches(1);
        int* t = ka; ka = kb; kb = t;
        t = va; va = vb; vb = t;
    }
    *keys_out = ka;
    *perm_out = va;
}

void launch_pack(const double* x, const double* y, const double* g, const double* sigma,
                 const int* perm, int64_t n, Src* src, cudaStream_t s) {
    k_pack<<<grid_for(n, 256), 256, 0, s>>>(x, y, g, sigma, perm, n, src);
    note_launches(1);
}

void launch_leaf_starts(const int* sorted_keys, int64_t n, int nleaves, int* leaf_starts,
                        cudaStream_t s) {
    k_leaf_starts<<<grid_for(n + 1, 256), 256, 0, s>>>(sorted_keys, n, nleaves, leaf_starts);
    note_launches(1);
}

void launch_counts(const Layout& L, const int* leaf_starts, int* counts, cudaStream_t s) {
    int64_t total = 0;
    for (int k = 0; k <= L.levels; ++k) total += 1ll << (2 * k);
    k_counts<<<grid_for(total, 256), 256, 0, s>>>(leaf_starts, L.levels, total, counts);
    note_launches(1);
}

void launch_tasks(const Layout& L, const int* leaf_starts, int* task_scratch, int2* tasks,
                  int* aux, Counters* ctr, cudaStream_t s) {
    const int nl = (int)L.nleaves;
    k_tasks_count<<<grid_for(nl, 256), 256, 0, s>>>(leaf_starts, nl, 32 * p2p_targets_per_lane(),
                                                  task_scratch);
    note_launches(1);
    launch_scan_i32(task_scratch, nl, aux, s);
    k_tasks_fill<<<grid_for(nl, 256), 256, 0, s>>>(leaf_starts, nl, 32 * p2p_targets_per_lane(),
                                                 task_scratch, tasks, ctr);
    note_launches(1);
}

}  // namespace vfmm
