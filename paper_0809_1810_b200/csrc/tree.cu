// Uniform-quadtree construction on the GPU (north-star item 1).
//
// Replaces quadtree.build_tree / grid_indices / Tree.__init__
// (quadtree.py:39-46, 116-134, 182-201) and the permutation in
// engine.evaluate (engine.py:355-358): a stable sort of the particles by
// leaf key (np.argsort(kind="stable")).
//
// k_zero_regions    the counters and the scratch regions; CTA 0 samples the
//                   input order and picks the sort path (probe)
// Counting path (coherent input order, every leaf <= kFastLeafMax particles;
// config 2: 3 kernels in all -- bucket mode with the scan fused into the pack,
// see k_bin_count / k_leaf_pack; 4 at l >= 8; 5 when the buckets do not fit
// the near-field slots, i.e. below ~5 particles per leaf):
//   k_bin_count     floor-rule binning with max-edge clamp + domain check;
//                   per-leaf counts (warp-aggregated atomics), four
//                   particles per thread in flight
//   k_scan_one      counts -> leaf_starts (exclusive, in place; one CTA,
//                   striped int4 accesses; k_scan for long arrays)
//   k_bin_scatter   particle index -> a slot of its leaf (atomic cursor per
//                   leaf: the order inside a leaf is not yet the stable one);
//                   flags the LSD path if a leaf is too large; its first
//                   CTAs compute the occupancy pyramid (Tree.counts) and the
//                   P2P task counts
//   k_leaf_pack     warp per leaf: bitonic sort of the leaf's indices (which
//                   restores the stable order exactly), then perm, sorted
//                   keys and the packed Src records
// LSD radix path (random input order, or a leaf above kFastLeafMax; decided
// on the device -- the kernels return at once otherwise, and a captured graph
// puts them in an IF conditional node):
//   k_keys_ghist    keys + global digit histograms of every pass (and zeroes
//                   its tile's look-back words)
//   k_onesweep      one stable LSD pass per launch over 2048-key tiles:
//                   warp match_any ranking, per-digit decoupled look-back,
//                   coalesced digit-run writes; the last pass moves the
//                   packed Src records (k_pack_orig)
//   k_leaf_starts   leaf_starts[4^l + 1] (== concatenate([0], cumsum(bincount)))
//   k_counts_tasks  the occupancy pyramid + task counts of this path
// Generic near field only: k_scan, k_tasks_fill (the warp task list).
#include <climits>
#include <algorithm>
#include <cstdlib>

#include "vfmm_internal.cuh"

namespace vfmm {

namespace {


__device__ __forceinline__ unsigned long long ordered_bits(double d) {
    unsigned long long b = (unsigned long long)__double_as_longlong(d);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

constexpr int kFastLeafMax = 128;  // leaves the counting path sorts with one warp
constexpr int kBinILP = 4;         // particles per thread in flight in the binning kernels
// Counters::sort_fallback: 0 counting path, else the LSD radix path because
// the input looked spatially incoherent (probe) or a leaf is too large.
constexpr int kSortLsdProbe = 1, kSortLsdBigLeaf = 2;
constexpr int64_t kLsdMinN = 3ll << 20;  // random order below this: the counting path


// quadtree.py:44-45: min(int((v - lo) / side * m), m - 1).  The division is
// replaced by a multiply by 1/side unless the scaled coordinate lies within
// 1e-9 of a cell edge (the two differ by a few ulps, i.e. < 1e-11 at
// m <= 8192), where the exact rule decides.
__device__ __forceinline__ int cell_of(double v, double lo, double side, double inv_side, int m) {
    const double d = v - lo;
    const double t = d * inv_side * (double)m;
    int i = (int)t;
    const double fr = t - (double)i;
    if (!(fr > 1e-9 && fr < 1.0 - 1e-9)) i = (int)(d / side * (double)m);
    return i < m - 1 ? i : m - 1;
}

// Path choice from a sample of the input order: 64 runs of 32 consecutive
// particles; many distinct leaves per run (a random order) make the per-leaf
// atomics and gathers of the counting path scattered, so the LSD sort (whose
// passes write digit runs) is used instead.
__device__ void sort_probe_impl(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                                double xmin, double ymin, double side, int levels, int probe_mode,
                                Counters* __restrict__ ctr) {
    __shared__ int distinct;
    if (threadIdx.x == 0) distinct = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int m = 1 << levels;
    const double inv = 1.0 / side;
    double xs[8], ys[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {  // all loads in flight together
        const int64_t i = (int64_t)(((double)(warp * 8 + r) / 64.0) * (double)n) + lane;
        xs[r] = i < n ? x[i] : NAN;
        ys[r] = i < n ? y[i] : NAN;
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {  // 64 runs of 32 spread over [0, n)
        int k = -1;
        if (!isnan(xs[r]) && !isnan(ys[r])) {
            const double xi = fmin(fmax(xs[r], xmin), xmin + side);
            const double yi = fmin(fmax(ys[r], ymin), ymin + side);
            k = cell_of(yi, ymin, side, inv, m) * m + cell_of(xi, xmin, side, inv, m);
        }
        const unsigned peers = __match_any_sync(0xffffffffu, k);
        if (k >= 0 && lane == __ffs(peers) - 1) atomicAdd(&distinct, 1);
    }
    __syncthreads();
    // more than 8 distinct leaves per 32 consecutive particles on average
    // and enough particles that the counting path's scattered accesses miss L2
    // (random order, build ms counting / LSD: N = 2^20 0.093 / 0.113, a rank
    // of an 8-way config-3 run (2.1M, 64 per leaf) counting 45 us faster, N =
    // 2^22 0.342 / 0.321, 2^24 1.90 / 1.17; tools/sort_probe.py)
    // (probe_mode: 0 auto, 1 force LSD, 2 never LSD by the probe -- A/B)
    if (threadIdx.x == 0 &&
        (probe_mode == 1 || (probe_mode == 0 && distinct > 64 * 8 && n > kLsdMinN)))
        ctr->sort_fallback = kSortLsdProbe;
}

// Keys, domain check and per-leaf counts (cnt zeroed; leaf_starts storage).
//
// Bucket mode (bucket != nullptr; launch_build picks it when the buckets fit
// the idle near-field slots): the count's atomic also claims the particle's
// slot in its leaf's fixed bucket of kFastLeafMax indices, so k_bin_scatter
// (a second pass over the keys with a second atomic per group) is not
// launched and the keys are not stored; a leaf above kFastLeafMax flags the
// LSD path, as k_bin_scatter would.
__global__ void __launch_bounds__(256)
    k_bin_count(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                double xmin, double ymin, double side, int levels, int* __restrict__ key,
                int* __restrict__ cnt, Counters* __restrict__ ctr, int* __restrict__ bucket) {
    pdl_enter();
    if (ctr->sort_fallback == kSortLsdProbe) return;
    const int lane = threadIdx.x & 31;
    bool big = false;
    const int m = 1 << levels;
    const double inv = 1.0 / side;
    const double xmax = xmin + side, ymax = ymin + side;  // Domain.xmax (model.py:51-57)
    // grid-stride over tiles of kBinILP x 256 particles; a thread's kBinILP
    // positions are loaded together (the single load per thread had every
    // warp waiting on memory: 1.5 TB/s), then binned one 256-slice at a time
    // (warp-aggregated atomics per slice)
    const int64_t tile = (int64_t)kBinILP * blockDim.x;
    for (int64_t t0 = (int64_t)blockIdx.x * tile; t0 < n; t0 += (int64_t)gridDim.x * tile) {
        double xs[kBinILP], ys[kBinILP];
#pragma unroll
        for (int u = 0; u < kBinILP; ++u) {
            const int64_t i = t0 + u * blockDim.x + threadIdx.x;
            xs[u] = i < n ? x[i] : 0.0;
            ys[u] = i < n ? y[i] : 0.0;
        }
        int ks[kBinILP], base[kBinILP];
        unsigned pe[kBinILP];
#pragma unroll
        for (int u = 0; u < kBinILP; ++u) {
            const int64_t i = t0 + u * blockDim.x + threadIdx.x;
            int k = -1;
            if (i < n) {
                const double xi = xs[u], yi = ys[u];
                int ix = 0, iy = 0;
                if ((xi >= xmin) && (xi <= xmax) && (yi >= ymin) && (yi <= ymax)) {
                    ix = cell_of(xi, xmin, side, inv, m);
                    iy = cell_of(yi, ymin, side, inv, m);
                } else {
                    atomicAdd(&ctr->bad_count, 1);
                    atomicMax(&ctr->first_bad_neg, INT_MAX - (int)i);
                }
                k = iy * m + ix;
                if (!bucket) key[i] = k;
            }
            const unsigned peers = __match_any_sync(0xffffffffu, k);
            ks[u] = k;
            pe[u] = peers;
            base[u] = 0;
            // the group's atomics of the kBinILP slices are all in flight before
            // the first returned base is used
            if (k >= 0 && lane == __ffs(peers) - 1) base[u] = atomicAdd(&cnt[k], __popc(peers));
        }
        if (bucket) {
#pragma unroll
            for (int u = 0; u < kBinILP; ++u) {
                const int64_t i = t0 + u * blockDim.x + threadIdx.x;
                const int b = __shfl_sync(0xffffffffu, base[u], __ffs(pe[u]) - 1);
                if (ks[u] >= 0) {
                    const int pos = b + __popc(pe[u] & ((1u << lane) - 1u));
                    if (pos < kFastLeafMax)
                        bucket[(int64_t)ks[u] * kFastLeafMax + pos] = (int)i;
                    else
                        big = true;
                }
            }
        }
    }
    if (bucket && __any_sync(0xffffffffu, big) && lane == 0)
        atomicMax(&ctr->sort_fallback, kSortLsdBigLeaf);
}

// Occupancy of every cell of every level (level 0 first) from leaf_starts
// (Tree.counts, quadtree.py:126-134):
// a level-k cell covers 2^(l-k) leaf rows, each a contiguous leaf range.
// Leaf cells also emit their P2P task count ceil(count / chunk).
struct CountsArgs {
    int ctas;  // CTAs of 256 threads doing this work (k_bin_scatter's first CTAs)
    int levels;
    int64_t total_threads;
    int chunk;
    Rows rows;
    int* counts;
    int* ntask;
};
// FROM_CNT: `ls` holds the raw per-leaf counts instead of leaf_starts (the
// fused-scan build, where leaf_starts is being written by the same kernel):
// a cell's rows are summed leaf by leaf (int4 loads).
template <bool FROM_CNT = false>
__device__ __forceinline__ void counts_tasks_body(int64_t t, const int* __restrict__ ls,
                                                  const CountsArgs& a, Counters* __restrict__ ctr) {
    // A cell of level k spans s = 2^(levels-k) leaf rows; g = min(32, s)
    // lanes split its rows and add their partial counts by xor shuffles (the
    // coarse cells were serial 32..128-row loops).  Thread ranges per level:
    // 4^k g_k threads, each level's range aligned to its g.
    const int levels = a.levels;
    const Rows rows = a.rows;
    int k = 0, g = 1;
    int64_t off = 0, cell_off = 0;
    for (;;) {
        const int s = 1 << (levels - k);
        g = s < 32 ? s : 32;
        const int64_t nt = (1ll << (2 * k)) * g;
        if (t < off + nt || k == levels) break;
        off += nt;
        cell_off += 1ll << (2 * k);
        ++k;
    }
    const bool valid = t < a.total_threads;
    const int64_t cell = valid ? (t - off) / g : 0;
    const int sub = valid ? (int)((t - off) % g) : 0;
    const int mk = 1 << k;
    const int ix = (int)(cell % mk), iy = (int)(cell / mk);
    const int m = 1 << levels;
    const int s = 1 << (levels - k);
    // only owned leaf rows are counted, so per-rank pyramids of a sharded run
    // are disjoint and their sum is the global occupancy
    const int r0 = max(iy * s, rows.lo), r1 = min((iy + 1) * s, rows.hi);
    int c = 0;
    if (valid)
        for (int r = r0 + sub; r < r1; r += g) {
            const int64_t row = (int64_t)r * m;
            if (!FROM_CNT) {
                c += ls[row + (int64_t)(ix + 1) * s] - ls[row + (int64_t)ix * s];
            } else if (s >= 4) {
                const int4* p4 = reinterpret_cast<const int4*>(ls + row + (int64_t)ix * s);
                int c4[4] = {0, 0, 0, 0};
#pragma unroll 4
                for (int j = 0; j < (s >> 2); ++j) {
                    const int4 q = p4[j];
                    c4[j & 3] += (q.x + q.y) + (q.z + q.w);
                }
                c += (c4[0] + c4[1]) + (c4[2] + c4[3]);
            } else {
                for (int j = 0; j < s; ++j) c += ls[row + (int64_t)ix * s + j];
            }
        }
    // every lane runs the same shuffles; a lane adds only within its g-group
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const int v = __shfl_xor_sync(0xffffffffu, c, o);
        if (o < g) c += v;
    }
    int full = 0;
    if (valid && sub == 0) {
        a.counts[cell_off + cell] = c;
        // only leaves of the owned row strip get near-field tasks
        if (k == levels) {
            a.ntask[cell] = (iy >= rows.lo && iy < rows.hi) ? (c + a.chunk - 1) / a.chunk : 0;
            // owned and halo rows (the symmetric P2P touches both)
            full = FROM_CNT ? ls[cell] : ls[cell + 1] - ls[cell];
        }
    }
    // largest leaf: one atomic per warp
    full = __reduce_max_sync(0xffffffffu, full);
    if ((threadIdx.x & 31) == 0 && full > 0) atomicMax(&ctr->max_leaf, full);
}

// The same after the LSD radix path (k_bin_scatter did it on the counting
// path; a big-leaf fallback recomputes identical values).
__global__ void __launch_bounds__(256)
    k_counts_tasks(const int* __restrict__ ls, CountsArgs a, Counters* __restrict__ ctr) {
    pdl_enter();
    if (!ctr->sort_fallback) return;
    counts_tasks_body((int64_t)blockIdx.x * blockDim.x + threadIdx.x, ls, a, ctr);
}

// Index i -> a slot of its leaf: one atomic per (warp, leaf) group, lanes
// ranked in index order inside the group.
//
// The first ca.ctas CTAs instead compute the occupancy pyramid and task
// counts (counts_tasks_body): leaf_starts is final once the scan ran, so the
// counts leave the critical chain (they were a separate launch after the
// record pack).
__global__ void __launch_bounds__(256)
    k_bin_scatter(const int* __restrict__ key, int64_t n, const int* __restrict__ ls,
                  int* __restrict__ fill, int* __restrict__ slot, Counters* __restrict__ ctr,
                  CountsArgs ca) {
    pdl_enter();
    if (ctr->sort_fallback == kSortLsdProbe) return;
    if ((int)blockIdx.x < ca.ctas) {
        counts_tasks_body((int64_t)blockIdx.x * blockDim.x + threadIdx.x, ls, ca, ctr);
        return;
    }
    const int lane = threadIdx.x & 31;
    bool big = false;
    const unsigned nb = gridDim.x - ca.ctas;
    // tiles of kBinILP x 256 particles: the keys, then their leaf ranges, are
    // loaded together before the slots are claimed one 256-slice at a time
    const int64_t tile = (int64_t)kBinILP * blockDim.x;
    for (int64_t t0 = (int64_t)(blockIdx.x - ca.ctas) * tile; t0 < n; t0 += (int64_t)nb * tile) {
        int ks[kBinILP], lo[kBinILP], hi[kBinILP];
#pragma unroll
        for (int u = 0; u < kBinILP; ++u) {
            const int64_t i = t0 + u * blockDim.x + threadIdx.x;
            ks[u] = i < n ? key[i] : -1;
        }
#pragma unroll
        for (int u = 0; u < kBinILP; ++u) {
            lo[u] = ks[u] >= 0 ? ls[ks[u]] : 0;
            hi[u] = ks[u] >= 0 ? ls[ks[u] + 1] : 0;
        }
#pragma unroll
        for (int u = 0; u < kBinILP; ++u) {
            const int64_t i = t0 + u * blockDim.x + threadIdx.x;
            const int k = ks[u];
            const unsigned peers = __match_any_sync(0xffffffffu, k);
            const int leader = __ffs(peers) - 1;
            int base = 0;
            if (k >= 0 && lane == leader) base = atomicAdd(&fill[k], __popc(peers));
            base = __shfl_sync(0xffffffffu, base, leader);
            if (k >= 0) {
                const int pos = lo[u] + base + __popc(peers & ((1u << lane) - 1u));
                VCHECK(lo[u] >= 0 && pos < hi[u]);
                slot[pos] = (int)i;
                big |= hi[u] - lo[u] > kFastLeafMax;
            }
        }
    }
    if (__any_sync(0xffffffffu, big) && lane == 0) atomicMax(&ctr->sort_fallback, kSortLsdBigLeaf);
}

// Ascending bitonic sort of 32 E values held as e[k] = element k * 32 + lane.
template <int E>
__device__ __forceinline__ void warp_bitonic(int (&e)[E]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int size = 2; size <= 32 * E; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            if (stride >= 32) {  // partner in the same lane
                const int ks = stride >> 5;
#pragma unroll
                for (int k = 0; k < E; ++k) {
                    if (k & ks) continue;
                    const bool up = (((k * 32 + lane) & size) == 0);
                    const int a = e[k], b = e[k ^ ks];
                    e[k] = up ? min(a, b) : max(a, b);
                    e[k ^ ks] = up ? max(a, b) : min(a, b);
                }
            } else {
#pragma unroll
                for (int k = 0; k < E; ++k) {
                    const int p = k * 32 + lane;
                    const int o = __shfl_xor_sync(0xffffffffu, e[k], stride);
                    const bool up = (p & size) == 0, lower = (p & stride) == 0;
                    e[k] = (up == lower) ? min(e[k], o) : max(e[k], o);
                }
            }
        }
    }
}

// -1 / (2 sigma^2 ln 2) (the exponent of engine.py:256 in log2 units), the
// IEEE division done only when sigma changes from the thread's previous
// particle (uniform core sizes: once per thread; it was a quarter of
// k_leaf_pack's stall samples).  Results are identical to dividing every time.
__device__ __forceinline__ double q2_of(double s, double& s_prev, double& q_prev) {
    if (!(s == s_prev)) {
        s_prev = s;
        q_prev = -1.4426950408889634 / (2.0 * s * s);
    }
    return q_prev;
}

template <int E>
__device__ __forceinline__ void leaf_pack(const int* __restrict__ sl, int lo, int c, int leaf,
                                          const double* __restrict__ x, const double* __restrict__ y,
                                          const double* __restrict__ g,
                                          const double* __restrict__ sigma, int sstride,
                                          int* __restrict__ keys, int* __restrict__ perm,
                                          Src* __restrict__ src, unsigned long long& smax,
                                          unsigned long long& smin, double& s_prev, double& q_prev) {
    const int lane = threadIdx.x & 31;
    int e[E];
#pragma unroll
    for (int k = 0; k < E; ++k) {
        const int p = k * 32 + lane;
        e[k] = p < c ? sl[p] : INT_MAX;
    }
    warp_bitonic<E>(e);
    // the gathers of two rounds in flight before the first record is packed (the
    // sigma-dependent branch of q2_of otherwise serialises the rounds of loads)
    constexpr int H = E < 2 ? E : 2;
#pragma unroll
    for (int k0 = 0; k0 < E; k0 += H) {
        double gx[H], gy[H], gg[H], gs[H];
#pragma unroll
        for (int j = 0; j < H; ++j) {
            const bool ok = (k0 + j) * 32 + lane < c;
            const int idx = ok ? e[k0 + j] : 0;
            gs[j] = (ok && sigma) ? sigma[(int64_t)idx * sstride] : 1.0;
            gx[j] = ok ? x[idx] : 0.0;
            gy[j] = ok ? y[idx] : 0.0;
            gg[j] = ok ? g[idx] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < H; ++j) {
            const int k = k0 + j;
            const int p = k * 32 + lane;
            if (p >= c) continue;
            const int idx = e[k];
            const double s = gs[j];
            Src r;
            r.x = gx[j];
            r.y = gy[j];
            r.g = gg[j];
            r.q2 = q2_of(s, s_prev, q_prev);  // -r^2 / (2 sigma^2) in log2 units
            src[lo + p] = r;
            perm[lo + p] = idx;
            keys[lo + p] = leaf;
            if (sigma) {
                const unsigned long long b = ordered_bits(s);
                smax = b > smax ? b : smax;
                smin = b < smin ? b : smin;
            }
        }
    }
}

// Warp per leaf: restore the stable order inside the leaf, write the sorted
// keys, the permutation and the packed records.
#ifndef VFMM_PACK_MINB
#define VFMM_PACK_MINB 5  // 48 registers: 5 CTAs per SM (config 2 build 46.3 -> 44.4 us; 6: 45.5, 8: 49.7)
#endif
constexpr int kPackFusedMaxLeaves = 1 << 14;  // fused-scan mode: l <= 7
constexpr int kPackFusedGrid = 148 * VFMM_PACK_MINB;
// Fused-scan mode (cnt != nullptr; bucket mode at l <= 7): `cnt` holds the raw
// per-leaf counts and this kernel also produces leaf_starts, so the scan
// launch between the count and the pack drops out.  A CTA owns a contiguous
// run of L <= 32 leaves: it sums the counts below its run (striped int4
// loads, one round trip; the whole array is 64 KB in L2), scans its own L
// counts in one warp, writes its part of leaf_starts and packs its leaves.
__global__ void __launch_bounds__(256, VFMM_PACK_MINB)
    k_leaf_pack(int* __restrict__ ls, const int* __restrict__ slot, int nleaves,
                const double* __restrict__ x, const double* __restrict__ y,
                const double* __restrict__ g, const double* __restrict__ sigma, int sstride,
                int* __restrict__ keys, int* __restrict__ perm, Src* __restrict__ src,
                Counters* __restrict__ ctr, GraphCond lsd_cond, int bucket_stride, CountsArgs ca,
                const int* __restrict__ cnt) {
    pdl_enter();
    // the path choice is final here (k_bin_scatter / k_bin_count's buckets): a
    // captured graph runs the LSD kernels (an IF node after this kernel) only
    // when it is taken
    graph_cond_set(lsd_cond, ctr->sort_fallback != 0 ? 1u : 0u);
    if (ctr->sort_fallback) return;
    // bucket mode: the first ca.ctas CTAs compute the occupancy pyramid and the
    // task counts (k_bin_scatter's first CTAs do otherwise)
    if ((int)blockIdx.x < ca.ctas) {
        if (cnt)
            counts_tasks_body<true>((int64_t)blockIdx.x * blockDim.x + threadIdx.x, cnt, ca, ctr);
        else
            counts_tasks_body((int64_t)blockIdx.x * blockDim.x + threadIdx.x, ls, ca, ctr);
        return;
    }
    __shared__ unsigned long long wmax[8], wmin[8];
    __shared__ int s_part[8], s_lo[32], s_c[32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long smax = 0ull, smin = ~0ull;
    double s_prev = __longlong_as_double(0x7ff8000000000000ll), q_prev = 0.0;  // NaN: nothing cached
    const int nb = gridDim.x - ca.ctas;
    if (cnt) {
        const int L = (nleaves + nb - 1) / nb;  // <= 32 (launch_build)
        const int first = (blockIdx.x - ca.ctas) * L;
        if (first >= nleaves) return;
        // the counts below the run
        int part = 0;
        const int4* c4 = reinterpret_cast<const int4*>(cnt);
        for (int i4 = threadIdx.x; i4 * 4 < first; i4 += 256) {
            const int4 q = c4[i4];
            const int e = i4 * 4;
            part += q.x + (e + 1 < first ? q.y : 0) + (e + 2 < first ? q.z : 0) + (e + 3 < first ? q.w : 0);
        }
        // the run's own counts (warp 0), meanwhile
        int cj = 0;
        if (warp == 0 && lane < L && first + lane < nleaves) cj = cnt[first + lane];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (lane == 0) s_part[warp] = part;
        __syncthreads();
        if (warp == 0) {
            int base = 0;
#pragma unroll
            for (int w = 0; w < 8; ++w) base += s_part[w];
            int incl = cj;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += u;
            }
            s_lo[lane] = base + incl - cj;
            s_c[lane] = cj;
            if (lane < L && first + lane < nleaves) {
                ls[first + lane] = base + incl - cj;
                if (first + lane == nleaves - 1) ls[nleaves] = base + incl;
            }
        }
        __syncthreads();
        for (int j = warp; j < L && first + j < nleaves; j += 8) {
            const int leaf = first + j, lo = s_lo[j], c = s_c[j];
            const int* sl = slot + (int64_t)leaf * bucket_stride;
            if (c > 64)
                leaf_pack<4>(sl, lo, c, leaf, x, y, g, sigma, sstride, keys, perm, src, smax, smin, s_prev, q_prev);
            else if (c > 32)
                leaf_pack<2>(sl, lo, c, leaf, x, y, g, sigma, sstride, keys, perm, src, smax, smin, s_prev, q_prev);
            else if (c > 0)
                leaf_pack<1>(sl, lo, c, leaf, x, y, g, sigma, sstride, keys, perm, src, smax, smin, s_prev, q_prev);
        }
    } else {
        for (int leaf = (blockIdx.x - ca.ctas) * 8 + warp; leaf < nleaves; leaf += nb * 8) {
            const int lo = ls[leaf], c = ls[leaf + 1] - lo;
            // the leaf's indices: its bucket, or its range of the scattered slots
            const int* sl = bucket_stride ? slot + (int64_t)leaf * bucket_stride : slot + lo;
            if (c > 64)
                leaf_pack<4>(sl, lo, c, leaf, x, y, g, sigma, sstride, keys, perm, src, smax, smin, s_prev, q_prev);
            else if (c > 32)
                leaf_pack<2>(sl, lo, c, leaf, x, y, g, sigma, sstride, keys, perm, src, smax, smin, s_prev, q_prev);
            else if (c > 0)
                leaf_pack<1>(sl, lo, c, leaf, x, y, g, sigma, sstride, keys, perm, src, smax, smin, s_prev, q_prev);
        }
    }
    if (!sigma) return;
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, smax, o);
        smax = t > smax ? t : smax;
        const unsigned long long u = __shfl_xor_sync(0xffffffffu, smin, o);
        smin = u < smin ? u : smin;
    }
    if (lane == 0) {
        wmax[warp] = smax;
        wmin[warp] = smin;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) {
            smax = wmax[w] > smax ? wmax[w] : smax;
            smin = wmin[w] < smin ? wmin[w] : smin;
        }
        if (smax) atomicMax(&ctr->sigma_max_bits, smax);
        if (smin != ~0ull) atomicMax(&ctr->sigma_min_neg, ~smin);
    }
}

// Source records in ORIGINAL order (coalesced), with the sigma statistics;
// the last radix pass then moves whole 32-byte records instead of gathering
// four arrays element by element.
__global__ void __launch_bounds__(256)
    k_pack_orig(const double* __restrict__ x, const double* __restrict__ y,
                const double* __restrict__ g, const double* __restrict__ sigma, int sstride,
                int64_t n, Src* __restrict__ out, Counters* __restrict__ ctr) {
    pdl_enter();
    if (!ctr->sort_fallback) return;
    __shared__ unsigned long long wmax[8], wmin[8];
    unsigned long long sbits = 0ull, smin = ~0ull;
    double s_prev = __longlong_as_double(0x7ff8000000000000ll), q_prev = 0.0;  // NaN: nothing cached
    // grid-stride (a small grid: the launch is cheap when the counting path ran)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double s = sigma ? sigma[i * sstride] : 1.0;
        Src r;
        r.x = x[i];
        r.y = y[i];
        r.g = g[i];
        // -r^2 / (2 sigma^2) (engine.py:256) expressed in log2 units
        r.q2 = q2_of(s, s_prev, q_prev);
        out[i] = r;
        if (sigma) {
            const unsigned long long b = ordered_bits(s);
            sbits = b > sbits ? b : sbits;
            smin = b < smin ? b : smin;
        }
    }
    if (!sigma) return;
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, sbits, o);
        sbits = t > sbits ? t : sbits;
        const unsigned long long u = __shfl_xor_sync(0xffffffffu, smin, o);
        smin = u < smin ? u : smin;
    }
    const int warp = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        wmax[warp] = sbits;
        wmin[warp] = smin;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            sbits = wmax[w] > sbits ? wmax[w] : sbits;
            smin = wmin[w] < smin ? wmin[w] : smin;
        }
        if (sbits) atomicMax(&ctr->sigma_max_bits, sbits);
        if (smin != ~0ull) atomicMax(&ctr->sigma_min_neg, ~smin);
    }
}

// ---- LSD radix path: one kernel per pass over tiles of kTile keys ----
//
// Tile = 256 threads x 8 keys.  Warp w ranks its 256 consecutive keys in 8
// rounds of 32 (match_any; lanes and rounds in index order), so ranks are
// stable.  Per-digit tile counts are chained across tiles by decoupled
// look-back (tiles numbered by ticket), the keys are staged in shared memory
// in tile-sorted order and written out digit run by digit run (coalesced).
constexpr int kTileThreads = 256;
constexpr int kTileItems = 8;
constexpr int kTile = kTileThreads * kTileItems;  // 2048
constexpr unsigned kLbAgg = 1u << 30, kLbIncl = 2u << 30, kLbMask = (1u << 30) - 1;

// Exclusive scan of one value per thread over a 256-thread block.
__device__ __forceinline__ int block_excl_256(int v, int* wsum) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = v;
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int add = 0;
    for (int w = 0; w < warp; ++w) add += wsum[w];
    return add + incl - v;
}

// Keys (floor rule, domain check) + the global digit histograms of every pass.
__global__ void __launch_bounds__(kTileThreads)
    k_keys_ghist(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                 double xmin, double ymin, double side, int levels, int bits, int passes,
                 int* __restrict__ key, int* __restrict__ ghist, unsigned* __restrict__ lb,
                 int64_t lb_words, Counters* __restrict__ ctr) {
    pdl_enter();
    if (!ctr->sort_fallback) return;  // the counting path built the tree
    // this tile's decoupled look-back words of every pass (zeroed here, on
    // the LSD path only, instead of in the build's first kernel)
    for (int i = threadIdx.x; i < passes << bits; i += kTileThreads)
        lb[(int64_t)(i >> bits) * lb_words + ((int64_t)blockIdx.x << bits) + (i & ((1 << bits) - 1))] = 0u;
    const bool probe_lsd = ctr->sort_fallback == kSortLsdProbe;
    __shared__ int h[4 * 256];
    const int B = 1 << bits;
    for (int i = threadIdx.x; i < passes * B; i += kTileThreads) h[i] = 0;
    __syncthreads();
    const int m = 1 << levels;
    const double inv = 1.0 / side;
    const double xmax = xmin + side, ymax = ymin + side;  // Domain.xmax (model.py:51-57)
    const int64_t base = (int64_t)blockIdx.x * kTile;
#pragma unroll 4
    for (int it = 0; it < kTileItems; ++it) {
        const int64_t i = base + it * kTileThreads + threadIdx.x;
        if (i >= n) break;
        const double xi = x[i], yi = y[i];
        int ix = 0, iy = 0;
        if ((xi >= xmin) && (xi <= xmax) && (yi >= ymin) && (yi <= ymax)) {
            ix = cell_of(xi, xmin, side, inv, m);
            iy = cell_of(yi, ymin, side, inv, m);
        } else if (probe_lsd) {  // otherwise k_bin_count counted them
            atomicAdd(&ctr->bad_count, 1);
            atomicMax(&ctr->first_bad_neg, INT_MAX - (int)i);
        }
        const int k = iy * m + ix;
        key[i] = k;
        for (int p = 0; p < passes; ++p) atomicAdd(&h[p * B + ((k >> (p * bits)) & (B - 1))], 1);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * B; i += kTileThreads)
        if (h[i]) atomicAdd(&ghist[i], h[i]);
}

// One stable LSD pass.  lb: per (tile, digit) look-back words (zeroed),
// ticket: tile counter (zeroed).  The last pass also moves the packed
// 32-byte source records (packed[val] -> src[pos]).
__global__ void __launch_bounds__(kTileThreads)
    k_onesweep(const int* __restrict__ kin, const int* __restrict__ vin, int* __restrict__ kout,
               int* __restrict__ vout, int64_t n, int shift, int bits,
               const int* __restrict__ ghist, unsigned* __restrict__ lb, int* __restrict__ ticket,
               const Src* __restrict__ packed, Src* __restrict__ src,
               const Counters* __restrict__ ctr) {
    pdl_enter();
    if (!ctr->sort_fallback) return;
    constexpr int W = kTileThreads / 32;
    __shared__ int wcnt[W][256];   // per-warp digit counts, then per-warp prefixes
    __shared__ int gbase[256];     // global position of the tile's first key of digit d, minus its local start
    __shared__ int lstart[256];
    __shared__ int skey[kTile];
    __shared__ int sval[kTile];
    __shared__ int tile_s;
    const int B = 1 << bits;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) tile_s = atomicAdd(ticket, 1);
    for (int i = threadIdx.x; i < W * 256; i += kTileThreads) (&wcnt[0][0])[i] = 0;
    __syncthreads();
    const int tile = tile_s;
    const int64_t base = (int64_t)tile * kTile;
    const int cnt = (int)min((int64_t)kTile, n - base);
    // ---- rank: warp w owns keys [w*512, (w+1)*512) of the tile ----
    int kr[kTileItems], vr[kTileItems], rk[kTileItems];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int it = 0; it < kTileItems; ++it) {
        const int j = warp * 32 * kTileItems + it * 32 + lane;
        const bool ok = j < cnt;
        kr[it] = ok ? kin[base + j] : 0;
        vr[it] = ok ? (vin ? vin[base + j] : (int)(base + j)) : 0;
    }
#pragma unroll
    for (int it = 0; it < kTileItems; ++it) {
        const int j = warp * 32 * kTileItems + it * 32 + lane;
        const bool ok = j < cnt;
        const int d = ok ? (kr[it] >> shift) & (B - 1) : 256 + lane;  // invalid: unique, unranked
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        int pre = 0;
        if (ok) pre = wcnt[warp][d];
        rk[it] = pre + __popc(peers & lt);
        __syncwarp();
        if (ok && (peers >> lane) == 1u) wcnt[warp][d] = pre + __popc(peers);  // highest lane of the group
        __syncwarp();
    }
    __syncthreads();
    // ---- per-digit tile counts, warp prefixes, local starts ----
    const int d = threadIdx.x;  // one thread per digit (B <= 256)
    int c = 0;
    if (d < B) {
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const int t = wcnt[w][d];
            wcnt[w][d] = c;
            c += t;
        }
    }
    __shared__ int wsum[2][W];
    lstart[d] = block_excl_256(c, wsum[0]);
    // global start of digit d: exclusive scan of this pass's global histogram
    const int gstart = block_excl_256(d < B ? ghist[d] : 0, wsum[1]);
    // ---- decoupled look-back per digit ----
    if (d < B) {
        volatile unsigned* st = lb + (size_t)tile * B;
        int prefix = 0;
        // flag and count share one word, so relaxed (volatile) accesses
        // suffice: no fences, which would also invalidate L1
        if (tile == 0) {
            st[d] = kLbIncl | (unsigned)c;
        } else {
            st[d] = kLbAgg | (unsigned)c;
            // walk back 8 predecessors per round (independent loads in flight)
            for (int j = tile - 1; j >= 0;) {
                unsigned w[8];
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    w[q] = j - q >= 0 ? (unsigned)((volatile unsigned*)(lb + (size_t)(j - q) * B))[d] : 0u + kLbIncl;
                int q = 0;
                bool done = false;
                for (; q < 8; ++q) {
                    if ((w[q] >> 30) == 0) break;  // not published yet: reload from here
                    prefix += (int)(w[q] & kLbMask);
                    if (w[q] & kLbIncl) {
                        done = true;
                        break;
                    }
                }
                if (done) break;
                j -= q;
            }
            st[d] = kLbIncl | (unsigned)(prefix + c);
        }
        gbase[d] = gstart + prefix - lstart[d];
    }
    __syncthreads();
    // ---- stage in tile-sorted order ----
#pragma unroll
    for (int it = 0; it < kTileItems; ++it) {
        const int j = warp * 32 * kTileItems + it * 32 + lane;
        if (j < cnt) {
            const int dd = (kr[it] >> shift) & (B - 1);
            const int lp = lstart[dd] + wcnt[warp][dd] + rk[it];
            skey[lp] = kr[it];
            sval[lp] = vr[it];
        }
    }
    __syncthreads();
    // ---- write out digit runs (consecutive j -> consecutive global positions) ----
    if (!packed) {
#pragma unroll 4
        for (int j = threadIdx.x; j < cnt; j += kTileThreads) {
            const int k = skey[j];
            const int pos = gbase[(k >> shift) & (B - 1)] + j;
            kout[pos] = k;
            vout[pos] = sval[j];
        }
        return;
    }
    // last pass: also one 32-byte record per key; the random record reads of
    // a thread's keys are issued together
#pragma unroll
    for (int it = 0; it < kTileItems; it += 4) {
        Src r[4];
        int pos[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int j = (it + q) * kTileThreads + threadIdx.x;
            pos[q] = -1;
            if (j < cnt) {
                const int k = skey[j], v = sval[j];
                pos[q] = gbase[(k >> shift) & (B - 1)] + j;
                kout[pos[q]] = k;
                vout[pos[q]] = v;
                r[q] = packed[v];
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (pos[q] >= 0) src[pos[q]] = r[q];
    }
}

// ---- single-pass exclusive scan (int32, in place), decoupled look-back ----
constexpr int kScanThreads = 512;
constexpr int kScanItems = 4;
constexpr int kScanSub = 4;
constexpr int kScanTile = kScanThreads * kScanItems * kScanSub;
constexpr unsigned long long kFlagAgg = 1ull << 62, kFlagIncl = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

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

// state[0] = tile ticket, state[1 + t] = status of tile t (all zero on entry).
// Tiles are numbered by ticket, so every predecessor of a running tile has
// started and the look-back always terminates.
// A tile is kScanSub sub-tiles of kScanThreads x 4 consecutive ints (int4
// loads, fully coalesced), scanned one after another with a running carry;
// one look-back per tile keeps the serial chain short (~n / 8192 tiles).
__global__ void __launch_bounds__(kScanThreads)
    k_scan(int* __restrict__ data, int64_t n, unsigned long long* __restrict__ state,
           const Counters* __restrict__ sym_skip, bool gauss, const int* __restrict__ skip_flag,
           int skip_val) {
    pdl_enter();
    // the near-field task list is not needed when the symmetric P2P kernel runs
    if (sym_skip && p2p_symmetric(sym_skip, gauss)) return;
    if (skip_flag && *skip_flag == skip_val) return;  // leaf-count scan: counting path only
    __shared__ int warp_sums[32];
    __shared__ int total;
    __shared__ int tile_s;
    __shared__ long long prefix_s;
    if (threadIdx.x == 0) tile_s = (int)atomicAdd(&state[0], 1ull);
    __syncthreads();
    const int tile = tile_s;
    const int64_t tile_base = (int64_t)tile * kScanTile;
    int vals[kScanSub][kScanItems];
    int run[kScanSub];
    int carry = 0;
#pragma unroll
    for (int sub = 0; sub < kScanSub; ++sub) {
        const int64_t base = tile_base + (int64_t)sub * kScanThreads * kScanItems +
                             (int64_t)threadIdx.x * kScanItems;
        if (base + kScanItems <= n && (reinterpret_cast<uintptr_t>(data + base) & 15) == 0) {
            const int4 q = *reinterpret_cast<const int4*>(data + base);
            vals[sub][0] = q.x;
            vals[sub][1] = q.y;
            vals[sub][2] = q.z;
            vals[sub][3] = q.w;
        } else {
#pragma unroll
            for (int j = 0; j < kScanItems; ++j) vals[sub][j] = (base + j < n) ? data[base + j] : 0;
        }
        int s = 0;
#pragma unroll
        for (int j = 0; j < kScanItems; ++j) s += vals[sub][j];
        run[sub] = carry + block_exclusive_scan(s, warp_sums, &total);
        carry += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        volatile unsigned long long* st = state + 1;
        long long prefix = 0;
        // flag and value share one 64-bit word: relaxed (volatile) accesses, no fences
        if (tile == 0) {
            st[0] = kFlagIncl | (unsigned long long)carry;
        } else {
            st[tile] = kFlagAgg | (unsigned long long)carry;
            for (int j = tile - 1; j >= 0;) {
                const unsigned long long w = st[j];
                if ((w >> 62) == 0) continue;  // predecessor not published yet
                prefix += (long long)(w & kValMask);
                if (w & kFlagIncl) break;
                --j;
            }
            st[tile] = kFlagIncl | (unsigned long long)(prefix + carry);
        }
        prefix_s = prefix;
    }
    __syncthreads();
    const int pre = (int)prefix_s;
#pragma unroll
    for (int sub = 0; sub < kScanSub; ++sub) {
        const int64_t base = tile_base + (int64_t)sub * kScanThreads * kScanItems +
                             (int64_t)threadIdx.x * kScanItems;
        int r = run[sub] + pre;
#pragma unroll
        for (int j = 0; j < kScanItems; ++j) {
            if (base + j < n) data[base + j] = r;
            r += vals[sub][j];
        }
    }
}

// One CTA of 1024 threads for short arrays (up to 24,576 ints: the leaf
// counts of l <= 7).  The array is read as J <= 6 stripes of 1,024 int4
// (thread t holds int4 t of every stripe: every warp load is 512 contiguous
// bytes, all loads in flight together), the J stripe scans run together
// (one shuffle ladder over J values), and the results go back to the same
// int4 slots.  One global round trip, fully coalesced (the previous
// contiguous-run-per-thread layout made every load a 32-sector request:
// 11.3 us for config 2's 16,385 leaf counts under ncu, lg_throttle stalls).
constexpr int kScanOneThreads = 1024;
constexpr int kScanOneJ = 6;
constexpr int64_t kScanOneMax = (int64_t)kScanOneThreads * 4 * kScanOneJ;
__global__ void __launch_bounds__(kScanOneThreads)
    k_scan_one(int* __restrict__ data, int64_t n, const int* __restrict__ skip_flag, int skip_val) {
    pdl_enter();
    if (skip_flag && *skip_flag == skip_val) return;  // leaf-count scan: counting path only
    __shared__ int wsum[kScanOneJ][32];
    __shared__ int stripe_base[kScanOneJ];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t n4 = (n + 3) >> 2;
    const bool vec = (reinterpret_cast<uintptr_t>(data) & 15) == 0;
    int4 q[kScanOneJ];
    int s[kScanOneJ], incl[kScanOneJ];
#pragma unroll
    for (int j = 0; j < kScanOneJ; ++j) {
        const int64_t i4 = (int64_t)j * kScanOneThreads + t;
        const int64_t e = i4 * 4;
        if (vec && e + 4 <= n) {
            q[j] = __ldcg(reinterpret_cast<const int4*>(data) + i4);
        } else {
            q[j].x = e < n ? __ldcg(data + e) : 0;
            q[j].y = e + 1 < n ? __ldcg(data + e + 1) : 0;
            q[j].z = e + 2 < n ? __ldcg(data + e + 2) : 0;
            q[j].w = e + 3 < n ? __ldcg(data + e + 3) : 0;
        }
        s[j] = q[j].x + q[j].y + q[j].z + q[j].w;
        incl[j] = s[j];
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
        for (int j = 0; j < kScanOneJ; ++j) {
            const int u = __shfl_up_sync(0xffffffffu, incl[j], o);
            if (lane >= o) incl[j] += u;
        }
    }
    if (lane == 31)
#pragma unroll
        for (int j = 0; j < kScanOneJ; ++j) wsum[j][warp] = incl[j];
    __syncthreads();
    if (warp < kScanOneJ) {  // warp j scans stripe j's 32 warp sums
        const int w = wsum[warp][lane];
        int wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += u;
        }
        wsum[warp][lane] = wi - w;
        if (lane == 31) stripe_base[warp] = wi;  // stripe total (made a prefix below)
    }
    __syncthreads();
    int base = 0;
#pragma unroll
    for (int j = 0; j < kScanOneJ; ++j) {
        const int tot = stripe_base[j];
        const int64_t i4 = (int64_t)j * kScanOneThreads + t;
        const int64_t e = i4 * 4;
        if (i4 < n4) {
            int4 r;
            r.x = base + wsum[j][warp] + incl[j] - s[j];
            r.y = r.x + q[j].x;
            r.z = r.y + q[j].y;
            r.w = r.z + q[j].z;
            if (vec && e + 4 <= n) {
                reinterpret_cast<int4*>(data)[i4] = r;
            } else {
                if (e < n) data[e] = r.x;
                if (e + 1 < n) data[e + 1] = r.y;
                if (e + 2 < n) data[e + 2] = r.z;
                if (e + 3 < n) data[e + 3] = r.w;
            }
        }
        base += tot;
    }
}

__global__ void k_leaf_starts(const int* __restrict__ keys, int64_t n, int nleaves,
                              int* __restrict__ ls, const Counters* __restrict__ ctr) {
    pdl_enter();
    if (ctr && !ctr->sort_fallback) return;
    // leaf-parallel lower_bound in the sorted keys: ls[k] = first i with
    // keys[i] >= k.  (A particle-parallel fill of the gaps between consecutive
    // keys left one thread filling every empty leaf of a long gap -- the
    // leaves outside a rank's row strip: 0.8 ms at config 3 on 8 ranks.)
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k <= nleaves;
         k += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (keys[mid] < k) lo = mid + 1;
            else hi = mid;
        }
        ls[k] = (int)lo;
    }
}

__global__ void k_tasks_fill(const int* __restrict__ ls, int levels, int chunk, Rows rows,
                             const int* __restrict__ off, int2* __restrict__ tasks, Counters* ctr,
                             bool gauss, bool sym_enabled) {
    pdl_enter();
    if (sym_enabled && p2p_symmetric(ctr, gauss)) return;  // symmetric P2P: no task list
    const int nleaves = 1 << (2 * levels);
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nleaves) return;
    const int iy = i >> levels;
    const int c = ls[i + 1] - ls[i];
    const int nt = (iy >= rows.lo && iy < rows.hi) ? (c + chunk - 1) / chunk : 0;
    const int o = off[i];
    for (int t = 0; t < nt; ++t) tasks[o + t] = make_int2(i, chunk * t);
    if (i == nleaves - 1) ctr->ntasks = o + nt;
}


// VFMM_SORT=lsd forces the LSD radix path, VFMM_SORT=count keeps the probe
// from choosing it (a leaf above kFastLeafMax still does) -- tuning / tests
int sort_probe_mode() {
    static const int f = [] {
        const char* e = getenv("VFMM_SORT");
        return e ? (e[0] == 'l' ? 1 : (e[0] == 'c' ? 2 : 0)) : 0;
    }();
    return f;
}

inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }
// grid-stride kernels of the LSD fallback: at most 148 x 4 blocks of 256
inline unsigned small_grid(int64_t n, unsigned cap = 592u) {
    const unsigned g = grid_for(n, 256);
    return g < cap ? g : cap;
}

}  // namespace

void launch_init_counters(Counters* ctr, cudaStream_t s) {
    cudaMemsetAsync(ctr, 0, sizeof(Counters), s);
}

size_t scan_tiles(int64_t n) { return (size_t)((n + kScanTile - 1) / kScanTile); }

void launch_scan_i32(int* data, int64_t n, unsigned long long* state, cudaStream_t s,
                     const Counters* sym_skip, bool gauss, const int* skip_flag, int skip_val) {
    if (n <= 0) return;
    if (!sym_skip && n <= kScanOneMax) {
        launch_k(k_scan_one, 1, kScanOneThreads, 0, s, data, n, skip_flag, skip_val);
        note_launches(1);
        return;
    }
    launch_k(k_scan, (unsigned)scan_tiles(n), kScanThreads, 0, s, data, n, state, sym_skip, gauss,
                                                              skip_flag, skip_val);
    note_launches(1);
}

// Zero up to four scratch regions in one launch (the build's look-back
// states, leaf counts, slot fills and LSD histograms; memset nodes would break
// the programmatic-launch chain).
struct ZeroRegions {
    int* p[5];
    int64_t n[5];  // ints
};
struct ProbeArgs {
    const double *x, *y;
    int64_t n;
    double xmin, ymin, side;
    int levels;
    int probe_mode;
};
__device__ void sort_probe(const ProbeArgs& a, Counters* ctr) {
    // below kLsdMinN the sample cannot choose the LSD path: skip its loads (the
    // probe was the longest dependency chain of the build's first kernel)
    if (a.probe_mode == 1) {
        if (threadIdx.x == 0) ctr->sort_fallback = kSortLsdProbe;
        return;
    }
    if (a.probe_mode != 0 || a.n <= kLsdMinN) return;
    sort_probe_impl(a.x, a.y, a.n, a.xmin, a.ymin, a.side, a.levels, a.probe_mode, ctr);
}
// The build's first kernel: zero the scratch regions, and CTA 0 also runs the
// sort-path probe (one launch instead of two; the counters are zeroed by the
// memset that precedes it).
__global__ void k_zero_regions(ZeroRegions z, ProbeArgs pa, Counters* ctr) {
    pdl_enter();
    if (blockIdx.x == 0) {
        // the counters first (instead of a memset node, which would break
        // the programmatic-launch chain), then the probe that sets one of them
        for (int i = threadIdx.x; i < (int)(sizeof(Counters) / sizeof(int)); i += blockDim.x)
            reinterpret_cast<int*>(ctr)[i] = 0;
        __syncthreads();
        sort_probe(pa, ctr);
        return;
    }
    const int64_t t0 = (int64_t)(blockIdx.x - 1) * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)(gridDim.x - 1) * blockDim.x;
#pragma unroll
    for (int r = 0; r < 5; ++r)
        for (int64_t i = t0; i < z.n[r]; i += stride) z.p[r][i] = 0;
}

// Occupancy pyramid + task counts: 4^k cells x min(32, 2^(levels-k)) lanes per level.
CountsArgs counts_args(const Layout& L, char* ws, Rows rows) {
    int64_t total = 0;
    for (int k = 0; k <= L.levels; ++k) {
        const int64_t rows_k = 1ll << (L.levels - k);
        total += (1ll << (2 * k)) * (rows_k < 32 ? rows_k : 32);
    }
    CountsArgs a;
    a.ctas = (int)grid_for(total, 256);
    a.levels = L.levels;
    a.total_threads = total;
    a.chunk = 32 * p2p_targets_per_lane();
    a.rows = rows;
    a.counts = (int*)(ws + L.counts);
    a.ntask = (int*)(ws + L.task_scratch);
    return a;
}

void launch_build(const Layout& L, const double* x, const double* y, const double* g,
                  const double* sigma, double xmin, double ymin, double side, char* ws,
                  Counters* ctr, cudaStream_t s, int** keys_out, int** perm_out,
                  cudaEvent_t gs_ready, int sigma_stride, Rows rows, cudaStream_t lsd_stream,
                  cudaEvent_t lsd_fork, cudaEvent_t lsd_join) {
    const CountsArgs ca = counts_args(L, ws, rows);
    int* kbuf[2] = {(int*)(ws + L.key_a), (int*)(ws + L.key_b)};
    int* vbuf[2] = {(int*)(ws + L.val_a), (int*)(ws + L.val_b)};
    const int bits = L.digit_bits;
    const int B = 1 << bits;
    auto state = [&](int i) {
        return (unsigned long long*)(ws + L.scan_state) + (size_t)i * (L.scan_state_tiles + 1);
    };
    int* ls = (int*)(ws + L.leaf_starts);
    int* fkeys = kbuf[L.passes & 1];  // final buffers of either path (vfmm_layout_of)
    int* fperm = vbuf[L.passes & 1];
    Src* src = (Src*)(ws + L.src);
    int* fill = (int*)(ws + L.fill);          // per-leaf slot cursors of k_bin_scatter
    int* ghist = (int*)(ws + L.hist);         // LSD: passes x B global digit counts, tickets, look-back
    {
        ZeroRegions z{{(int*)(ws + L.scan_state), ls, fill, ghist, (int*)(ws + L.near_done)},
                      {(int64_t)(L.scan_state_bytes / sizeof(int)), (int64_t)L.nleaves + 1,
                       (int64_t)L.nleaves, (int64_t)L.passes * B + 8, (int64_t)L.nleaves}};
        const ProbeArgs pa{x, y, L.n, xmin, ymin, side, L.levels, sort_probe_mode()};
        launch_k(k_zero_regions, 297, 256, 0, s, z, pa, ctr);
        note_launches(1);
    }
    // ---- counting path (kernels return at once if the probe chose LSD) ----
    // Bucket mode: fixed buckets of kFastLeafMax indices per leaf in the
    // near-field slots (idle until the near field runs; the LSD path's packed
    // records use the same region later) when they fit: the count claims the
    // slots and k_bin_scatter is not launched.  VFMM_BUILD_BUCKET=0: A/B.
    static const bool bucket_env = !(getenv("VFMM_BUILD_BUCKET") && getenv("VFMM_BUILD_BUCKET")[0] == '0');
    const bool bucket = bucket_env && (size_t)L.nleaves * kFastLeafMax * sizeof(int) <=
                                          sizeof(double2) * (size_t)L.n * kNearSlotsAlloc;
    int* slot = bucket ? (int*)(ws + L.near_uv) : vbuf[(L.passes + 1) & 1];
    // Fused scan (bucket mode, l <= 7): the counts go to the (zeroed, otherwise
    // unused) slot-cursor array and k_leaf_pack derives leaf_starts from them;
    // no scan launch.  VFMM_BUILD_FUSED_SCAN=0: A/B.
    static const bool fused_env = !(getenv("VFMM_BUILD_FUSED_SCAN") && getenv("VFMM_BUILD_FUSED_SCAN")[0] == '0');
    const bool fused = bucket && fused_env && L.nleaves <= kPackFusedMaxLeaves;
    int* cnt = fused ? fill : ls;
    launch_k(k_bin_count, small_grid((L.n + kBinILP - 1) / kBinILP, 2368), 256, 0, s, x, y, L.n, xmin, ymin, side, L.levels,
                                                  kbuf[(L.passes + 1) & 1], cnt, ctr, bucket ? slot : nullptr);
    note_launches(1);
    if (!fused)
        launch_scan_i32(ls, (int64_t)L.nleaves + 1, state(L.passes + 1), s, nullptr, false,
                        &ctr->sort_fallback, kSortLsdProbe);
    if (!bucket) {
        launch_k(k_bin_scatter, small_grid((L.n + kBinILP - 1) / kBinILP, 2368) + ca.ctas, 256, 0, s, kbuf[(L.passes + 1) & 1], L.n,
                 ls, fill, slot, ctr, ca);
        note_launches(1);
    }
    CountsArgs ca_pack = ca;
    if (!bucket) ca_pack.ctas = 0;
    // The path choice is final after k_bin_scatter (a leaf > 128 switches to
    // LSD there).  With a side stream the LSD kernels -- which return at once
    // on the counting path -- run as a parallel branch joined after
    // k_leaf_pack, off the counting path's critical chain (and vice versa).
    // graph capture: the LSD kernels go into an IF node set by k_leaf_pack
    const GraphCond lsd_cond = gs_ready ? GraphCond{} : graph_cond_create(s);
    const bool branch = lsd_stream && lsd_fork && lsd_join && !lsd_cond.on;
    cudaStream_t ls_s = branch ? lsd_stream : s;
    if (branch) {
        cudaEventRecord(lsd_fork, s);
        cudaStreamWaitEvent(lsd_stream, lsd_fork, 0);
    }
    // gamma and sigma are first read by the record pack (host mode: their
    // copies overlap the binning)
    if (gs_ready) cudaStreamWaitEvent(s, gs_ready, 0);
    const unsigned pack_grid = fused ? std::min(grid_for((int64_t)L.nleaves, 8), (unsigned)kPackFusedGrid)
                                     : std::min(grid_for((int64_t)L.nleaves, 8), 2368u);
    launch_k(k_leaf_pack, pack_grid + (unsigned)ca_pack.ctas, 256, 0, s, ls, slot,
                                                              (int)L.nleaves, x, y, g,
                                                              sigma, sigma_stride, fkeys, fperm,
                                                              src, ctr, lsd_cond, bucket ? kFastLeafMax : 0, ca_pack,
                                                              fused ? (const int*)cnt : (const int*)nullptr);
    note_launches(1);
    cudaGraphNode_t lsd_node = nullptr;
    if (lsd_cond.on) ls_s = graph_cond_begin(s, lsd_cond, &lsd_node);

    // ---- LSD radix path (kernels return at once unless ctr->sort_fallback) ----
    Src* packed = (Src*)(ws + L.near_uv);  // free until the near field runs (>= 32 B per particle)
    int* tickets = ghist + L.passes * B;
    unsigned* lbase = (unsigned*)(tickets + 8);
    const size_t lb_words = (size_t)L.nchunks * B;
    const unsigned tiles = (unsigned)L.nchunks;
    launch_k(k_keys_ghist, tiles, kTileThreads, 0, ls_s, x, y, L.n, xmin, ymin, side, L.levels, bits,
             L.passes, kbuf[0], ghist, lbase, (int64_t)lb_words, ctr);
    note_launches(1);
    for (int p = 0; p < L.passes; ++p) {
        const bool last = p == L.passes - 1;
        if (last) {
            if (branch && gs_ready) cudaStreamWaitEvent(ls_s, gs_ready, 0);
            launch_k(k_pack_orig, small_grid(L.n), 256, 0, ls_s, x, y, g, sigma, sigma_stride, L.n, packed,
                                                          ctr);
            note_launches(1);
        }
        launch_k(k_onesweep, tiles, kTileThreads, 0, ls_s, 
            kbuf[p & 1], p == 0 ? nullptr : vbuf[p & 1], kbuf[(p + 1) & 1], vbuf[(p + 1) & 1], L.n,
            p * bits, bits, ghist + p * B, lbase + p * lb_words, tickets + p, last ? packed : nullptr,
            src, ctr);
        note_launches(1);
    }
    *keys_out = fkeys;
    *perm_out = fperm;
    launch_k(k_leaf_starts, small_grid((int64_t)L.nleaves + 1, 2368), 256, 0, ls_s, fkeys, L.n,
             (int)L.nleaves, ls, ctr);
    note_launches(1);
    launch_k(k_counts_tasks, (unsigned)ca.ctas, 256, 0, ls_s, (const int*)ls, ca, ctr);
    note_launches(1);
    if (lsd_cond.on) graph_cond_end(s, ls_s, lsd_node);
    if (branch) {
        cudaEventRecord(lsd_join, lsd_stream);
        cudaStreamWaitEvent(s, lsd_join, 0);
    }
}

void launch_leaf_starts(const int* sorted_keys, int64_t n, int nleaves, int* leaf_starts,
                        cudaStream_t s) {
    launch_k(k_leaf_starts, grid_for((int64_t)nleaves + 1, 256), 256, 0, s, sorted_keys, n, nleaves, leaf_starts,
                                                        nullptr);
    note_launches(1);
}

// Near-field task list of the generic kernel (launched on the near stream
// right before it, after the symmetric kernel; both return at once when the
// symmetric kernel ran).
void launch_tasks(const Layout& L, char* ws, Counters* ctr, Rows rows, bool gauss, cudaStream_t s) {
    const int* ls = (const int*)(ws + L.leaf_starts);
    int* nt = (int*)(ws + L.task_scratch);
    const int chunk = 32 * p2p_targets_per_lane();
    const int nl = (int)L.nleaves;
    const bool sym = !sym_disabled();
    launch_scan_i32(nt, nl, (unsigned long long*)(ws + L.scan_state) +
                                (size_t)L.passes * (L.scan_state_tiles + 1), s,
                    sym ? ctr : nullptr, gauss);
    launch_k(k_tasks_fill, grid_for(nl, 256), 256, 0, s, ls, L.levels, chunk, rows, nt,
                                                 (int2*)(ws + L.tasks), ctr, gauss, sym);
    note_launches(1);
}

}  // namespace vfmm
