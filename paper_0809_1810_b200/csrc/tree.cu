// Uniform-quadtree construction on the GPU (north-star item 1).
//
// Replaces quadtree.build_tree / grid_indices / Tree.__init__
// (quadtree.py:39-46, 116-134, 182-201) and the permutation in
// engine.evaluate (engine.py:355-358).  Kernel sequence (config 2: 9 launches):
//   k_keys_hist     floor-rule binning with max-edge clamp + domain check + max
//                   sigma + digit-0 histogram per warp chunk; zeroes scratch
//   k_scan          single-pass exclusive scan (decoupled look-back)
//   k_radix_scatter stable LSD scatter; also histograms the next digit per
//                   output chunk; the last pass gathers x, y, gamma, sigma
//                   into the sorted Src records (np.argsort(kind="stable"))
//   k_leaf_starts   leaf_starts[4^l + 1] (== concatenate([0], cumsum(bincount)))
//   k_counts_tasks  per-level occupancy pyramid (Tree.counts) + P2P task counts
//   k_scan, k_tasks_fill   near-field warp task list
#include <climits>

#include "vfmm_internal.cuh"

namespace vfmm {

namespace {

constexpr int kWPB = 8;  // warps per block in the radix kernels

__device__ __forceinline__ unsigned long long ordered_bits(double d) {
    unsigned long long b = (unsigned long long)__double_as_longlong(d);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

// Warp chunk c = elements [c*wc, (c+1)*wc).  Also zeroes the scratch words
// (later histograms, scan look-back state) with a grid-stride loop.
__global__ void __launch_bounds__(kWPB * 32)
    k_keys_hist(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                double xmin, double ymin, double side,
                int levels, int bits, int wc, int nchunks, int* __restrict__ key,
                int* __restrict__ hist0, unsigned* __restrict__ zero, int64_t nzero,
                Counters* __restrict__ ctr) {
    extern __shared__ int sh[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t z = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; z < nzero;
         z += (int64_t)gridDim.x * blockDim.x)
        zero[z] = 0u;
    const int B = 1 << bits;
    int* h = sh + warp * B;
    for (int d = lane; d < B; d += 32) h[d] = 0;
    __syncwarp();
    const int m = 1 << levels;
    const double xmax = xmin + side, ymax = ymin + side;  // Domain.xmax (model.py:51-57)
    const int64_t chunk = (int64_t)blockIdx.x * kWPB + warp;
    if (chunk < nchunks) {
        const int64_t beg = chunk * wc;
        const int64_t end = beg + wc < n ? beg + wc : n;
        constexpr int R = 8;  // rounds whose loads are issued together
        for (int64_t b0 = beg; b0 < end; b0 += 32 * R) {
            double xr[R], yr[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int64_t i = b0 + 32 * r + lane;
                xr[r] = i < end ? x[i] : 0.0;
                yr[r] = i < end ? y[i] : 0.0;
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int64_t i = b0 + 32 * r + lane;
                if (i >= end) continue;
                const double xi = xr[r], yi = yr[r];
                const bool inside = (xi >= xmin) && (xi <= xmax) && (yi >= ymin) && (yi <= ymax);
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
                    atomicMax(&ctr->first_bad_neg, INT_MAX - (int)i);
                }
                const int k = iy * m + ix;
                key[i] = k;
                atomicAdd(&h[k & (B - 1)], 1);
            }
        }
        __syncwarp();
        for (int d = lane; d < B; d += 32) hist0[(int64_t)d * nchunks + chunk] = h[d];
    }
}

// Source records in ORIGINAL order (coalesced), with the sigma statistics;
// the last radix pass then moves whole 32-byte records instead of gathering
// four arrays element by element.
__global__ void __launch_bounds__(256)
    k_pack_orig(const double* __restrict__ x, const double* __restrict__ y,
                const double* __restrict__ g, const double* __restrict__ sigma, int64_t n,
                Src* __restrict__ out, Counters* __restrict__ ctr) {
    __shared__ unsigned long long wmax[8], wmin[8];
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long sbits = 0ull, smin = ~0ull;
    if (i < n) {
        const double s = sigma ? sigma[i] : 1.0;
        if (sigma) sbits = smin = ordered_bits(s);
        Src r;
        r.x = x[i];
        r.y = y[i];
        r.g = g[i];
        // -r^2 / (2 sigma^2) (engine.py:256) expressed in log2 units
        r.q2 = -1.4426950408889634 / (2.0 * s * s);
        out[i] = r;
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

// Stable scatter of one LSD pass: warp chunks are processed in index order,
// lanes in index order within a round, equal digits ranked by lane
// (match_any), so the relative order of equal keys is preserved.  Non-final
// passes histogram the next digit per OUTPUT chunk (integer atomics: the
// counts are exact); the final pass writes the packed Src records.
__global__ void __launch_bounds__(kWPB * 32)
    k_radix_scatter(const int* __restrict__ kin, const int* __restrict__ vin,
                    int* __restrict__ kout, int* __restrict__ vout, int64_t n, int shift, int bits,
                    int wc, int nchunks, const int* __restrict__ offs, int* __restrict__ hist_next,
                    const Src* __restrict__ packed, Src* __restrict__ src) {
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
    constexpr int R = 8;  // rounds whose loads are issued together
    for (int64_t base0 = beg; base0 < end; base0 += 32 * R) {
        int kr[R], vr[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int64_t i = base0 + 32 * r + lane;
            kr[r] = i < end ? kin[i] : 0;
            vr[r] = i < end ? (vin ? vin[i] : (int)i) : 0;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int64_t i = base0 + 32 * r + lane;
            const bool valid = i < end;
            const int k = kr[r], v = vr[r];
            const int d = valid ? (k >> shift) & (B - 1) : B + lane;
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            const int rank = __popc(peers & lt);
            if (valid) {
                const int pos = run[d] + rank;
                kout[pos] = k;
                vout[pos] = v;
                if (hist_next)
                    atomicAdd(&hist_next[(int64_t)((k >> (shift + bits)) & (B - 1)) * nchunks + pos / wc], 1);
                else
                    src[pos] = packed[v];  // one 32-byte record
            }
            __syncwarp();
            if (valid && rank == __popc(peers) - 1) run[d] += __popc(peers);
            __syncwarp();
        }
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
           const Counters* __restrict__ sym_skip, bool gauss) {
    // the near-field task list is not needed when the symmetric P2P kernel runs
    if (sym_skip && p2p_symmetric(sym_skip, gauss)) return;
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
        if (tile == 0) {
            __threadfence();
            st[0] = kFlagIncl | (unsigned long long)carry;
        } else {
            st[tile] = kFlagAgg | (unsigned long long)carry;
            __threadfence();
            for (int j = tile - 1; j >= 0;) {
                const unsigned long long w = st[j];
                if ((w >> 62) == 0) continue;  // predecessor not published yet
                prefix += (long long)(w & kValMask);
                if (w & kFlagIncl) break;
                --j;
            }
            __threadfence();
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

__global__ void k_leaf_starts(const int* __restrict__ keys, int64_t n, int nleaves,
                              int* __restrict__ ls) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n) return;
    const int prev = i > 0 ? keys[i - 1] : -1;
    const int cur = i < n ? keys[i] : nleaves;
    for (int k = prev + 1; k <= cur; ++k) ls[k] = (int)i;
}

// Occupancy of every cell of every level (level 0 first) from leaf_starts
// (Tree.counts, quadtree.py:126-134):
// a level-k cell covers 2^(l-k) leaf rows, each a contiguous leaf range.
// Leaf cells also emit their P2P task count ceil(count / chunk).
__global__ void k_counts_tasks(const int* __restrict__ ls, int levels, int64_t total_cells,
                               int chunk, Rows rows, int* __restrict__ counts,
                               int* __restrict__ ntask, Counters* __restrict__ ctr) {
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
    // only owned leaf rows are counted, so per-rank pyramids of a sharded run
    // are disjoint and their sum is the global occupancy
    const int r0 = max(iy * s, rows.lo), r1 = min((iy + 1) * s, rows.hi);
    int c = 0;
    for (int r = r0; r < r1; ++r) {
        const int64_t row = (int64_t)r * m;
        c += ls[row + (int64_t)(ix + 1) * s] - ls[row + (int64_t)ix * s];
    }
    counts[t] = c;
    // only leaves of the owned row strip get near-field tasks
    int full = 0;
    if (k == levels) {
        ntask[cell] = (iy >= rows.lo && iy < rows.hi) ? (c + chunk - 1) / chunk : 0;
        full = ls[cell + 1] - ls[cell];  // owned and halo rows (the symmetric P2P touches both)
    }
    // largest leaf: one atomic per warp
    full = __reduce_max_sync(__activemask(), full);
    if ((threadIdx.x & 31) == (__ffs(__activemask()) - 1) && full > 0) atomicMax(&ctr->max_leaf, full);
}

__global__ void k_tasks_fill(const int* __restrict__ ls, int levels, int chunk, Rows rows,
                             const int* __restrict__ off, int2* __restrict__ tasks, Counters* ctr,
                             bool gauss, bool sym_enabled) {
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


inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }

}  // namespace

void launch_init_counters(Counters* ctr, cudaStream_t s) {
    cudaMemsetAsync(ctr, 0, sizeof(Counters), s);
}

size_t scan_tiles(int64_t n) { return (size_t)((n + kScanTile - 1) / kScanTile); }

void launch_scan_i32(int* data, int64_t n, unsigned long long* state, cudaStream_t s,
                     const Counters* sym_skip, bool gauss) {
    if (n <= 0) return;
    k_scan<<<(unsigned)scan_tiles(n), kScanThreads, 0, s>>>(data, n, state, sym_skip, gauss);
    note_launches(1);
}

void launch_build(const Layout& L, const double* x, const double* y, const double* g,
                  const double* sigma, double xmin, double ymin, double side, char* ws,
                  Counters* ctr, cudaStream_t s, int** keys_out, int** perm_out,
                  cudaEvent_t gs_ready) {
    int* kbuf[2] = {(int*)(ws + L.key_a), (int*)(ws + L.key_b)};
    int* vbuf[2] = {(int*)(ws + L.val_a), (int*)(ws + L.val_b)};
    const int bits = L.digit_bits;
    const int B = 1 << bits;
    const int64_t hsize = (int64_t)B * L.nchunks;
    auto hist = [&](int p) { return (int*)(ws + L.hist) + p * hsize; };
    auto state = [&](int i) {
        return (unsigned long long*)(ws + L.scan_state) + (size_t)i * (L.scan_state_tiles + 1);
    };
    const unsigned blocks = (unsigned)((L.nchunks + kWPB - 1) / kWPB);
    const size_t shm = (size_t)kWPB * B * sizeof(int);
    Src* packed = (Src*)(ws + L.near_uv);  // free until the near field runs (9 x 16 B >= 32 B per particle)
    // scratch zeroed by the first kernel: histograms of passes 1.. and all scan states
    unsigned* zero = (unsigned*)(ws + L.hist) + hsize;
    const int64_t nzero_hist = hsize * (L.passes - 1);
    k_keys_hist<<<blocks, kWPB * 32, shm, s>>>(x, y, L.n, xmin, ymin, side, L.levels, bits,
                                              L.wc, L.nchunks, kbuf[0], hist(0), zero, nzero_hist,
                                              ctr);
    note_launches(1);
    cudaMemsetAsync(ws + L.scan_state, 0, L.scan_state_bytes, s);
    for (int p = 0; p < L.passes; ++p) {
        launch_scan_i32(hist(p), hsize, state(p), s, nullptr, false);
        const bool last = p == L.passes - 1;
        // gamma and sigma are first read by the record pack before the last
        // pass (host mode: their copies overlap the key / sort work)
        if (last) {
            if (gs_ready) cudaStreamWaitEvent(s, gs_ready, 0);
            k_pack_orig<<<grid_for(L.n, 256), 256, 0, s>>>(x, y, g, sigma, L.n, packed, ctr);
            note_launches(1);
        }
        k_radix_scatter<<<blocks, kWPB * 32, shm, s>>>(
            kbuf[p & 1], p == 0 ? nullptr : vbuf[p & 1], kbuf[(p + 1) & 1], vbuf[(p + 1) & 1], L.n,
            p * bits, bits, L.wc, L.nchunks, hist(p), last ? nullptr : hist(p + 1), packed,
            (Src*)(ws + L.src));
        note_launches(1);
    }
    *keys_out = kbuf[L.passes & 1];
    *perm_out = vbuf[L.passes & 1];
    int* ls = (int*)(ws + L.leaf_starts);
    launch_leaf_starts(*keys_out, L.n, (int)L.nleaves, ls, s);
}

void launch_leaf_starts(const int* sorted_keys, int64_t n, int nleaves, int* leaf_starts,
                        cudaStream_t s) {
    k_leaf_starts<<<grid_for(n + 1, 256), 256, 0, s>>>(sorted_keys, n, nleaves, leaf_starts);
    note_launches(1);
}

void launch_counts_tasks(const Layout& L, char* ws, Counters* ctr, bool tasks, Rows rows,
                         bool gauss, cudaStream_t s) {
    const int* ls = (const int*)(ws + L.leaf_starts);
    int* counts = (int*)(ws + L.counts);
    int* nt = (int*)(ws + L.task_scratch);
    int64_t total = 0;
    for (int k = 0; k <= L.levels; ++k) total += 1ll << (2 * k);
    const int chunk = 32 * p2p_targets_per_lane();
    k_counts_tasks<<<grid_for(total, 256), 256, 0, s>>>(ls, L.levels, total, chunk, rows, counts,
                                                       nt, ctr);
    note_launches(1);
    if (!tasks) return;
    const int nl = (int)L.nleaves;
    const bool sym = !sym_disabled();
    launch_scan_i32(nt, nl, (unsigned long long*)(ws + L.scan_state) +
                                (size_t)L.passes * (L.scan_state_tiles + 1), s,
                    sym ? ctr : nullptr, gauss);
    k_tasks_fill<<<grid_for(nl, 256), 256, 0, s>>>(ls, L.levels, chunk, rows, nt,
                                                 (int2*)(ws + L.tasks), ctr, gauss, sym);
    note_launches(1);
}

}  // namespace vfmm
