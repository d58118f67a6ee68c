// Subtree-fused M2M and L2L (the level loops of engine.upward_pass,
// engine.py:136-146, and engine.downward_pass, engine.py:190-202).
//
// One CTA owns the subtree of one cell and walks `depth` levels inside shared
// memory, so the level-by-level sweep of the pyramid costs ceil(levels/3)
// launches instead of one launch (and one global round trip) per level.
// The arithmetic is the scaled operators of vfmm_internal.cuh:
//   M2M  P_m  = 2^-(m+1) sum_{k<=m} M_k E_q[m-k]         children in quadrant order
//   L2L  Lh'_n = M2L_n + sum_{m>=n} (2^-m Lh_m) F_q[m-n]  (M2L part + parent shift)
// Local cell ids: sub-level s (0 = the CTA's root cell) holds a 2^s x 2^s grid.
#include <cstdio>
#include <cstdlib>

#include "vfmm_internal.cuh"

namespace vfmm {

namespace {

constexpr int kSubThreads = 256;


__device__ __forceinline__ int sub_off(int s) { return ((1 << (2 * s)) - 1) / 3; }  // cells before sub-level s

// Upward: CTA per cell at level lt = lf - depth; reads the 4^depth cells at
// level lf (global, planar), writes levels lf-1 .. lt.
__global__ void __launch_bounds__(kSubThreads)
    k_m2m_subtree(double2* __restrict__ mult, int lf, int depth, int P, size_t off_lf,
                  const Tables* __restrict__ T, int levels, Rows rows) {
    pdl_enter();
    {
        // sharded runs are strip-local: a subtree outside the owned row strip
        // is not visited (its cells are neither read nor written here; the
        // multipole exchange supplies what the strip's M2L needs)
        const int lt0 = lf - depth, mt0 = 1 << lt0;
        if (!rows_touch(rows, (int)(blockIdx.x / mt0), levels - lt0)) return;
    }
    extern __shared__ double2 sm[];  // [sub_off(depth+1)][P] cells + tables
    double2* sE = sm + (size_t)sub_off(depth + 1) * P;  // [4][P]
    double* s2 = reinterpret_cast<double*>(sE + 4 * P);  // [P + 1]
    for (int i = threadIdx.x; i < 4 * P; i += blockDim.x) sE[i] = T->E[i / P][i % P];
    for (int i = threadIdx.x; i <= P; i += blockDim.x) s2[i] = T->pow2neg[i];
    const int lt = lf - depth;
    const int mt = 1 << lt;
    const int cx = blockIdx.x % mt, cy = blockIdx.x / mt;
    // load the leaf-side cells of the subtree
    {
        const int side = 1 << depth;
        const int ncell = side * side;
        const double2* src = mult + off_lf;
        const int64_t cs = coef_stride(lf);
        double2* dst = sm + (size_t)sub_off(depth) * P;
        // coefficient-major order with the subtree's cells of one parity plane
        // row consecutive: runs of side/2 cells are contiguous in the planar
        // layout (the cell-major order read 16 B per coefficient stride)
        const int hs = side >> 1;  // cells per plane row of the subtree (side >= 2)
        // the whole subtree inside the strip (always on one GPU): no masking
        const bool inside = ((cy * side) << (levels - lf)) >= rows.lo &&
                            ((cy * side + side) << (levels - lf)) <= rows.hi;
        for (int i = threadIdx.x; i < ncell * P; i += blockDim.x) {
            // (powers of two: shifts and masks instead of runtime divisions)
            const int k = i >> (2 * depth), r = i & (ncell - 1);
            const int plane = r >> (2 * depth - 2), hy = (r >> (depth - 1)) & (hs - 1), hx = r & (hs - 1);
            const int lx = 2 * hx + (plane & 1), ly = 2 * hy + (plane >> 1);
            // cells whose leaf rows lie outside the strip contribute nothing
            // (sharded partial sums: a coarse parent collects only this rank's
            // children; the exchange adds the other ranks' partials)
            const int gy = cy * side + ly;
            dst[(ly * side + lx) * P + k] = (inside || rows_touch(rows, gy, levels - lf))
                                                ? src[coef_base(lf, cx * side + lx, gy) + k * cs]
                                                : make_double2(0.0, 0.0);
        }
    }
    __syncthreads();
    // reduce level by level: sub-level s+1 -> s
    size_t off_level = off_lf;  // running global offset of the level being written
    for (int s = depth - 1; s >= 0; --s) {
        const int lvl = lt + s;
        off_level -= (size_t)(1ll << (2 * lvl)) * P;  // levels are stored coarse-first
        const int side = 1 << s;
        const double2* child = sm + (size_t)sub_off(s + 1) * P;
        double2* par = sm + (size_t)sub_off(s) * P;
        double2* gout = mult + off_level;
        const int64_t cs = coef_stride(lvl);
        // 8 lanes per output coefficient: lane l8 sums the terms (q, k) with
        // 4k + q = l8 mod 8 of the 4 (mm+1) terms, then an xor-shuffle
        // reduction (the serial chains were up to 72 terms long, on 18 of 256
        // threads at the subtree root)
        const int nitem = side * side * P;
        const int l8 = threadIdx.x & 7;
        for (int i0 = 0; i0 < nitem; i0 += kSubThreads / 8) {  // block-uniform trip count
            const int i = i0 + (threadIdx.x >> 3);
            const bool act = i < nitem;
            // coefficient-major: consecutive groups write consecutive cells
            const int c = act ? i & (side * side - 1) : 0, mm = act ? i >> (2 * s) : 0;
            const int px = c & (side - 1), py = c >> s;
            double ax = 0.0, ay = 0.0;
            if (act) {
                for (int t = l8; t < 4 * (mm + 1); t += 8) {
                    const int q = t & 3, k = t >> 2;
                    const int chx = 2 * px + (q & 1), chy = 2 * py + (q >> 1);
                    const double2 a = child[(size_t)(chy * 2 * side + chx) * P + k];
                    const double2 e = sE[q * P + mm - k];
                    ax = fma(a.x, e.x, fma(-a.y, e.y, ax));
                    ay = fma(a.x, e.y, fma(a.y, e.x, ay));
                }
            }
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) {
                ax += __shfl_xor_sync(0xffffffffu, ax, o);
                ay += __shfl_xor_sync(0xffffffffu, ay, o);
            }
            if (act && l8 == 0) {
                const double2 r = make_double2(ax * s2[mm + 1], ay * s2[mm + 1]);
                par[c * P + mm] = r;
                gout[coef_base(lvl, cx * side + px, cy * side + py) + mm * cs] = r;
            }
        }
        __syncthreads();
    }
}

// Whole L2L in ONE launch: CTA per cell at the split level ls (the deepest
// level whose subtree fits shared memory).  Each CTA first walks the chain of
// its ancestors 2 -> ls (P outputs per level; the ancestors are recomputed by
// every CTA below them -- identical arithmetic, so identical values -- and
// written by the first CTA of each), then completes its subtree as above.
// Replaces ceil((levels - 2) / depth) dependent launches whose first ones
// ran on a handful of CTAs.
// coefficient offset of level k (>= 2) in mult / loc: cells of levels 2..k-1
__device__ __forceinline__ int64_t lvl_off(int k, int P) {
    return (((int64_t)1 << (2 * k)) - 16) / 3 * P;
}

// CTA size: 128 threads (8 CTAs/SM: config 2's 1,024 CTAs in one wave;
// downward 0.050 -> 0.043 ms, config 3 1.69 -> 1.47 ms) unless the grid is
// small (config 1: 64 CTAs, where 256 threads per CTA are faster).
// STAGED (large inputs; launch_l2l): when the build found the input order random
// (the LSD sort path), the un-permuting stores -- 16-byte writes to random
// sectors of an output far larger than L2, i.e. a DRAM read-modify-write each
// -- go through k_unpermute's buckets instead (see there).  Its own instance,
// so the instance every other call uses is unchanged.
template <int kL2LThreads, bool STAGED = false>
__global__ void __launch_bounds__(kL2LThreads, kL2LThreads == 128 ? 8 : 4)
    k_l2l_fused(double2* __restrict__ loc, double2* __restrict__ leaf_loc,
                const double2* __restrict__ anc_m2l, int ls, int levels, int P,
                const Tables* __restrict__ T, Rows rows, FusedOut fo) {
#ifdef VFMM_L2L_TRACE
    unsigned long long tr[8];
    int ntr = 0;
    auto mark = [&]() { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr[ntr])); ++ntr; };
    mark();
#else
    auto mark = [&]() {};
#endif
    pdl_enter();
    mark();
    // a staged call launches both instances: each runs only on its sort path
    if (fo.stage && (fo.ctr->sort_fallback == kSortPathLsdProbe) != STAGED) return;
    extern __shared__ double2 sm[];
    const int depth = levels - ls;
    double2* sF = sm + (size_t)sub_off(depth + 1) * P;  // [4][P]
    double* s2 = reinterpret_cast<double*>(sF + 4 * P);  // [P]
    double2* anc = reinterpret_cast<double2*>(s2 + ((P + 1) & ~1));  // [2][P] ping-pong
    double* sfact = reinterpret_cast<double*>(anc + 2 * P);           // [P] 1/k!
    double2* apart = reinterpret_cast<double2*>(sfact + ((P + 1) & ~1));  // [ls - 2][P] M2L parts
    const int mt = 1 << ls;
    const int cx = blockIdx.x % mt, cy = blockIdx.x / mt;
    if (!rows_touch(rows, cy, levels - ls)) return;  // subtree outside the owned strip
    // ---- every global read of the tables, the chain and the subtree, issued
    // together: element e of one flat index space [F tables 4P | level 2 P |
    // ancestors' M2L parts (ls-2)P | subtree levels 1..depth] is fetched into
    // registers by thread e mod blockDim in round e / blockDim, all rounds'
    // loads before any shared-memory store (the level-by-level loops had
    // waited one memory latency per loop and round: ~5 us of the CTA's life).
    // The chain's M2L parts of shared ancestors (k < ls) come from the
    // read-only copy, since their writer CTA completes them in loc while
    // others still read.
    const unsigned pmag = (unsigned)((0x100000000ull + P - 1) / P);  // i / P = umulhi(i, pmag), i < 2^16
    const int nA = (4 + 1 + (ls - 2)) * P, nAll = nA + sub_off(depth + 1) * P - P;
    auto fetch = [&](int e, double2*& dst) -> double2 {
        if (e < 4 * P) {  // L2L quadrant tables
            const int q = (int)__umulhi((unsigned)e, pmag);
            dst = sF + e;
            return T->F[q][e - q * P];
        }
        if (e < 5 * P) {  // level 2 ancestor
            const int n = e - 4 * P, sh = ls - 2;
            dst = anc + n;
            return loc[lvl_off(2, P) + coef_base(2, cx >> sh, cy >> sh) + n * coef_stride(2)];
        }
        if (e < nA) {  // M2L parts of the ancestors 3..ls
            const int i = e - 5 * P;
            const int kk = (int)__umulhi((unsigned)i, pmag), n = i - kk * P, k = 3 + kk, sh = ls - k;
            const int64_t gi = lvl_off(k, P) + coef_base(k, cx >> sh, cy >> sh) + n * coef_stride(k);
            dst = apart + i;
            return k < ls ? anc_m2l[gi] : loc[gi];
        }
        // subtree: cell c >= 1 (sub-level sl) coefficient k
        const int i = e - nA + P;  // index into sm (cells from 1)
        const int c = (int)__umulhi((unsigned)i, pmag), k = i - c * P;
        int sl = 1;
        while (sub_off(sl + 1) <= c) ++sl;
        const int side = 1 << sl, lc = c - sub_off(sl), lvl = ls + sl;
        dst = sm + i;
        return loc[lvl_off(lvl, P) + coef_base(lvl, cx * side + (lc & (side - 1)), cy * side + (lc >> sl)) +
                   k * coef_stride(lvl)];
    };
    constexpr int kPre = 8;
    for (int e0 = 0; e0 < nAll; e0 += kPre * kL2LThreads) {
        double2 v[kPre];
        double2* d[kPre];
#pragma unroll
        for (int j = 0; j < kPre; ++j) {
            const int e = e0 + j * kL2LThreads + threadIdx.x;
            d[j] = nullptr;
            if (e < nAll) v[j] = fetch(e, d[j]);
        }
#pragma unroll
        for (int j = 0; j < kPre; ++j)
            if (d[j]) *d[j] = v[j];
    }
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        s2[i] = T->pow2neg[i];
        sfact[i] = T->invfact[i];
    }
    __syncthreads();
    mark();
    // ---- ancestor chain: level 2 (complete after M2L) down to ls ----
    // output n of a level is summed by 8 lanes (terms mm = n + lane8, step 8)
    // and reduced by xor shuffles: P x 8 threads instead of P serial sums
    int cur = 0;
    const int l8 = threadIdx.x & 7;
    for (int k = 3; k <= ls; ++k) {
        const int sh = ls - k;
        const int ax = cx >> sh, ay = cy >> sh;
        const double2* Lp = anc + cur * P;
        const double2* Fq = sF + (2 * (ay & 1) + (ax & 1)) * P;
        for (int n0 = 0; n0 < P; n0 += kL2LThreads / 8) {  // block-uniform trip count
            const int n = n0 + (threadIdx.x >> 3);
            const bool nact = n < P;
            double sx = 0.0, sy = 0.0;
            if (nact) {
                for (int mm = n + l8; mm < P; mm += 8) {
                    const double2 a = Lp[mm];
                    const double axs = a.x * s2[mm], ays = a.y * s2[mm];
                    const double2 f = Fq[mm - n];
                    sx = fma(axs, f.x, fma(-ays, f.y, sx));
                    sy = fma(axs, f.y, fma(ays, f.x, sy));
                }
            }
            // 8-lane groups are aligned within a warp; every lane takes part
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) {
                sx += __shfl_xor_sync(0xffffffffu, sx, o);
                sy += __shfl_xor_sync(0xffffffffu, sy, o);
            }
            if (nact && l8 == 0) {
                const int64_t gi = lvl_off(k, P) + coef_base(k, ax, ay) + n * coef_stride(k);
                double2 r = apart[(k - 3) * P + n];
                r.x += sx;
                r.y += sy;
                anc[(cur ^ 1) * P + n] = r;
                const int mask = (1 << sh) - 1;
                if ((cx & mask) == 0 && (cy & mask) == 0) {  // first CTA below: the writer
                    if (k == levels)
                        leaf_loc[((int64_t)ay * (1 << k) + ax) * P + n] = r;
                    else
                        loc[gi] = r;
                }
            }
        }
        __syncthreads();
        cur ^= 1;
    }
    mark();
    if (depth == 0) return;
    // ---- subtree below the root ----
    // parents are kept in shared memory pre-multiplied by 2^-m (exact: a
    // power of two), the factor the shift applies to every term
    for (int k = threadIdx.x; k < P; k += blockDim.x) {
        const double2 a = anc[cur * P + k];
        sm[k] = make_double2(a.x * s2[k], a.y * s2[k]);
    }
    __syncthreads();
    for (int s = 1; s <= depth; ++s) {
        const int lvl = ls + s;
        const int side = 1 << s;
        const double2* par = sm + (size_t)sub_off(s - 1) * P;
        double2* cu = sm + (size_t)sub_off(s) * P;
        double2* g = loc + lvl_off(lvl, P);
        const int64_t cs = coef_stride(lvl);
        const bool leaf = lvl == levels;
        const int m = 1 << lvl;
        for (int i = threadIdx.x; i < side * side * P; i += blockDim.x) {
            const int c = (int)__umulhi((unsigned)i, pmag), nn = i - c * P;
            const int lx = c & (side - 1), ly = c >> s;
            const int q = 2 * (ly & 1) + (lx & 1);
            const double2* Lp = par + (size_t)((ly >> 1) * (side >> 1) + (lx >> 1)) * P;
            const double2* Fq = sF + q * P;
            double sx = 0.0, sy = 0.0;
            for (int mm = nn; mm < P; ++mm) {
                const double2 a = Lp[mm];  // 2^-mm Lh_mm
                const double2 f = Fq[mm - nn];
                sx = fma(a.x, f.x, fma(-a.y, f.y, sx));
                sy = fma(a.x, f.y, fma(a.y, f.x, sy));
            }
            double2 r = cu[i];  // M2L part (staged)
            r.x += sx;
            r.y += sy;
            // next level's parents: 2^-n Lh_n; the leaf level keeps Lh_n / n!
            // for the fused L2P (eval_local's per-particle products, formed
            // once per leaf)
            const double sc = leaf ? sfact[nn] : s2[nn];
            cu[i] = leaf && !fo.u ? r : make_double2(r.x * sc, r.y * sc);
            const int gx = cx * side + lx, gy = cy * side + ly;
            if (leaf)
                leaf_loc[((int64_t)gy * m + gx) * P + nn] = r;
            else
                g[coef_base(lvl, gx, gy) + nn * cs] = r;
        }
        __syncthreads();
    }
    mark();
    if (!fo.u) return;
    // ---- fused L2P + combine over the particles of this CTA's leaves ----
    // (the leaf locals are in shared memory; one contiguous particle range per
    // leaf row of the subtree)
    const int side = 1 << depth, m = 1 << levels;
    const double r = fo.side / m, inv_r = 1.0 / r;
    const double2* leafs = sm + (size_t)sub_off(depth) * P;
    // the particles of the subtree's leaf rows (one contiguous sorted range per
    // row) as one flat index space, so each thread batches kB particles' loads
    __shared__ int rb[16], rp[17];
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int ly = 0; ly < side; ++ly) {
            const int gy = cy * side + ly;
            rb[ly] = 0;
            rp[ly] = acc;
            if (gy < rows.lo || gy >= rows.hi) continue;  // halo rows of a sharded run
            const int row = gy * m + cx * side;
            const int a0 = fo.ls[row], a1 = fo.ls[row + side];
            rb[ly] = a0;
            acc += a1 - a0;
        }
        rp[side] = acc;
    }
    __syncthreads();
    const int total = rp[side];
    // Staged output: the CTA counts its particles per destination bucket in
    // shared memory, claims one range per bucket from the global cursors
    // (~4 particles per claim at config 3 instead of one global atomic each),
    // then places its records by shared-memory ranks.
    __shared__ int s_cnt[STAGED ? 1024 : 1], s_base[STAGED ? 1024 : 1];
    if (STAGED) {
        const int nbk = (int)(((int64_t)fo.n_total + ((int64_t)1 << fo.stage_shift) - 1) >> fo.stage_shift);
        for (int b = threadIdx.x; b < nbk; b += kL2LThreads) s_cnt[b] = 0;
        __syncthreads();
        for (int idx = threadIdx.x; idx < total; idx += kL2LThreads) {
            int ly = 0;
            while (ly + 1 < side && rp[ly + 1] <= idx) ++ly;
            atomicAdd(&s_cnt[fo.perm[rb[ly] + idx - rp[ly]] >> fo.stage_shift], 1);
        }
        __syncthreads();
        for (int b = threadIdx.x; b < nbk; b += kL2LThreads) {
            const int c = s_cnt[b];
            s_base[b] = c ? atomicAdd(&fo.stage_cursor[(size_t)b * kUnpermCursorStride], c) : 0;
            s_cnt[b] = 0;
        }
        __syncthreads();
    }
    constexpr int kB = 4;
    for (int base = threadIdx.x; base < total; base += kB * kL2LThreads) {
        int jj[kB], lyy[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int idx = base + u * kL2LThreads;
            int ly = 0;
            while (ly + 1 < side && rp[ly + 1] <= idx) ++ly;
            lyy[u] = ly;
            jj[u] = idx < total ? rb[ly] + idx - rp[ly] : -1;
        }
        int key[kB], o[kB];
        double2 sj[kB];
        double2 nv[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int j = jj[u] < 0 ? 0 : jj[u];
            key[u] = fo.keys[j];
            sj[u] = *reinterpret_cast<const double2*>(&fo.src[j]);  // x, y of the record
            nv[u] = fo.near[j];
            o[u] = fo.perm[j];
        }
        // the kB particles' Horner chains advance together (ILP)
        const double2* lp[kB];
        double wx[kB], wy[kB];
        double2 ff[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int ly = lyy[u], gy = cy * side + ly;
            const int lx = jj[u] < 0 ? 0 : (key[u] & (m - 1)) - cx * side;
            const double ccx = cell_center(fo.xmin, cx * side + lx, r);
            const double ccy = cell_center(fo.ymin, gy, r);
            lp[u] = leafs + (size_t)(ly * side + lx) * P;
            wx[u] = (sj[u].x - ccx) * inv_r;
            wy[u] = (sj[u].y - ccy) * inv_r;
        }
        eval_local_multi<kB>(lp, P, wx, wy, ff);
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            if (jj[u] < 0) continue;
            const double2 f = ff[u];
            // f_to_velocity: u = Im f / 2pi, v = Re f / 2pi; then far + near
            const double uo = f.y * kInv2Pi + nv[u].x, vo = f.x * kInv2Pi + nv[u].y;
            if (STAGED) {
                const int b = o[u] >> fo.stage_shift;
                const int pos = s_base[b] + atomicAdd(&s_cnt[b], 1);
                VCHECK(pos >= 0 && pos < (1 << fo.stage_shift) &&
                       (((int64_t)b << fo.stage_shift) + pos) < fo.n_total);
                UnpermRec rcd;
                rcd.u = uo;
                rcd.v = vo;
                rcd.dest = o[u];
                rcd.pad[0] = rcd.pad[1] = rcd.pad[2] = 0;
                fo.stage[((size_t)b << fo.stage_shift) + pos] = rcd;
            } else if (fo.v) {
                fo.u[o[u]] = uo;
                fo.v[o[u]] = vo;
            } else {
                reinterpret_cast<double2*>(fo.u)[o[u]] = make_double2(uo, vo);
            }
        }
    }
#ifdef VFMM_L2L_TRACE
    __syncthreads();
    mark();
    if (threadIdx.x == 0 && (blockIdx.x % 97) == 0)
        printf("l2l cta %d: wait %.2f prefetch %.2f anc %.2f subtree %.2f l2p %.2f us\n", blockIdx.x,
               (tr[1] - tr[0]) * 1e-3, (tr[2] - tr[1]) * 1e-3, (tr[3] - tr[2]) * 1e-3, (tr[4] - tr[3]) * 1e-3,
               (tr[5] - tr[4]) * 1e-3);
#endif
}

size_t sub_smem(int depth, int P) {
    return sizeof(double2) * ((size_t)(((1 << (2 * (depth + 1))) - 1) / 3) * P + 4 * P) +
           sizeof(double) * (P + 1);
}

int sub_depth(int P) { return sub_smem(3, P) <= 48 * 1024 ? 3 : 2; }

}  // namespace

void launch_m2m(const Layout& L, const Tables* T, double2* mult, Rows rows, cudaStream_t s) {
    const int d0 = sub_depth(L.P);
    for (int lf = L.levels; lf > 2;) {
        const int d = lf - 2 < d0 ? lf - 2 : d0;
        const int lt = lf - d;
        const size_t off_lf = L.level_cell_off[lf] * L.P;
        launch_k(k_m2m_subtree, (unsigned)(1ll << (2 * lt)), kSubThreads, sub_smem(d, L.P), s, 
            mult, lf, d, L.P, off_lf, T, L.levels, rows);
        note_launches(1);
        lf = lt;
    }
}

int l2l_split_level(int levels, int P) {
    // CTAs at level l-2 (depth-2 subtrees): enough CTAs for the fused L2P +
    // combine at small l, short ancestor chains at large l.  Measured (graph
    // replay, depth 1 / 2 / 3): config 2 0.788 / 0.759 / 0.767 ms, config 1
    // 0.216 / 0.221 / 0.243 ms, config 3 14.66 / 14.22 / 14.22 ms.
    // VFMM_L2L_DEPTH overrides (tuning).
    static const int depth_env = [] {
        const char* e = getenv("VFMM_L2L_DEPTH");
        return e ? atoi(e) : 2;
    }();
    int d = depth_env > 0 ? depth_env : 2;
    if (d > sub_depth(P)) d = sub_depth(P);
    return levels - d > 2 ? levels - d : 2;
}

void launch_l2l(const Layout& L, const Tables* T, double2* loc, double2* leaf_loc,
                const double2* anc, Rows rows, const FusedOut& fo, cudaStream_t s) {
    if (L.levels == 2) {
        launch_leaf_locals_copy(L, loc, leaf_loc, s);
        return;
    }
    const int ls = l2l_split_level(L.levels, L.P);
    const size_t shm = sub_smem(L.levels - ls, L.P) + sizeof(double2) * (2 * L.P + 1) +
                       sizeof(double) * (L.P + 1) + sizeof(double2) * (ls - 2) * L.P;
    const unsigned ctas = (unsigned)(1ll << (2 * ls));
    if (fo.stage && ctas >= 148 * 4) {  // both instances: each returns at once off its path
        launch_k(k_l2l_fused<128, true>, ctas, 128, shm, s, loc, leaf_loc, anc, ls, L.levels, L.P, T, rows, fo);
        note_launches(1);
    }
    if (ctas >= 148 * 4)
        launch_k(k_l2l_fused<128>, ctas, 128, shm, s, loc, leaf_loc, anc, ls, L.levels, L.P, T, rows, fo);
    else
        launch_k(k_l2l_fused<256>, ctas, 256, shm, s, loc, leaf_loc, anc, ls, L.levels, L.P, T, rows, fo);
    note_launches(1);
}

// ---------------------------------------------------------------------------
// Staged un-permute.  With a random input order the fused L2P's output stores
// are 16-byte writes to random sectors of an array far larger than L2: every
// store becomes a DRAM read-modify-write (config 3: the downward pass read
// 2.1 GB and wrote 1.3 GB for 0.27 GB of velocities).  Staged: the fused L2P
// appends (u, v, destination) records -- 32 bytes, a full sector each -- to the
// bucket of its destination's high bits (every bucket of a permutation fills
// exactly, so bucket b owns records [b 2^shift, (b + 1) 2^shift)), and this
// kernel walks the records in bucket order: the CTAs resident at any time
// write into a window of a few buckets (tens of MB), where the two halves of an
// output sector meet in L2 before it is written back once.
#ifndef VFMM_UNPERM_PER
#define VFMM_UNPERM_PER 2  // records per thread: 1 / 2 / 4 -> config 3 downward 0.998 / 1.041 / 1.093 ms, idle launch (coherent order) +0.09 / +0.055 / +0.04 ms
#endif
constexpr int kUnpermPer = VFMM_UNPERM_PER;
constexpr int kUnpermChunk = 256 * kUnpermPer;
__global__ void __launch_bounds__(256)
    k_unpermute(const UnpermRec* __restrict__ stage, int64_t n, double* __restrict__ u,
                double* __restrict__ v, const Counters* __restrict__ ctr) {
    pdl_enter();
    if (ctr->sort_fallback != kSortPathLsdProbe) return;
    // a CTA owns kUnpermChunk consecutive records (one bucket's, mostly), its
    // threads kUnpermPer of them each, all loads in flight together; CTAs run in
    // index order, so the records being written at any time are a sliding window
    // of a few buckets
    const int64_t base = (int64_t)blockIdx.x * kUnpermChunk + threadIdx.x;
    UnpermRec r[kUnpermPer];
#pragma unroll
    for (int k = 0; k < kUnpermPer; ++k) {
        const int64_t t = base + k * 256;
        if (t < n) r[k] = stage[t];
    }
#pragma unroll
    for (int k = 0; k < kUnpermPer; ++k) {
        const int64_t t = base + k * 256;
        if (t >= n) break;
        if (v) {
            u[r[k].dest] = r[k].u;
            v[r[k].dest] = r[k].v;
        } else {
            reinterpret_cast<double2*>(u)[r[k].dest] = make_double2(r[k].u, r[k].v);
        }
    }
}

__global__ void k_unpermute_zero(int* __restrict__ cursor, int nbuckets, const Counters* __restrict__ ctr) {
    pdl_enter();
    if (ctr->sort_fallback != kSortPathLsdProbe) return;
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nbuckets; b += gridDim.x * blockDim.x)
        cursor[(size_t)b * kUnpermCursorStride] = 0;
}

bool l2l_stageable(const Layout& L) {  // the fused L2L's large-grid instance has the staged variant
    return L.levels > 2 && (1ll << (2 * l2l_split_level(L.levels, L.P))) >= 148 * 4;
}

int unperm_shift(int64_t n) {
    int shift = 16;
    while ((n >> shift) >= 1024) ++shift;
    return shift;
}

void launch_unpermute_prepare(const Layout& L, const FusedOut& fo, cudaStream_t s) {
    const int nb = (int)((L.n + ((int64_t)1 << fo.stage_shift) - 1) >> fo.stage_shift);
    launch_k(k_unpermute_zero, 4, 256, 0, s, fo.stage_cursor, nb, fo.ctr);
    note_launches(1);
}

void launch_unpermute(const Layout& L, const FusedOut& fo, cudaStream_t s) {
    launch_k(k_unpermute, (unsigned)((L.n + kUnpermChunk - 1) / kUnpermChunk), 256, 0, s,
             (const UnpermRec*)fo.stage, L.n, fo.u, fo.v, fo.ctr);
    note_launches(1);
}

}  // namespace vfmm
