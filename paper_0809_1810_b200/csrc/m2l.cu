// M2L over every cell's interaction list, all levels in ONE launch
// (north-star item 3).
//
// Replaces engine.translate_pass (engine.py:150-187), engine._il_offsets
// (engine.py:77-89), engine._parity_grid (engine.py:92-98) and
// expansions.m2l_matrix (expansions.py:133-145).
//
// In the scaled representation the translation of offset o = (dx, dy) is a
// Hankel product  Lh_m = sum_n H_o[m+n] M_n,  H_o[q] = q! tau^{-(q+1)},
// tau = -(dx + i dy), identical at every level.  A block owns one
// (level, parity class, m-chunk); its 27 offsets' H rows sit in shared memory
// and every lane (one destination cell) reads them as warp-wide broadcasts.
// Each thread keeps TN complex accumulators (outputs m0..m0+TN-1) in
// registers across all 27 offsets, so a loaded multipole coefficient feeds
// TN complex FMAs.  Per destination, offsets apply in row-major source order
// (the accumulation order of engine.py:166-185); empty sources are skipped
// when a whole warp's sources are empty and multiply as exact zeros otherwise.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "vfmm_internal.cuh"

namespace vfmm {

namespace {


// Offsets of the interaction list of parity class (px, py) in row-major
// order (engine._il_offsets, engine.py:77-89), as (dx, dy) pairs.
__device__ __forceinline__ void il_offset(int px, int py, int o, int& dx, int& dy) {
    int idx = 0;
    for (int yy = -2 - py; yy < 4 - py; ++yy)
        for (int xx = -2 - px; xx < 4 - px; ++xx) {
            const int ax = xx < 0 ? -xx : xx, ay = yy < 0 ? -yy : yy;
            if ((ax > ay ? ax : ay) >= 2) {
                if (idx == o) { dx = xx; dy = yy; }
                ++idx;
            }
        }
}

// Block = 32 destinations j of one parity plane x one chunk of TN outputs, as
// kGroups warps: warp g accumulates the offsets [27g/G, 27(g+1)/G) of the parity
// class (row-major order, engine.py:166-185) and the partial sums are added
// in group order through shared memory (deterministic).  With the planar
// layout the source of offset (dx, dy) for consecutive destinations is a run
// of consecutive cells of one source plane, so each multipole coefficient
// load is coalesced; the Hankel rows are block-uniform smem broadcasts.
// G offset-unit groups (warps) per CTA, one CTA = 32 destinations: G = 3 (8
// CTAs of 3 warps per SM; 5 of the 15 units per warp) by default; G = 9 (3
// CTAs of 9 warps) for tiny grids (< 600 CTAs), where more, shorter warps
// fill the SMs.  Measured (median t_m2l, 15-unit kernel): config 1 0.0225
// (G 3) / 0.0143 ms (G 9); config 2 0.0706-0.0717 (G 3) / 0.0727 (G 5) /
// 0.0778 ms (G 9); config 3 1.20 ms (G 3).
constexpr int kDestPerBlock = 32;

// Symmetric offsets share their Hankel row up to conjugation and signs
// (tau_o = -(dx + i dy)):
//   -o        : tau -> -tau        H[q] -> (-1)^(q+1) H[q]        (kind 1)
//   (dx, -dy) : tau -> conj(tau)   H[q] -> conj(H[q])             (kind 2)
//   (-dx, dy) : tau -> -conj(tau)  H[q] -> (-1)^(q+1) conj(H[q])  (kind 3)
// so the translations of a destination from a source M1 at o and a source M2
// at the partner offset collapse into ONE product with the row h = H_o:
//   kind 1:   Lh_m += sum_n h[m+n] X_n,  X = M1 - M2 (m+n even), M1 + M2 (odd)
//   kind 2/3: Lh_m += sum_n (Re h[m+n] X_n + i Im h[m+n] Y_n), S = M1 + M2,
//             D = M1 - M2; kind 2: X = S, Y = D; kind 3: (X, Y) = (D, S) for
//             m+n even, (S, D) for m+n odd
// (H M1 + conj(H) B = Re H (M1 + B) + i Im H (M1 - B)).  Each costs 4 real
// FMA per (m, n), like one plain translation.  Of the 27 offsets of a parity
// class the 16 of the 5x5 ring pair as +-o (kind 1), the outer column and row
// give two mirror pairs each (kinds 2 and 3) and 3 stay single: 15 products
// per destination instead of 27.  Units in row-major order of their first
// offset; o2 = -1 for a single offset.
constexpr int kUnits = 15;
struct UnitTab {
    int8_t o1[4][kUnits], o2[4][kUnits], kind[4][kUnits];
    int count[4];
};
constexpr UnitTab make_units() {
    UnitTab t{};
    for (int par = 0; par < 4; ++par) {
        const int px = par & 1, py = par >> 1;
        int dxs[27] = {}, dys[27] = {};
        int idx = 0;
        for (int yy = -2 - py; yy < 4 - py; ++yy)
            for (int xx = -2 - px; xx < 4 - px; ++xx) {
                const int ax = xx < 0 ? -xx : xx, ay = yy < 0 ? -yy : yy;
                if ((ax > ay ? ax : ay) >= 2) {
                    dxs[idx] = xx;
                    dys[idx] = yy;
                    ++idx;
                }
            }
        bool used[27] = {};
        int nu = 0;
        for (int o = 0; o < 27; ++o) {
            if (used[o]) continue;
            used[o] = true;
            int partner = -1, kind = 0;
            for (int k = 0; k < 3 && partner < 0; ++k) {
                if ((k == 1 && dys[o] == 0) || (k == 2 && dxs[o] == 0)) continue;
                const int wx = k == 1 ? dxs[o] : -dxs[o], wy = k == 2 ? dys[o] : -dys[o];
                for (int q = 0; q < 27; ++q)
                    if (!used[q] && dxs[q] == wx && dys[q] == wy) {
                        partner = q;
                        kind = k + 1;
                    }
            }
            if (partner >= 0) used[partner] = true;
            if (nu < kUnits) {
                t.o1[par][nu] = (int8_t)o;
                t.o2[par][nu] = (int8_t)partner;
                t.kind[par][nu] = (int8_t)kind;
            }
            ++nu;
        }
        t.count[par] = nu;
    }
    return t;
}
constexpr UnitTab kUnitTab = make_units();
static_assert(kUnitTab.count[0] == kUnits && kUnitTab.count[1] == kUnits &&
                  kUnitTab.count[2] == kUnits && kUnitTab.count[3] == kUnits,
              "15 units per parity class");
__constant__ UnitTab c_units = kUnitTab;

// Multipole source for destinations whose source is empty / outside the grid:
// a zero coefficient read with stride 0 (no per-coefficient select).
__device__ const double2 g_zero_coef = {0.0, 0.0};

// One paired unit (see the unit table) for outputs m0 .. m0+TN-1; MP = parity
// of m0, so the per-(t, n) choices of X / Y are compile-time.
template <int TN, int KIND, int MP>
__device__ __forceinline__ void m2l_pair_step(double2 a1, double2 a2, const double2* h, int np,
                                              double (&ax)[TN], double (&ay)[TN]) {
    const double sr = a1.x + a2.x, si = a1.y + a2.y;
    const double dr = a1.x - a2.x, di = a1.y - a2.y;
#pragma unroll
    for (int t = 0; t < TN; ++t) {
        const bool odd = ((MP + t + np) & 1) != 0;  // parity of m + n
        const bool swap = KIND != 2 && odd;          // kinds 1, 3: S where m + n is odd
        const double xr = swap ? sr : dr, xi = swap ? si : di;
        const double2 hh = h[t];
        if (KIND == 1) {  // h * X, X = D (m+n even) / S (odd)
            ax[t] = fma(hh.x, xr, fma(-hh.y, xi, ax[t]));
            ay[t] = fma(hh.x, xi, fma(hh.y, xr, ay[t]));
        } else {  // Re h * X + i Im h * Y
            const bool xs = KIND == 2 || odd;  // X = S (kind 2, or kind 3 at odd m+n)
            const double Xr = xs ? sr : dr, Xi = xs ? si : di;
            const double Yr = xs ? dr : sr, Yi = xs ? di : si;
            ax[t] = fma(hh.x, Xr, fma(-hh.y, Yi, ax[t]));
            ay[t] = fma(hh.x, Xi, fma(hh.y, Yr, ay[t]));
        }
    }
}
template <int TN, int KIND, int MP>
__device__ __forceinline__ void m2l_pair(const double2* M1, int64_t st1, const double2* M2,
                                         int64_t st2, const double2* h, int P, double (&ax)[TN],
                                         double (&ay)[TN]) {
    int n = 0;
#pragma unroll 1
    for (; n + 1 < P; n += 2) {
        const double2 a1 = M1[0], a2 = M2[0], b1 = M1[st1], b2 = M2[st2];
        m2l_pair_step<TN, KIND, MP>(a1, a2, h + n, 0, ax, ay);
        m2l_pair_step<TN, KIND, MP>(b1, b2, h + n + 1, 1, ax, ay);
        M1 += 2 * st1;
        M2 += 2 * st2;
    }
    if (n < P) {
        if (n & 1)
            m2l_pair_step<TN, KIND, MP>(*M1, *M2, h + n, 1, ax, ay);
        else
            m2l_pair_step<TN, KIND, MP>(*M1, *M2, h + n, 0, ax, ay);
    }
}

template <int TN, int kGroups>
#ifndef VFMM_M2L_MB3
#define VFMM_M2L_MB3 8
#endif
#ifndef VFMM_M2L_MB9
#define VFMM_M2L_MB9 3
#endif
__global__ void __launch_bounds__(kDestPerBlock * kGroups, kGroups == 3 ? VFMM_M2L_MB3 : VFMM_M2L_MB9)
    k_m2l(const double2* __restrict__ mult, const int* __restrict__ counts, double2* __restrict__ loc,
          double2* __restrict__ anc, int anc_end, int levels, int P, int nchunks,
          const Tables* __restrict__ T, unsigned long long* __restrict__ m2l_count, Rows rows) {
    pdl_enter();
    extern __shared__ double2 sH[];  // [27][TN + P - 1], then [kGroups - 1][TN][32] partials
    // ---- decode (level, parity, chunk, block-in-class) from blockIdx.x ----
    int64_t b = blockIdx.x;
    int level = 2;
    size_t cell_off = 0;  // cells before this level in mult/loc (level 2 first)
    size_t cnt_off = 5;   // cells before this level in counts (levels 0, 1 first)
    int64_t bpc = 0;      // blocks per (parity, chunk) at this level
    for (;;) {
        const int64_t dests = 1ll << (2 * (level - 1));
        bpc = (dests + kDestPerBlock - 1) / kDestPerBlock;
        const int64_t nb = bpc * 4 * nchunks;
        if (b < nb || level == levels) break;
        b -= nb;
        cell_off += (size_t)1 << (2 * level);
        cnt_off += (size_t)1 << (2 * level);
        ++level;
    }
    const int chunk = (int)(b / (4 * bpc));
    const int parity = (int)((b / bpc) % 4);
    const int64_t blk = b % bpc;
    const int px = parity & 1, py = parity >> 1;
    const int m0 = chunk * TN;
    const int HL = TN + P - 1;
    const int group = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // sharded runs: CTAs whose 32 destinations all lie outside the owned row
    // strip exit before staging the tables
    {
        const int half0 = 1 << (level - 1);
        const int64_t psz0 = (int64_t)half0 * half0;
        const int64_t j0 = blk * kDestPerBlock + lane;
        const int iy0 = 2 * (j0 < psz0 ? (int)(j0 / half0) : 0) + py;
        const bool act0 = j0 < psz0 && rows_touch(rows, iy0, levels - level);
        if (!__syncthreads_or(act0)) return;
    }
    // ---- stage the 27 offsets and their H rows of this parity class ----
    __shared__ int2 soff[27];
    if (threadIdx.x < 27) {
        int dxo = 0, dyo = 0;
        il_offset(px, py, threadIdx.x, dxo, dyo);
        soff[threadIdx.x] = make_int2(dxo, dyo);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 27 * HL; i += blockDim.x) {
        const int o = i / HL, q = i % HL;
        const int2 d = soff[o];
        sH[i] = T->H[(d.y + 3) * 7 + (d.x + 3)][m0 + q];
    }
    __syncthreads();

    const int mk = 1 << level, half = mk >> 1;
    const int64_t psz = (int64_t)half * half;  // cells per plane
    const int64_t j = blk * kDestPerBlock + lane;
    const int jx = j < psz ? (int)(j % half) : 0;
    const int jy = j < psz ? (int)(j / half) : 0;
    const int ix = 2 * jx + px, iy = 2 * jy + py;
    // destinations whose leaf rows touch the owned strip; a destination is
    // counted by the strip that owns its first leaf row (sharded runs)
    const int shift = levels - level;
    const bool active = j < psz && rows_touch(rows, iy, shift);
    const bool counts_here = active && (iy << shift) >= rows.lo;
    const double2* M = mult + cell_off * P;
    const int* cnt = counts + cnt_off;
    const int64_t cstride = 4 * psz;

    double ax[TN], ay[TN];
#pragma unroll
    for (int t = 0; t < TN; ++t) ax[t] = ay[t] = 0.0;
    int ntrans = 0;
    // this warp's units: [kUnits g / G, kUnits (g + 1) / G)
    const int u_end = kUnits * (group + 1) / kGroups;
    for (int u = kUnits * group / kGroups; u < u_end; ++u) {
        const int o1 = c_units.o1[parity][u], o2 = c_units.o2[parity][u];
        const int kind = c_units.kind[parity][u];
        const int2 d = soff[o1];
        const int sx = ix + d.x, sy = iy + d.y;
        const bool inr = active && sx >= 0 && sx < mk && sy >= 0 && sy < mk;
        const bool live = inr && cnt[(int64_t)sy * mk + sx] > 0;
        ntrans += (live && counts_here) ? 1 : 0;
        // source plane / index (floor division of the shifted coordinates)
        const double2* Ms = live ? M + (((sy & 1) << 1) | (sx & 1)) * psz +
                                       (int64_t)(sy >> 1) * half + (sx >> 1)
                                 : &g_zero_coef;
        const int64_t step = live ? cstride : 0;
        const double2* h = sH + o1 * HL;
        if (o2 < 0) {
            if (!__any_sync(0xffffffffu, live)) continue;
#pragma unroll 3
            for (int n = 0; n < P; ++n) {
                const double2 a = *Ms;
                Ms += step;
#pragma unroll
                for (int t = 0; t < TN; ++t) {
                    const double2 hh = h[t + n];
                    ax[t] = fma(hh.x, a.x, fma(-hh.y, a.y, ax[t]));
                    ay[t] = fma(hh.x, a.y, fma(hh.y, a.x, ay[t]));
                }
            }
            continue;
        }
        // the partner source (offset -o1, or its y / x mirror)
        const int2 d2 = soff[o2];
        const int tx = ix + d2.x, ty = iy + d2.y;
        const bool inr2 = active && tx >= 0 && tx < mk && ty >= 0 && ty < mk;
        const bool live2 = inr2 && cnt[(int64_t)ty * mk + tx] > 0;
        ntrans += (live2 && counts_here) ? 1 : 0;
        if (!__any_sync(0xffffffffu, live || live2)) continue;
        const double2* Ms2 = live2 ? M + (((ty & 1) << 1) | (tx & 1)) * psz +
                                         (int64_t)(ty >> 1) * half + (tx >> 1)
                                   : &g_zero_coef;
        const int64_t step2 = live2 ? cstride : 0;
        const bool mo = (m0 & 1) != 0;
        if (kind == 1) {
            if (mo) m2l_pair<TN, 1, 1>(Ms, step, Ms2, step2, h, P, ax, ay);
            else m2l_pair<TN, 1, 0>(Ms, step, Ms2, step2, h, P, ax, ay);
        } else if (kind == 2) {
            m2l_pair<TN, 2, 0>(Ms, step, Ms2, step2, h, P, ax, ay);
        } else {
            if (mo) m2l_pair<TN, 3, 1>(Ms, step, Ms2, step2, h, P, ax, ay);
            else m2l_pair<TN, 3, 0>(Ms, step, Ms2, step2, h, P, ax, ay);
        }
    }
    // ---- combine the group partials in group order ----
    double2* part = sH + 27 * HL;
    if (group > 0) {
#pragma unroll
        for (int t = 0; t < TN; ++t) part[((group - 1) * TN + t) * 32 + lane] = make_double2(ax[t], ay[t]);
    }
    __syncthreads();
    if (group == 0 && active) {
        double2* out = loc + cell_off * P + parity * psz + j;
#pragma unroll
        for (int t = 0; t < TN; ++t) {
            double sx = ax[t], sy = ay[t];
            for (int g = 1; g < kGroups; ++g) {
                const double2 p = part[((g - 1) * TN + t) * 32 + lane];
                sx += p.x;
                sy += p.y;
            }
            if (m0 + t < P) {
                out[(m0 + t) * cstride] = make_double2(sx, sy);
                // M2L parts of the fused L2L's shared ancestors (read-only copy)
                if (level < anc_end) anc[(out - loc) + (m0 + t) * cstride] = make_double2(sx, sy);
            }
        }
    }
    if (chunk == 0) {
        // m2l_count counts (destination, nonempty source) pairs at every level
        // including empty destinations (engine.py:173-180)
        for (int s = 16; s > 0; s >>= 1) ntrans += __shfl_xor_sync(0xffffffffu, ntrans, s);
        if (lane == 0 && ntrans) atomicAdd(m2l_count, (unsigned long long)ntrans);
    }
}


// ============================================================================
// Tiled M2L (P <= kTileMaxP): a CTA owns a tile of 8 x 4 destination PARENTS
// of one level -- 128 destination cells, one warp per parity class -- and one
// chunk of TN output coefficients.  Every source its 128 destinations need
// lies in the children of the tile's parents grown by one parent on each side
// (dx in [-2-px, 3-px] -> source parent jx-1 .. jx+1), i.e. a window of
// 10 x 6 parents = 4 planes x 6 rows x 10 cells, which is ONE box of the
// planar layout [P][4 planes][half][half]: a single TMA (cp.async.bulk.tensor,
// 4-D, out-of-grid cells zero-filled by the copy engine) stages all P
// coefficients of the window in shared memory, and every source coefficient
// is then read from shared memory by all the destinations that use it (27
// per cell) instead of from L2 once per (destination, offset, chunk).
// L2 -> SM traffic per CTA: 240 cells x P x 16 B for 128 destinations (1.9x
// the destination data) plus the Hankel rows of the chunk.  Small levels
// (half < 10 parents per side) fill the window with bounds-checked loads.
// The arithmetic per destination is the 15-unit symmetric-offset schedule of
// k_m2l (same units, same order), with the Hankel values of two consecutive
// n held in registers (TN + 1 loads per two n instead of 2 TN).
constexpr int kTPX = 8, kTPY = 4;                 // destination parents per tile
constexpr int kWX = kTPX + 2, kWY = kTPY + 2;     // window parents (one-parent halo)
constexpr int kWinCells = 4 * kWY * kWX;          // window cells per coefficient (240)
constexpr int kTileMaxP = 26;                     // window <= 100 KB of shared memory

struct M2LMaps {
    CUtensorMap map[VFMM_LEVELS_CAP + 1];  // per level (levels with half >= kWX)
};

// (dx, dy) of offset o of parity class par, engine._il_offsets order
struct OffTab {
    int8_t dx[4][27], dy[4][27];
};
constexpr OffTab make_offtab() {
    OffTab t{};
    for (int par = 0; par < 4; ++par) {
        const int px = par & 1, py = par >> 1;
        int idx = 0;
        for (int yy = -2 - py; yy < 4 - py; ++yy)
            for (int xx = -2 - px; xx < 4 - px; ++xx) {
                const int ax = xx < 0 ? -xx : xx, ay = yy < 0 ? -yy : yy;
                if ((ax > ay ? ax : ay) >= 2) {
                    t.dx[par][idx] = (int8_t)xx;
                    t.dy[par][idx] = (int8_t)yy;
                    ++idx;
                }
            }
    }
    return t;
}
__constant__ OffTab c_off = make_offtab();

// Units of the tiled kernel: as the unit table above, but offsets whose
// four-member orbit {o, -o, o', -o'} (o' = (dx, -dy)) lies in the class share
// ONE product (kind 4): with s = (-1)^(m+n+1), A = M(o) + s M(-o) and
// B = M(o') + s M(-o'), H_o A + conj(H_o) B = Re H_o (A + B) + i Im H_o (A - B)
// -- four real FMA per (m, n) for four translations, after 16 adds per n
// shared by the chunk's outputs.  The 5 x 5 ring gives three orbits and two
// axis pairs, the outer row / column two mirror pairs each, three offsets stay
// single: 12 products per destination (15 with pairs only).
#ifndef VFMM_M2L_QUADS
#define VFMM_M2L_QUADS 1
#endif
#ifndef VFMM_M2L_QUADS_GMAX
#define VFMM_M2L_QUADS_GMAX 3
#endif
constexpr int kQUnits = 12;
struct QuadTab {
    int8_t o[4][kQUnits][4], kind[4][kQUnits];
    int count[4];
};
constexpr QuadTab make_quads() {
    QuadTab t{};
    for (int par = 0; par < 4; ++par) {
        const int px = par & 1, py = par >> 1;
        int dxs[27] = {}, dys[27] = {};
        int idx = 0;
        for (int yy = -2 - py; yy < 4 - py; ++yy)
            for (int xx = -2 - px; xx < 4 - px; ++xx) {
                const int ax = xx < 0 ? -xx : xx, ay = yy < 0 ? -yy : yy;
                if ((ax > ay ? ax : ay) >= 2) {
                    dxs[idx] = xx;
                    dys[idx] = yy;
                    ++idx;
                }
            }
        auto find = [&](int wx, int wy, const bool* used) {
            for (int q = 0; q < 27; ++q)
                if (!used[q] && dxs[q] == wx && dys[q] == wy) return q;
            return -1;
        };
        bool used[27] = {};
        int nu = 0;
        for (int o = 0; o < 27; ++o) {
            if (used[o]) continue;
            used[o] = true;
            int mem[4] = {o, -1, -1, -1};
            int kind = 0;
            if (dxs[o] != 0 && dys[o] != 0) {
                const int a = find(-dxs[o], -dys[o], used), b = find(dxs[o], -dys[o], used),
                          c = find(-dxs[o], dys[o], used);
                if (a >= 0 && b >= 0 && c >= 0) {
                    mem[1] = a;
                    mem[2] = b;
                    mem[3] = c;
                    used[a] = used[b] = used[c] = true;
                    kind = 4;
                }
            }
            for (int k = 0; k < 3 && kind == 0; ++k) {
                if ((k == 1 && dys[o] == 0) || (k == 2 && dxs[o] == 0)) continue;
                const int wx = k == 1 ? dxs[o] : -dxs[o], wy = k == 2 ? dys[o] : -dys[o];
                const int q = find(wx, wy, used);
                if (q >= 0) {
                    mem[1] = q;
                    used[q] = true;
                    kind = k + 1;
                }
            }
            if (nu < kQUnits) {
                for (int j = 0; j < 4; ++j) t.o[par][nu][j] = (int8_t)mem[j];
                t.kind[par][nu] = (int8_t)kind;
            }
            ++nu;
        }
        t.count[par] = nu;
        // Balanced order: (orbit, pair, pair, single) x 3, so every third of
        // the units costs the same (per coefficient 16 adds + 4 TN FMA for an
        // orbit, 4 adds + 4 TN for a pair, 4 TN for a single) and three unit
        // groups (sparse grids) stay balanced.
        if (nu == kQUnits) {
            int8_t oo[kQUnits][4] = {}, kk[kQUnits] = {};
            int qi = 0, pi = 0, si = 0, w = 0;
            int q[kQUnits] = {}, pr[kQUnits] = {}, sg[kQUnits] = {};
            for (int u = 0; u < kQUnits; ++u) {
                if (t.kind[par][u] == 4) q[qi++] = u;
                else if (t.kind[par][u] == 0) sg[si++] = u;
                else pr[pi++] = u;
            }
            int a = 0, b = 0, c = 0;
            const bool ok = qi == 3 && pi == 6 && si == 3;
            for (int g = 0; ok && g < 3; ++g) {
                const int us[4] = {q[a++], pr[b++], pr[b++], sg[c++]};
                for (int j = 0; j < 4; ++j, ++w) {
                    for (int m = 0; m < 4; ++m) oo[w][m] = t.o[par][us[j]][m];
                    kk[w] = t.kind[par][us[j]];
                }
            }
            if (ok)
                for (int u = 0; u < kQUnits; ++u) {
                    for (int m = 0; m < 4; ++m) t.o[par][u][m] = oo[u][m];
                    t.kind[par][u] = kk[u];
                }
        }
    }
    return t;
}
constexpr QuadTab kQuadTab = make_quads();
static_assert(kQuadTab.count[0] == kQUnits && kQuadTab.count[1] == kQUnits &&
                  kQuadTab.count[2] == kQUnits && kQuadTab.count[3] == kQUnits,
              "12 units per parity class");
__constant__ QuadTab c_quads = kQuadTab;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}

// Accumulators: the real and imaginary parts of every output are split in
// two partial sums (acc[0][t] += hr xr, acc[1][t] -= hi xi; acc[2][t] += hr xi,
// acc[3][t] += hi xr), so the four FMAs of a complex product are independent
// and one coefficient step has no dependent DFMA pair (ncu: "wait" was the top
// stall of the nested form); the halves are added once at the end.
template <int TN>
struct TileAcc {
    double a[4][TN];
};

// one complex product h * X (X = (xr, xi)) into output t
template <int TN>
__device__ __forceinline__ void cmac(TileAcc<TN>& A, int t, double2 h, double xr, double xi) {
    A.a[0][t] = fma(h.x, xr, A.a[0][t]);
    A.a[1][t] = fma(-h.y, xi, A.a[1][t]);
    A.a[2][t] = fma(h.x, xi, A.a[2][t]);
    A.a[3][t] = fma(h.y, xr, A.a[3][t]);
}
// Re h * X + i Im h * Y into output t
template <int TN>
__device__ __forceinline__ void rmac(TileAcc<TN>& A, int t, double2 h, double Xr, double Xi, double Yr,
                                     double Yi) {
    A.a[0][t] = fma(h.x, Xr, A.a[0][t]);
    A.a[1][t] = fma(-h.y, Yi, A.a[1][t]);
    A.a[2][t] = fma(h.x, Xi, A.a[2][t]);
    A.a[3][t] = fma(h.y, Yr, A.a[3][t]);
}

template <int TN, int KIND, int MP>
__device__ __forceinline__ void tile_pair_step(double2 a1, double2 a2, const double2* hv, int np,
                                               TileAcc<TN>& A) {
    const double sr = a1.x + a2.x, si = a1.y + a2.y;
    const double dr = a1.x - a2.x, di = a1.y - a2.y;
#pragma unroll
    for (int t = 0; t < TN; ++t) {
        const bool odd = ((MP + t + np) & 1) != 0;  // parity of m + n
        if (KIND == 1) {  // h * X, X = D (m+n even) / S (odd)
            cmac(A, t, hv[t], odd ? sr : dr, odd ? si : di);
        } else {  // Re h * X + i Im h * Y; X = S for kind 2, or kind 3 at odd m+n
            const bool xs = KIND == 2 || odd;
            rmac(A, t, hv[t], xs ? sr : dr, xs ? si : di, xs ? dr : sr, xs ? di : si);
        }
    }
}

template <int TN>
__device__ __forceinline__ void tile_plain(const double2* __restrict__ s1, const double2* __restrict__ h,
                                           int P, TileAcc<TN>& A) {
    int n = 0;
#pragma unroll 1
    for (; n + 1 < P; n += 2) {
        double2 hv[TN + 1];
#pragma unroll
        for (int t = 0; t <= TN; ++t) hv[t] = h[n + t];
        const double2 a = s1[n * kWinCells], b = s1[(n + 1) * kWinCells];
#pragma unroll
        for (int t = 0; t < TN; ++t) cmac(A, t, hv[t], a.x, a.y);
#pragma unroll
        for (int t = 0; t < TN; ++t) cmac(A, t, hv[t + 1], b.x, b.y);
    }
    if (n < P) {
        const double2 a = s1[n * kWinCells];
#pragma unroll
        for (int t = 0; t < TN; ++t) cmac(A, t, h[n + t], a.x, a.y);
    }
}

template <int TN, int KIND, int MP>
__device__ __forceinline__ void tile_pair(const double2* __restrict__ s1, const double2* __restrict__ s2,
                                          const double2* __restrict__ h, int P, TileAcc<TN>& A) {
    int n = 0;
#pragma unroll 1
    for (; n + 1 < P; n += 2) {
        double2 hv[TN + 1];
#pragma unroll
        for (int t = 0; t <= TN; ++t) hv[t] = h[n + t];
        const double2 a1 = s1[n * kWinCells], a2 = s2[n * kWinCells];
        const double2 b1 = s1[(n + 1) * kWinCells], b2 = s2[(n + 1) * kWinCells];
        tile_pair_step<TN, KIND, MP>(a1, a2, hv, 0, A);
        tile_pair_step<TN, KIND, MP>(b1, b2, hv + 1, 1, A);
    }
    if (n < P) {  // n even
        double2 hv[TN];
#pragma unroll
        for (int t = 0; t < TN; ++t) hv[t] = h[n + t];
        tile_pair_step<TN, KIND, MP>(s1[n * kWinCells], s2[n * kWinCells], hv, 0, A);
    }
}

// One four-member orbit unit (kind 4) for outputs m0 .. m0+TN-1 (MP =
// parity of m0): X = A + B, Y = A - B with A = M1 + s M2, B = M3 + s M4,
// s = (-1)^(m+n+1) (m + n odd: s = +1).
template <int TN, int MP>
__device__ __forceinline__ void tile_quad_step(double2 a1, double2 a2, double2 a3, double2 a4,
                                               const double2* hv, int np, TileAcc<TN>& A) {
    const double apr = a1.x + a2.x, api = a1.y + a2.y, amr = a1.x - a2.x, ami = a1.y - a2.y;
    const double bpr = a3.x + a4.x, bpi = a3.y + a4.y, bmr = a3.x - a4.x, bmi = a3.y - a4.y;
    const double xor_ = apr + bpr, xoi = api + bpi, yor = apr - bpr, yoi = api - bpi;  // m+n odd
    const double xer = amr + bmr, xei = ami + bmi, yer = amr - bmr, yei = ami - bmi;   // m+n even
#pragma unroll
    for (int t = 0; t < TN; ++t) {
        const bool odd = ((MP + t + np) & 1) != 0;
        rmac(A, t, hv[t], odd ? xor_ : xer, odd ? xoi : xei, odd ? yor : yer, odd ? yoi : yei);
    }
}
template <int TN, int MP>
__device__ __forceinline__ void tile_quad(const double2* __restrict__ s1, const double2* __restrict__ s2,
                                          const double2* __restrict__ s3, const double2* __restrict__ s4,
                                          const double2* __restrict__ h, int P, TileAcc<TN>& A) {
    int n = 0;
#pragma unroll 1
    for (; n + 1 < P; n += 2) {
        double2 hv[TN + 1];
#pragma unroll
        for (int t = 0; t <= TN; ++t) hv[t] = h[n + t];
        tile_quad_step<TN, MP>(s1[n * kWinCells], s2[n * kWinCells], s3[n * kWinCells], s4[n * kWinCells],
                               hv, 0, A);
        tile_quad_step<TN, MP>(s1[(n + 1) * kWinCells], s2[(n + 1) * kWinCells], s3[(n + 1) * kWinCells],
                               s4[(n + 1) * kWinCells], hv + 1, 1, A);
    }
    if (n < P) {  // n even
        double2 hv[TN];
#pragma unroll
        for (int t = 0; t < TN; ++t) hv[t] = h[n + t];
        tile_quad_step<TN, MP>(s1[n * kWinCells], s2[n * kWinCells], s3[n * kWinCells], s4[n * kWinCells],
                               hv, 0, A);
    }
}

// Warps: 4 parity classes x CW chunks x G unit groups.  G > 1 (small or
// strip-restricted grids) splits the 15 units of a destination over G warps,
// whose partial sums are added in group order through shared memory
// (deterministic); CW > 1 (large grids) shares the window between chunks.
template <int TN, int CW, int G>
__global__ void __launch_bounds__(128 * CW * G, CW * G <= 2 ? 2 : 1)
    k_m2l_tile(const __grid_constant__ M2LMaps maps, const double2* __restrict__ mult,
               const int* __restrict__ counts, double2* __restrict__ loc, double2* __restrict__ anc,
               int anc_end, int levels, int P, int nchunks, const Tables* __restrict__ T,
               unsigned long long* __restrict__ m2l_count, Rows rows) {
    pdl_enter();
    extern __shared__ __align__(1024) unsigned char m2l_smem[];
    double2* win = reinterpret_cast<double2*>(m2l_smem);  // [P][4][kWY][kWX]
    double2* sH = win + (size_t)P * kWinCells;            // [49][HL]
    __shared__ int scnt[kWinCells];                       // occupancy of the window cells
    __shared__ __align__(8) unsigned long long bar;
    // ---- decode (level, tile, chunk) ----
    int64_t b = blockIdx.x;
    int level = 2;
    size_t cell_off = 0, cnt_off = 5;
    int half = 2, tiles_x = 1;
    for (;;) {
        half = 1 << (level - 1);
        tiles_x = (half + kTPX - 1) / kTPX;
        const int tiles_y = (half + kTPY - 1) / kTPY;
        const int64_t nb = (int64_t)tiles_x * tiles_y * ((nchunks + CW - 1) / CW);
        if (b < nb || level == levels) break;
        b -= nb;
        cell_off += (size_t)1 << (2 * level);
        cnt_off += (size_t)1 << (2 * level);
        ++level;
    }
    const int ngroups = (nchunks + CW - 1) / CW;  // chunk groups of CW chunks (one per warp quad)
    const int warp_id = threadIdx.x >> 5;
    const int chunk = (int)(b % ngroups) * CW + (warp_id >> 2) % CW;
    const int group = (warp_id >> 2) / CW;  // unit group
    const int64_t tile = b / ngroups;
    const int jx0 = (int)(tile % tiles_x) * kTPX, jy0 = (int)(tile / tiles_x) * kTPY;
    const int parity = (threadIdx.x >> 5) & 3, lane = threadIdx.x & 31;
    const int px = parity & 1, py = parity >> 1;
    const int jx = jx0 + (lane & 7), jy = jy0 + (lane >> 3);
    const int ix = 2 * jx + px, iy = 2 * jy + py;
    const int shift = levels - level;
    const bool active = chunk < nchunks && jx < half && jy < half && rows_touch(rows, iy, shift);
    if (!__syncthreads_or(active)) return;  // sharded runs: tile outside the strip

    const int mk = 1 << level;
    const int64_t psz = (int64_t)half * half, cstride = 4 * psz;
    const double2* M = mult + cell_off * P;
    const bool tma = half >= kWX;
    if (tma && threadIdx.x == 0) {
        const unsigned ba = smem_u32(&bar);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(ba));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const unsigned bytes = (unsigned)(P * kWinCells * sizeof(double2));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ba), "r"(bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(win)),
            "l"(reinterpret_cast<unsigned long long>(&maps.map[level])), "r"(2 * (jx0 - 1)),
            "r"(jy0 - 1), "r"(0), "r"(0), "r"(ba)
            : "memory");
    }
    if (!tma) {  // small levels: bounds-checked cooperative fill
        for (int i = threadIdx.x; i < P * kWinCells; i += blockDim.x) {
            const int n = i / kWinCells, r = i % kWinCells;
            const int plane = r / (kWX * kWY), rr = r % (kWX * kWY);
            const int gy = jy0 - 1 + rr / kWX, gx = jx0 - 1 + rr % kWX;
            win[i] = (gx >= 0 && gx < half && gy >= 0 && gy < half)
                         ? M[n * cstride + plane * psz + (int64_t)gy * half + gx]
                         : make_double2(0.0, 0.0);
        }
    }
    // occupancy of the window cells (the reference skips empty sources and
    // counts the (destination, nonempty source) pairs, engine.py:173-180)
    for (int r = threadIdx.x; r < kWinCells; r += blockDim.x) {
        const int plane = r / (kWX * kWY), rr = r % (kWX * kWY);
        const int sx = 2 * (jx0 - 1 + rr % kWX) + (plane & 1);
        const int sy = 2 * (jy0 - 1 + rr / kWX) + (plane >> 1);
        scnt[r] = (sx >= 0 && sx < mk && sy >= 0 && sy < mk) ? counts[cnt_off + (int64_t)sy * mk + sx] : 0;
    }
    // Hankel rows of this chunk group for the 7 x 7 offset grid: entries
    // mg .. mg + CW TN + P - 1 (one pad for the two-coefficient loop)
    const int mg = (chunk / CW) * CW * TN, m0 = chunk * TN;
    const int HL = CW * TN + P;
    for (int i = threadIdx.x; i < kOffsets * HL; i += blockDim.x) {
        const int o = i / HL, q = i % HL;
        sH[i] = T->H[o][mg + q];
    }
    __syncthreads();
    if (tma) {
        const unsigned ba = smem_u32(&bar);
        asm volatile(
            "{\n .reg .pred p;\n WAIT_%=:\n"
            " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
            " @!p bra WAIT_%=;\n}" ::"r"(ba)
            : "memory");
    }

    // destination's own parent sits at window (lane & 7) + 1, (lane >> 3) + 1
    const int counts_here = active && (iy << shift) >= rows.lo;
    TileAcc<TN> A;
#pragma unroll
    for (int t = 0; t < TN; ++t) A.a[0][t] = A.a[1][t] = A.a[2][t] = A.a[3][t] = 0.0;
    int ntrans = 0;
    const bool mo = (m0 & 1) != 0;
    auto src_of = [&](int o, bool& live) {
        const int sx = ix + c_off.dx[parity][o], sy = iy + c_off.dy[parity][o];
        const int r = (((sy & 1) << 1) | (sx & 1)) * (kWX * kWY) + ((sy >> 1) - jy0 + 1) * kWX +
                      ((sx >> 1) - jx0 + 1);
        VCHECK(!active || (r >= 0 && r < kWinCells));
        live = active && scnt[r] > 0;
        return r;
    };
    // orbit units (config 2, G = 2: 0.0608 -> 0.0567 ms; config 3: 0.918 ->
    // 0.812 ms); their balanced order keeps three unit groups (sparse grids)
    // even; VFMM_M2L_QUADS=0 / _GMAX restrict them (A/B)
    if constexpr (VFMM_M2L_QUADS && G <= VFMM_M2L_QUADS_GMAX) {
    const int u_end = kQUnits * (group + 1) / G;
#pragma unroll 1
    for (int u = kQUnits * group / G; u < u_end; ++u) {
        const int o1 = c_quads.o[parity][u][0], o2 = c_quads.o[parity][u][1];
        const int kind = c_quads.kind[parity][u];
        bool live1, live2 = false, live3 = false, live4 = false;
        const int r1 = src_of(o1, live1);
        const int r2 = o2 >= 0 ? src_of(o2, live2) : r1;
        int r3 = r1, r4 = r1;
        if (kind == 4) {
            r3 = src_of(c_quads.o[parity][u][2], live3);
            r4 = src_of(c_quads.o[parity][u][3], live4);
        }
        ntrans += (counts_here && live1 ? 1 : 0) + (counts_here && live2 ? 1 : 0) +
                  (counts_here && live3 ? 1 : 0) + (counts_here && live4 ? 1 : 0);
        if (!__any_sync(0xffffffffu, live1 || live2 || live3 || live4)) continue;
        // empty sources hold zero multipoles: they multiply as exact zeros
        const double2* h =
            sH + ((c_off.dy[parity][o1] + 3) * 7 + (c_off.dx[parity][o1] + 3)) * HL + (m0 - mg);
        const double2* s1 = win + r1;
        VCHECK(m0 - mg + TN + P <= HL + TN);
        VJITTER();
        if (o2 < 0) {
            tile_plain<TN>(s1, h, P, A);
            continue;
        }
        const double2* s2 = win + r2;
        if (kind == 4) {
            if (mo) tile_quad<TN, 1>(s1, s2, win + r3, win + r4, h, P, A);
            else tile_quad<TN, 0>(s1, s2, win + r3, win + r4, h, P, A);
        } else if (kind == 1) {
            if (mo) tile_pair<TN, 1, 1>(s1, s2, h, P, A);
            else tile_pair<TN, 1, 0>(s1, s2, h, P, A);
        } else if (kind == 2) {
            tile_pair<TN, 2, 0>(s1, s2, h, P, A);
        } else {
            if (mo) tile_pair<TN, 3, 1>(s1, s2, h, P, A);
            else tile_pair<TN, 3, 0>(s1, s2, h, P, A);
        }
    }
    } else {
    const int u_end = kUnits * (group + 1) / G;
#pragma unroll 1
    for (int u = kUnits * group / G; u < u_end; ++u) {
        const int o1 = c_units.o1[parity][u], o2 = c_units.o2[parity][u];
        const int kind = c_units.kind[parity][u];
        bool live1, live2 = false;
        const int r1 = src_of(o1, live1);
        const int r2 = o2 >= 0 ? src_of(o2, live2) : r1;
        ntrans += (counts_here && live1 ? 1 : 0) + (counts_here && live2 ? 1 : 0);
        if (!__any_sync(0xffffffffu, live1 || live2)) continue;
        // empty sources hold zero multipoles: they multiply as exact zeros
        const double2* h =
            sH + ((c_off.dy[parity][o1] + 3) * 7 + (c_off.dx[parity][o1] + 3)) * HL + (m0 - mg);
        const double2* s1 = win + r1;
        VCHECK(m0 - mg + TN + P <= HL + TN);
        VJITTER();
        if (o2 < 0) {
            tile_plain<TN>(s1, h, P, A);
            continue;
        }
        const double2* s2 = win + r2;
        if (kind == 1) {
            if (mo) tile_pair<TN, 1, 1>(s1, s2, h, P, A);
            else tile_pair<TN, 1, 0>(s1, s2, h, P, A);
        } else if (kind == 2) {
            tile_pair<TN, 2, 0>(s1, s2, h, P, A);
        } else {
            if (mo) tile_pair<TN, 3, 1>(s1, s2, h, P, A);
            else tile_pair<TN, 3, 0>(s1, s2, h, P, A);
        }
    }
    }
    double2 res[TN];
#pragma unroll
    for (int t = 0; t < TN; ++t) res[t] = make_double2(A.a[0][t] + A.a[1][t], A.a[2][t] + A.a[3][t]);
    if (G > 1) {  // groups 1.. hand their partials to group 0 through the (now free) window
        __syncthreads();
        double2* part = win;  // [G - 1][CW][4][TN][32]
        const int slot = ((warp_id >> 2) % CW) * 4 + parity;
        if (group > 0) {
#pragma unroll
            for (int t = 0; t < TN; ++t) part[(((group - 1) * CW * 4 + slot) * TN + t) * 32 + lane] = res[t];
        }
        __syncthreads();
        if (group == 0) {
            for (int gg = 1; gg < G; ++gg) {
#pragma unroll
                for (int t = 0; t < TN; ++t) {
                    const double2 q = part[(((gg - 1) * CW * 4 + slot) * TN + t) * 32 + lane];
                    res[t].x += q.x;
                    res[t].y += q.y;
                }
            }
        }
    }
    if (active && group == 0) {
        double2* out = loc + cell_off * P + parity * psz + (int64_t)jy * half + jx;
#pragma unroll
        for (int t = 0; t < TN; ++t) {
            if (m0 + t < P) {
                out[(m0 + t) * cstride] = res[t];
                if (level < anc_end) anc[(out - loc) + (m0 + t) * cstride] = res[t];
            }
        }
    }
    if (chunk == 0) {  // warp-uniform
        for (int sft = 16; sft > 0; sft >>= 1) ntrans += __shfl_xor_sync(0xffffffffu, ntrans, sft);
        if (lane == 0 && ntrans) atomicAdd(m2l_count, (unsigned long long)ntrans);
    }
}

// Tensor maps of the multipole levels (driver entry point; no -lcuda), cached
// per (multipole base, levels, P): encoding is host work, reused by every call
// on the same workspace.
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    return fn;
}

bool m2l_maps(const Layout& L, const double2* mult, M2LMaps* out) {
    struct Entry {
        const double2* mult;
        int levels, P;
        M2LMaps maps;
    };
    static std::mutex mu;
    static std::vector<Entry> cache;
    std::lock_guard<std::mutex> lk(mu);
    for (const auto& e : cache)
        if (e.mult == mult && e.levels == L.levels && e.P == L.P) {
            *out = e.maps;
            return true;
        }
    auto enc = encode_fn();
    if (!enc) return false;
    Entry e{mult, L.levels, L.P, {}};
    std::memset(&e.maps, 0, sizeof(e.maps));
    for (int k = 2; k <= L.levels; ++k) {
        const uint64_t half = 1ull << (k - 1);
        if (half < (uint64_t)kWX) continue;
        const cuuint64_t dims[4] = {2 * half, half, 4, (cuuint64_t)L.P};
        const cuuint64_t strides[3] = {half * 16, half * half * 16, 4 * half * half * 16};
        const cuuint32_t box[4] = {2 * kWX, kWY, 4, (cuuint32_t)L.P};
        const cuuint32_t estr[4] = {1, 1, 1, 1};
        void* base = (void*)(mult + L.level_cell_off[k] * L.P);
        if (enc(&e.maps.map[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, base, dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    }
    if (cache.size() >= 64) cache.erase(cache.begin());
    cache.push_back(e);
    *out = e.maps;
    return true;
}

template <int TN, int CW, int G>
void launch_tile_cw(const Layout& L, const M2LMaps& maps, const Tables* T, const double2* mult,
                    const int* counts, double2* loc, double2* anc, Counters* ctr, Rows rows,
                    int64_t tiles, int nchunks, cudaStream_t s) {
    const int64_t blocks = tiles * ((nchunks + CW - 1) / CW);
    size_t smem = (size_t)L.P * kWinCells * sizeof(double2) +
                  (size_t)kOffsets * (CW * TN + L.P) * sizeof(double2);
    const size_t parts = (size_t)(G - 1) * CW * 4 * TN * 32 * sizeof(double2);  // reuses the window
    if (parts > smem) smem = parts;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_m2l_tile<TN, CW, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_set = true;
    }
    launch_k(k_m2l_tile<TN, CW, G>, (unsigned)blocks, 128 * CW * G, smem, s, maps, mult, counts, loc, anc,
             l2l_split_level(L.levels, L.P), L.levels, L.P, nchunks, T, &ctr->m2l_count, rows);
    note_launches(1);
}

// Tile kernel when the grid fills the GPU (>= 2 CTAs per SM); the direct-load
// kernel (k_m2l, many small CTAs) below that.  All chunks of a tile share one
// CTA (CW = nchunks <= 3, one window per 4 CW warps) once the grid is >= 8
// waves of single-chunk CTAs, one chunk per CTA otherwise (balance: config 2
// has 516 single-chunk CTAs).  VFMM_M2L_CW=1|3 overrides (tuning).
template <int TN>
bool launch_tile_tn(const Layout& L, const Tables* T, const double2* mult, const int* counts,
                    double2* loc, double2* anc, Counters* ctr, Rows rows, cudaStream_t s) {
    const int nchunks = (L.P + TN - 1) / TN;
    int64_t tiles = 0, active = 0;  // active: tiles touching the owned strip (sharded runs)
    for (int level = 2; level <= L.levels; ++level) {
        const int half = 1 << (level - 1);
        const int ty = (half + kTPY - 1) / kTPY, tx = (half + kTPX - 1) / kTPX;
        tiles += (int64_t)tx * ty;
        for (int t = 0; t < ty; ++t) {  // tile t covers cell rows [8 t, 8 t + 8) of the level
            const int s = L.levels - level;
            if (((8 * t) << s) < rows.hi && ((8 * t + 8) << s) > rows.lo) active += tx;
        }
    }
    if (active * nchunks < 32) return false;
    M2LMaps maps;
    if (!m2l_maps(L, mult, &maps)) return false;
    static const int cw_env = getenv("VFMM_M2L_CW") ? atoi(getenv("VFMM_M2L_CW")) : 0;
    static const int g_env = getenv("VFMM_M2L_TG") ? atoi(getenv("VFMM_M2L_TG")) : 0;
    const int64_t work = active * nchunks;  // single-chunk CTAs that do work
    // Measured (median t_m2l): config 2 G = 1 / 2 / 3: 0.0686 / 0.0604 / 0.0666 ms;
    // config 3 G = 2: 0.912 ms, all chunks per CTA (CW = 3): 0.953, G = 1: 0.993.
    // Two unit groups per tile (8 warps, 2 CTAs / SM = 16 warps / SM at <= 128
    // registers) by default; three for sparse grids (a rank's strip).
    int cw = 1;
    int g = work < 2 * 148 ? 3 : 2;
    if (cw_env >= 1 && cw_env <= 3) cw = cw_env;
    if (g_env >= 1 && g_env <= 3) g = g_env;
    if (g > 1) cw = 1;
    if (cw == 1 && g == 1)
        launch_tile_cw<TN, 1, 1>(L, maps, T, mult, counts, loc, anc, ctr, rows, tiles, nchunks, s);
    else if (g == 2)
        launch_tile_cw<TN, 1, 2>(L, maps, T, mult, counts, loc, anc, ctr, rows, tiles, nchunks, s);
    else if (g == 3)
        launch_tile_cw<TN, 1, 3>(L, maps, T, mult, counts, loc, anc, ctr, rows, tiles, nchunks, s);
    else if (cw == 2)
        launch_tile_cw<TN, 2, 1>(L, maps, T, mult, counts, loc, anc, ctr, rows, tiles, nchunks, s);
    else
        launch_tile_cw<TN, 3, 1>(L, maps, T, mult, counts, loc, anc, ctr, rows, tiles, nchunks, s);
    return true;
}

template <int TN>
void launch_tn(const Layout& L, const Tables* T, const double2* mult, const int* counts,
               double2* loc, double2* anc, Counters* ctr, Rows rows, cudaStream_t s) {
    const int nchunks = (L.P + TN - 1) / TN;
    int64_t blocks = 0;
    for (int level = 2; level <= L.levels; ++level) {
        const int64_t dests = 1ll << (2 * (level - 1));
        blocks += (dests + kDestPerBlock - 1) / kDestPerBlock * 4 * nchunks;
    }
    auto shm_of = [&](int groups) {
        return (size_t)27 * (TN + L.P - 1) * sizeof(double2) +
               (size_t)(groups - 1) * TN * 32 * sizeof(double2);
    };
    const int anc_end = l2l_split_level(L.levels, L.P);
    // offset groups (warps) per CTA by grid size, see the kernel comment;
    // VFMM_M2L_G = 3 / 9 overrides (tuning)
    static const int g_env = getenv("VFMM_M2L_G") ? atoi(getenv("VFMM_M2L_G")) : 0;
    int g = blocks < 600 ? 9 : 3;
    if (g_env == 3 || g_env == 9) g = g_env;
    if (g == 9 && shm_of(9) > 48 * 1024) g = 3;
    if (g == 9)
        launch_k(k_m2l<TN, 9>, (unsigned)blocks, kDestPerBlock * 9, shm_of(9), s,
            mult, counts, loc, anc, anc_end, L.levels, L.P, nchunks, T, &ctr->m2l_count, rows);
    else
        launch_k(k_m2l<TN, 3>, (unsigned)blocks, kDestPerBlock * 3, shm_of(3), s, 
            mult, counts, loc, anc, anc_end, L.levels, L.P, nchunks, T, &ctr->m2l_count, rows);
    note_launches(1);
}

}  // namespace

void launch_m2l(const Layout& L, const Tables* T, const double2* mult, const int* counts,
                double2* loc, double2* anc, Counters* ctr, Rows rows, cudaStream_t s) {
    // the shared-memory window kernel (TMA) for P <= 26; VFMM_M2L_TILE=0 keeps
    // the direct-load kernel (A/B measurement)
    static const bool tile_on = !(getenv("VFMM_M2L_TILE") && getenv("VFMM_M2L_TILE")[0] == '0');
    if (tile_on && L.P <= kTileMaxP) {
        bool ok = false;
        switch (coef_chunk(L.P)) {
            case 4: ok = launch_tile_tn<4>(L, T, mult, counts, loc, anc, ctr, rows, s); break;
            case 5: ok = launch_tile_tn<5>(L, T, mult, counts, loc, anc, ctr, rows, s); break;
            case 6: ok = launch_tile_tn<6>(L, T, mult, counts, loc, anc, ctr, rows, s); break;
            case 7: ok = launch_tile_tn<7>(L, T, mult, counts, loc, anc, ctr, rows, s); break;
            default: ok = launch_tile_tn<8>(L, T, mult, counts, loc, anc, ctr, rows, s); break;
        }
        if (ok) return;
    }
    switch (coef_chunk(L.P)) {
        case 4: launch_tn<4>(L, T, mult, counts, loc, anc, ctr, rows, s); break;
        case 5: launch_tn<5>(L, T, mult, counts, loc, anc, ctr, rows, s); break;
        case 6: launch_tn<6>(L, T, mult, counts, loc, anc, ctr, rows, s); break;
        case 7: launch_tn<7>(L, T, mult, counts, loc, anc, ctr, rows, s); break;
        default: launch_tn<8>(L, T, mult, counts, loc, anc, ctr, rows, s); break;
    }
}

}  // namespace vfmm
