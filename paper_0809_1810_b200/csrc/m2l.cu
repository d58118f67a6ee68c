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
#include <cstdlib>

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
    switch (coef_chunk(L.P)) {
        case 4: launch_tn<4>(L, T, mult, counts, loc, anc, ctr, rows, s); break;
        case 5: launch_tn<5>(L, T, mult, counts, loc, anc, ctr, rows, s); break;
        case 6: launch_tn<6>(L, T, mult, counts, loc, anc, ctr, rows, s); break;
        case 7: launch_tn<7>(L, T, mult, counts, loc, anc, ctr, rows, s); break;
        default: launch_tn<8>(L, T, mult, counts, loc, anc, ctr, rows, s); break;
    }
}

}  // namespace vfmm
