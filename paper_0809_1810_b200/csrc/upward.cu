// Upward pass (north-star item 2): P2M at the leaves, then M2M up to level 2.
//
// Replaces engine.upward_pass (engine.py:114-147), expansions.p2m
// (expansions.py:88-101) and expansions.multipole_shift_matrix
// (expansions.py:119-130).  Coefficients are stored in the scaled form
// M_n = a_n / (r^{n+1} n!) (vfmm_internal.cuh), which makes the shift
// operator level independent:  P_m = 2^{-(m+1)} sum_{k<=m} M_k E_q[m-k],
// in the planar coefficient layout (coef_base / coef_stride).
#include <cstdlib>
#include <type_traits>

#include "vfmm_internal.cuh"

namespace vfmm {

namespace {

constexpr int kP2MWarps = 2;

// One warp per leaf.  Lanes own particles; the powers Gamma w^k of a round of
// 32 particles are transposed through shared memory so that lane k sums
// coefficient k over the particles in sorted order (np.add.reduceat order).
__global__ void __launch_bounds__(kP2MWarps * 32)
    k_p2m(const Src* __restrict__ src, const int* __restrict__ ls, int levels, int P, double xmin,
          double ymin, double side, const Tables* __restrict__ T, Rows rows,
          double2* __restrict__ mult) {
    pdl_enter();
    __shared__ double2 buf[kP2MWarps][32][33];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m = 1 << levels;
    // the grid covers the leaves of the owned row strip only (all leaves on one GPU)
    const int64_t leaf = (int64_t)rows.lo * m + (int64_t)blockIdx.x * kP2MWarps + warp;
    if (leaf >= (int64_t)rows.hi * m) return;
    const int lo = ls[leaf], hi = ls[leaf + 1];
    const int ix = (int)(leaf % m), iy = (int)(leaf / m);
    double2* out = mult + coef_base(levels, ix, iy);
    const int64_t cs = coef_stride(levels);
    // empty leaves carry zero
    if (lo == hi) {
        for (int k = lane; k < P; k += 32) out[k * cs] = make_double2(0.0, 0.0);
        return;
    }
    const double r = side / m;  // Tree.cell_side (quadtree.py:140-141)
    const double cx = cell_center(xmin, ix, r), cy = cell_center(ymin, iy, r);
    const double inv_r = 1.0 / r;
    const int ngroups = (P + 31) >> 5;  // <= 2 for P <= 61
    double2 acc0 = make_double2(0.0, 0.0), acc1 = make_double2(0.0, 0.0);
    for (int base = lo; base < hi; base += 32) {
        const int j = base + lane;
        double2 term = make_double2(0.0, 0.0), w = make_double2(0.0, 0.0);
        if (j < hi) {
            const Src s = src[j];
            term.x = s.g;
            w.x = (s.x - cx) * inv_r;
            w.y = (s.y - cy) * inv_r;
        }
        for (int g = 0; g < ngroups; ++g) {
            const int kmax = min(32, P - g * 32);
            for (int kk = 0; kk < kmax; ++kk) {
                buf[warp][kk][lane] = term;
                const double tx = term.x * w.x - term.y * w.y;
                const double ty = term.x * w.y + term.y * w.x;
                term.x = tx;
                term.y = ty;
            }
            __syncwarp();
            if (lane < kmax) {
                double2 a = g == 0 ? acc0 : acc1;
                const int cnt = min(32, hi - base);
                for (int q = 0; q < cnt; ++q) {
                    const double2 t = buf[warp][lane][q];
                    a.x += t.x;
                    a.y += t.y;
                }
                if (g == 0) acc0 = a; else acc1 = a;
            }
            __syncwarp();
        }
    }
    for (int g = 0; g < ngroups; ++g) {
        const int k = g * 32 + lane;
        if (k < P) {
            const double2 a = g == 0 ? acc0 : acc1;
            const double sc = T->invfact[k] * inv_r;
            out[k * cs] = make_double2(a.x * sc, a.y * sc);
        }
    }
}


// Sub-warp P2M for P <= PMAX (the common orders): G lanes per leaf, each lane
// sums Gamma w^k over a strided subset of the leaf's particles into PMAX
// register accumulators, then one butterfly over the G lanes combines them.
// No shared-memory transpose, so the kernel is bound by its (small) FP64
// work and the source reads rather than by shared-memory wavefronts.
template <int G, int PMAX>
__global__ void __launch_bounds__(128)
    k_p2m_grp(const Src* __restrict__ src, const int* __restrict__ ls, int levels, int P,
              double xmin, double ymin, double side, const Tables* __restrict__ T, Rows rows,
              double2* __restrict__ mult) {
    pdl_enter();
    const int sub = threadIdx.x & (G - 1);
    const int m = 1 << levels;
    // the grid covers the leaves of the owned row strip only (all leaves on one GPU)
    const int64_t leaf = (int64_t)rows.lo * m + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
    const bool valid = leaf < (int64_t)rows.hi * m;  // whole groups are (in)valid together
    if (!valid) return;
    const int lo = ls[leaf], hi = ls[leaf + 1];
    const int ix = (int)(leaf % m), iy = (int)(leaf / m);
    double2* out = mult + coef_base(levels, ix, iy);
    const int64_t cs = coef_stride(levels);
    const bool live = lo < hi;  // uniform per group
    double ax[PMAX], ay[PMAX];
#pragma unroll
    for (int k = 0; k < PMAX; ++k) ax[k] = ay[k] = 0.0;
    const double r = side / m;  // Tree.cell_side (quadtree.py:140-141)
    const double cx = cell_center(xmin, ix, r), cy = cell_center(ymin, iy, r);
    const double inv_r = 1.0 / r;
    if (live) {
        // the next particle's record is loaded while the current one's powers
        // are summed (the load had stalled every iteration: long_scoreboard);
        // the power loop leaves at k = P (uniform) instead of predicating
        // PMAX - P idle steps
        int j = lo + sub;
        double3 nxt = make_double3(0.0, 0.0, 0.0);
        if (j < hi) nxt = make_double3(src[j].x, src[j].y, src[j].g);
        for (; j < hi; j += G) {
            const double3 sj = nxt;
            if (j + G < hi) nxt = make_double3(src[j + G].x, src[j + G].y, src[j + G].g);
            const double wx = (sj.x - cx) * inv_r, wy = (sj.y - cy) * inv_r;
            double tx = sj.z, ty = 0.0;
#pragma unroll
            for (int k = 0; k < PMAX; ++k) {
                if (k >= P) break;
                ax[k] += tx;
                ay[k] += ty;
                const double nx = tx * wx - ty * wy;
                ty = tx * wy + ty * wx;
                tx = nx;
            }
        }
    }
    // the group's lanes are consecutive and G-aligned: xor butterflies stay inside it
#pragma unroll
    for (int k = 0; k < PMAX; ++k) {
        if (k < P) {
#pragma unroll
            for (int o = G / 2; o > 0; o >>= 1) {
                ax[k] += __shfl_xor_sync(0xffffffffu, ax[k], o, G);
                ay[k] += __shfl_xor_sync(0xffffffffu, ay[k], o, G);
            }
            if ((k & (G - 1)) == sub) {
                const double sc = T->invfact[k] * inv_r;
                out[k * cs] = make_double2(ax[k] * sc, ay[k] * sc);
            }
        }
    }
}

}  // namespace

int coef_chunk(int P) {
    int best = 8, waste = 1 << 30;
    for (int tn = 8; tn >= 4; --tn) {
        const int w = (P + tn - 1) / tn * tn - P;
        if (w < waste) { waste = w; best = tn; }
    }
    return best;
}

void launch_p2m(const Layout& L, const Src* src, const int* leaf_starts, double xmin, double ymin,
                double side, double2* mult_leaf, const Tables* T, Rows rows, cudaStream_t s) {
    // strip-local: only the leaves of the owned rows are visited (sharded runs
    // leave the other leaves' multipoles alone; the exchange fills the halo)
    const int64_t nl = (int64_t)(rows.hi - rows.lo) << L.levels;
    if (nl <= 0) return;
    // sub-warp groups while leaves are small enough for 8 lanes to sweep them
    // (mean occupancy <= 256); the warp-per-leaf transpose kernel otherwise
    const bool grp = L.P <= 32 && L.n <= 256 * (int64_t)L.nleaves;
    if (grp) {
        // Lanes per leaf: the fewest of 2 / 4 / 8 that still give ~12 warps
        // per SM (fewer lanes: longer per-lane sums, a shorter butterfly).
        // Measured upward pass (P2M + M2M), G = 8 / 4 / 2: config 2 54.2 /
        // 52.3 / 55.6 us, config 3 0.562 / 0.507 / 0.486 ms, config 1 21.5 /
        // 25.6 / 33.8 us.  VFMM_P2M_G=2|4|8|16 overrides (A/B).
        static const int genv = getenv("VFMM_P2M_G") ? atoi(getenv("VFMM_P2M_G")) : 0;
        int gsel = genv;
        if (gsel <= 0) {
            const int64_t want = 148 * 384;  // threads
            gsel = nl * 2 >= want ? 2 : (nl * 4 >= want ? 4 : 8);
        }
        auto go = [&](auto g_tag) {
            constexpr int G = decltype(g_tag)::value;
            const unsigned blocks = (unsigned)((nl * G + 127) / 128);
            if (L.P <= 16)
                launch_k(k_p2m_grp<G, 16>, blocks, 128, 0, s, src, leaf_starts, L.levels, L.P, xmin,
                         ymin, side, T, rows, mult_leaf);
            else if (L.P <= 24)
                launch_k(k_p2m_grp<G, 24>, blocks, 128, 0, s, src, leaf_starts, L.levels, L.P, xmin,
                         ymin, side, T, rows, mult_leaf);
            else
                launch_k(k_p2m_grp<G, 32>, blocks, 128, 0, s, src, leaf_starts, L.levels, L.P, xmin,
                         ymin, side, T, rows, mult_leaf);
        };
        if (gsel == 2)
            go(std::integral_constant<int, 2>{});
        else if (gsel == 4)
            go(std::integral_constant<int, 4>{});
        else if (gsel == 16)
            go(std::integral_constant<int, 16>{});
        else
            go(std::integral_constant<int, 8>{});
    } else {
        launch_k(k_p2m, (unsigned)((nl + kP2MWarps - 1) / kP2MWarps), kP2MWarps * 32, 0, s, 
            src, leaf_starts, L.levels, L.P, xmin, ymin, side, T, rows, mult_leaf);
    }
    note_launches(1);
}

}  // namespace vfmm
