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
#include "vfmm_internal.cuh"

namespace vfmm {

namespace {

constexpr int kSubThreads = 256;

__device__ __forceinline__ int sub_off(int s) { return ((1 << (2 * s)) - 1) / 3; }  // cells before sub-level s

// Upward: CTA per cell at level lt = lf - depth; reads the 4^depth cells at
// level lf (global, planar), writes levels lf-1 .. lt.
__global__ void __launch_bounds__(kSubThreads)
    k_m2m_subtree(double2* __restrict__ mult, int lf, int depth, int P, size_t off_lf,
                  const Tables* __restrict__ T) {
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
        for (int i = threadIdx.x; i < ncell * P; i += blockDim.x) {
            const int c = i / P, k = i % P;
            const int gx = cx * side + (c % side), gy = cy * side + (c / side);
            dst[i] = src[coef_base(lf, gx, gy) + k * cs];
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
        for (int i = threadIdx.x; i < side * side * P; i += blockDim.x) {
            const int c = i / P, mm = i % P;
            const int px = c % side, py = c / side;
            double ax = 0.0, ay = 0.0;
            for (int q = 0; q < 4; ++q) {
                const int chx = 2 * px + (q & 1), chy = 2 * py + (q >> 1);
                const double2* M = child + (size_t)(chy * 2 * side + chx) * P;
                for (int k = 0; k <= mm; ++k) {
                    const double2 a = M[k], e = sE[q * P + mm - k];
                    ax = fma(a.x, e.x, fma(-a.y, e.y, ax));
                    ay = fma(a.x, e.y, fma(a.y, e.x, ay));
                }
            }
            const double2 r = make_double2(ax * s2[mm + 1], ay * s2[mm + 1]);
            par[i] = r;
            gout[coef_base(lvl, cx * side + px, cy * side + py) + mm * cs] = r;
        }
        __syncthreads();
    }
}

// Downward: CTA per cell at level lt (complete local in `loc`), completes the
// locals of levels lt+1 .. lt+depth of its subtree.  The leaf level (when
// reached) is written cell-major to leaf_loc, other levels in place (planar).
__global__ void __launch_bounds__(kSubThreads)
    k_l2l_subtree(double2* __restrict__ loc, double2* __restrict__ leaf_loc, int lt, int depth,
                  int levels, int P, size_t off_lt, const Tables* __restrict__ T, Rows rows) {
    extern __shared__ double2 sm[];
    double2* sF = sm + (size_t)sub_off(depth + 1) * P;  // [4][P]
    double* s2 = reinterpret_cast<double*>(sF + 4 * P);  // [P]
    const int mt = 1 << lt;
    const int cx = blockIdx.x % mt, cy = blockIdx.x / mt;
    if (!rows_touch(rows, cy, levels - lt)) return;  // subtree outside the owned strip
    for (int i = threadIdx.x; i < 4 * P; i += blockDim.x) sF[i] = T->F[i / P][i % P];
    for (int i = threadIdx.x; i < P; i += blockDim.x) s2[i] = T->pow2neg[i];
    {
        const double2* g = loc + off_lt;
        const int64_t cs = coef_stride(lt);
        for (int k = threadIdx.x; k < P; k += blockDim.x) sm[k] = g[coef_base(lt, cx, cy) + k * cs];
    }
    __syncthreads();
    size_t off_level = off_lt;
    for (int s = 1; s <= depth; ++s) {
        const int lvl = lt + s;
        off_level += (size_t)(1ll << (2 * (lvl - 1))) * P;
        const int side = 1 << s;
        const double2* par = sm + (size_t)sub_off(s - 1) * P;
        double2* cur = sm + (size_t)sub_off(s) * P;
        double2* g = loc + off_level;
        const int64_t cs = coef_stride(lvl);
        const bool leaf = lvl == levels;
        const int m = 1 << lvl;
        for (int i = threadIdx.x; i < side * side * P; i += blockDim.x) {
            const int c = i / P, nn = i % P;
            const int lx = c % side, ly = c / side;
            const int q = 2 * (ly & 1) + (lx & 1);
            const double2* Lp = par + (size_t)((ly >> 1) * (side >> 1) + (lx >> 1)) * P;
            const double2* Fq = sF + q * P;
            double ax = 0.0, ay = 0.0;
            for (int mm = nn; mm < P; ++mm) {
                const double2 a = Lp[mm];
                const double axs = a.x * s2[mm], ays = a.y * s2[mm];
                const double2 f = Fq[mm - nn];
                ax = fma(axs, f.x, fma(-ays, f.y, ax));
                ay = fma(axs, f.y, fma(ays, f.x, ay));
            }
            const int gx = cx * side + lx, gy = cy * side + ly;
            const int64_t gi = coef_base(lvl, gx, gy) + nn * cs;
            double2 r = g[gi];  // M2L part
            r.x += ax;
            r.y += ay;
            cur[i] = r;
            if (leaf)
                leaf_loc[((int64_t)gy * m + gx) * P + nn] = r;
            else
                g[gi] = r;
        }
        __syncthreads();
    }
}

size_t sub_smem(int depth, int P) {
    return sizeof(double2) * ((size_t)(((1 << (2 * (depth + 1))) - 1) / 3) * P + 4 * P) +
           sizeof(double) * (P + 1);
}

int sub_depth(int P) { return sub_smem(3, P) <= 48 * 1024 ? 3 : 2; }

}  // namespace

void launch_m2m(const Layout& L, const Tables* T, double2* mult, cudaStream_t s) {
    const int d0 = sub_depth(L.P);
    for (int lf = L.levels; lf > 2;) {
        const int d = lf - 2 < d0 ? lf - 2 : d0;
        const int lt = lf - d;
        const size_t off_lf = L.level_cell_off[lf] * L.P;
        k_m2m_subtree<<<(unsigned)(1ll << (2 * lt)), kSubThreads, sub_smem(d, L.P), s>>>(
            mult, lf, d, L.P, off_lf, T);
        note_launches(1);
        lf = lt;
    }
}

void launch_l2l(const Layout& L, const Tables* T, double2* loc, double2* leaf_loc, Rows rows,
                cudaStream_t s) {
    if (L.levels == 2) {
        launch_leaf_locals_copy(L, loc, leaf_loc, s);
        return;
    }
    const int d0 = sub_depth(L.P);
    for (int lt = 2; lt < L.levels;) {
        const int d = L.levels - lt < d0 ? L.levels - lt : d0;
        k_l2l_subtree<<<(unsigned)(1ll << (2 * lt)), kSubThreads, sub_smem(d, L.P), s>>>(
            loc, leaf_loc, lt, d, L.levels, L.P, L.level_cell_off[lt] * L.P, T, rows);
        note_launches(1);
        lt += d;
    }
}

}  // namespace vfmm
