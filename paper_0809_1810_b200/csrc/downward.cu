// Downward pass (north-star item 4): L2L to the leaves, then L2P fused with
// the near/far combine and the un-permutation to the caller's order.
//
// Replaces engine.downward_pass (engine.py:190-202),
// expansions.local_shift_matrix (expansions.py:148-155), engine.far_field
// (engine.py:205-213), expansions.f_to_velocity (expansions.py:217-225), the
// combine in engine.evaluate (engine.py:394-396) and the far + near parts of
// engine.evaluate_at (engine.py:434-459).
#include <algorithm>
#include <climits>

#include "vfmm_internal.cuh"

namespace vfmm {

namespace {

// levels == 2 has no L2L: copy the level-2 planar locals to the cell-major leaf array
__global__ void k_leaf_locals_copy(const double2* __restrict__ loc2, int P, double2* __restrict__ out) {
    pdl_enter();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 16 * P) return;
    const int cell = t / P, n = t % P;
    out[t] = loc2[n * coef_stride(2) + coef_base(2, cell & 3, cell >> 2)];
}

// Near-field total per particle, in place in slot 0, right after the near
// field (on its stream, so it overlaps the far-field chain): symmetric
// kernel -- slot 0 (the leaf's own blocks) + the reactions of the existing
// backward neighbours in kind order; generic kernel -- the three
// neighbourhood-row partial sums in row order.  Symmetric mode: one warp per
// leaf, the neighbour test made once per leaf and the leaf's particles (one
// contiguous sorted range) summed with coalesced slot loads; generic mode
// (leaves of any size): one thread per particle.
__global__ void __launch_bounds__(256)
    k_near_sum(const int* __restrict__ keys, double2* __restrict__ near_uv, int64_t n, int levels, Rows rows,
               const int* __restrict__ ls, const Counters* __restrict__ ctr, bool gauss,
               int sym_enabled, int split_from, int item_base, int sym_fused) {
    pdl_enter();
    const int m = 1 << levels;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool sym = sym_enabled && p2p_symmetric(ctr, gauss);
    if (sym && sym_fused) return;  // k_p2p_sym's last writers summed the slots
    if (!sym) {  // generic kernel (leaves of any size): thread per particle
        if (t >= n) return;
        const int64_t i = t;
        const int lf = keys[i];
        if ((lf >> levels) < rows.lo || (lf >> levels) >= rows.hi) return;  // halo particle
        const double2 n0 = near_uv[i], n1 = near_uv[n + i], n2 = near_uv[2 * n + i];
        near_uv[i] = make_double2((n0.x + n1.x) + n2.x, (n0.y + n1.y) + n2.y);
        return;
    }
    // symmetric kernel (leaves of <= 128 particles): warp per leaf
    const int leaf = (int)(t >> 5);
    const int lane = threadIdx.x & 31;
    if (leaf >= m * m) return;
    const int ix = leaf & (m - 1), iy = leaf >> levels;
    if (iy < rows.lo || iy >= rows.hi) return;  // halo leaves of a sharded run
    const int lo = ls[leaf], hi = ls[leaf + 1];
    bool ok[kNearSlots];
    {
#pragma unroll
        for (int k = 1; k < kNearSlots; ++k) {
            // the item of leaf (ix, iy) - d_k wrote slot k; d = (1,0), (-1,1), (0,1), (1,1)
            const int ax = ix - (k == 2 ? -1 : (k == 3 ? 0 : 1)), ay = iy - (k == 1 ? 0 : 1);
            ok[k] = ax >= 0 && ax < m && ay >= 0 && ls[ay * m + ax + 1] != ls[ay * m + ax];
        }
    }
    for (int i = lo + lane; i < hi; i += 32) {
        double2 nv;
        {
            double2 t[kNearSlots];
#pragma unroll
            for (int k = 0; k < kNearSlots; ++k) t[k] = near_uv[(int64_t)k * n + i];
            nv = t[0];
            if (sym_leaf_split(leaf, item_base, split_from) == 2) {  // the leaf's second item
                const double2 t5 = near_uv[(int64_t)kSplitSlot * n + i];
                nv.x += t5.x;
                nv.y += t5.y;
            }
#pragma unroll
            for (int k = 1; k < kNearSlots; ++k) {
                if (ok[k]) {
                    nv.x += t[k].x;
                    nv.y += t[k].y;
                }
            }
        }
        near_uv[i] = nv;
    }
}

// Far field (L2P) + the near total, un-permuted to the caller's order.
__global__ void __launch_bounds__(256)
    k_l2p_combine(const Src* __restrict__ src, const int* __restrict__ keys,
                  const int* __restrict__ perm, const double2* __restrict__ loc,
                  const double2* __restrict__ near_uv, int64_t n, int levels, int P, double xmin,
                  double ymin, double side, const Tables* __restrict__ T, double* __restrict__ u,
                  double* __restrict__ v, Rows rows) {
    pdl_enter();
    __shared__ double sfact[kOrderCap + 16];
    for (int i = threadIdx.x; i < P; i += blockDim.x) sfact[i] = T->invfact[i];
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int m = 1 << levels;
    const int leaf = keys[i];
    const int ix = leaf % m, iy = leaf / m;
    if (iy < rows.lo || iy >= rows.hi) return;  // halo particle of a sharded run
    const double r = side / m;
    const double cx = cell_center(xmin, ix, r), cy = cell_center(ymin, iy, r);
    const double inv_r = 1.0 / r;
    const double2 nv = near_uv[i];
    const Src s = src[i];
    const double2 f =
        eval_local(loc + (int64_t)leaf * P, 1, P, (s.x - cx) * inv_r, (s.y - cy) * inv_r, sfact);
    // f_to_velocity: u = Im f / 2pi, v = Re f / 2pi; then far + near
    const int o = perm[i];
    const double uo = f.y * kInv2Pi + nv.x, vo = f.x * kInv2Pi + nv.y;
    if (v) {
        u[o] = uo;
        v[o] = vo;
    } else {  // interleaved (N, 2) output: one 16-byte store per particle
        reinterpret_cast<double2*>(u)[o] = make_double2(uo, vo);
    }
}

// evaluate_at: one thread per target, far field from the target's leaf local
// expansion, then the near field over the 3x3 neighbourhood (engine.py:434-459).
template <bool GAUSS>
__global__ void __launch_bounds__(256)
    k_eval_at(const double* __restrict__ tx, const double* __restrict__ ty, int64_t mt,
              const Src* __restrict__ src, const int* __restrict__ ls,
              const double2* __restrict__ loc, int levels, int P, double xmin, double ymin,
              double side, const Tables* __restrict__ T, double* __restrict__ u,
              double* __restrict__ v, Counters* ctr) {
    pdl_enter();
    __shared__ double sfact[kOrderCap + 16];
    __shared__ double sexp[kExpTab];
    for (int i = threadIdx.x; i < P; i += blockDim.x) sfact[i] = T->invfact[i];
    const double* stab = stage_exp_table(sexp, T->exp2tab);
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= mt) return;
    const double x = tx[i], y = ty[i];
    const double xmax = xmin + side, ymax = ymin + side;
    if (!((x >= xmin) && (x <= xmax) && (y >= ymin) && (y <= ymax))) {
        atomicAdd(&ctr->bad_count, 1);
        atomicMax(&ctr->first_bad_neg, INT_MAX - (int)i);
        u[i] = 0.0;
        v[i] = 0.0;
        return;
    }
    const int m = 1 << levels;
    int ix = (int)((x - xmin) / side * (double)m);
    int iy = (int)((y - ymin) / side * (double)m);
    ix = ix < m - 1 ? ix : m - 1;
    iy = iy < m - 1 ? iy : m - 1;
    const double r = side / m;
    const double cx = cell_center(xmin, ix, r), cy = cell_center(ymin, iy, r);
    const double inv_r = 1.0 / r;
    const double2 f = eval_local(loc + ((int64_t)iy * m + ix) * P, 1, P, (x - cx) * inv_r,
                                 (y - cy) * inv_r, sfact);
    double nu = 0.0, nv = 0.0;
    const int xlo = ix > 0 ? ix - 1 : 0, xhi = ix < m - 1 ? ix + 1 : m - 1;
    for (int ny = iy - 1; ny <= iy + 1; ++ny) {
        if (ny < 0 || ny >= m) continue;
        const int lo = ls[(int64_t)ny * m + xlo], hi = ls[(int64_t)ny * m + xhi + 1];
        for (int jj = lo; jj < hi; ++jj) {
            const Src s = src[jj];
            pair_acc<GAUSS>(x, y, s.x, s.y, s.g, s.q2, stab, nu, nv);
        }
    }
    u[i] = f.y * kInv2Pi + nu * kInv2Pi;
    v[i] = f.x * kInv2Pi + nv * kInv2Pi;
}

}  // namespace

void launch_leaf_locals_copy(const Layout& L, const double2* loc, double2* leaf_loc, cudaStream_t s) {
    launch_k(k_leaf_locals_copy, (16 * L.P + 127) / 128, 128, 0, s, loc, L.P, leaf_loc);
    note_launches(1);
}

void launch_l2p_combine(const Layout& L, const Tables* T, const Src* src, const int* keys,
                        const int* perm, const double2* loc, const double2* near_uv, double xmin,
                        double ymin, double side, double* u, double* v, Rows rows,
                        cudaStream_t s) {
    launch_k(k_l2p_combine, (unsigned)((L.n + 255) / 256), 256, 0, s, 
        src, keys, perm, loc, near_uv, L.n, L.levels, L.P, xmin, ymin, side, T, u, v, rows);
    note_launches(1);
}

void launch_near_sum(const Layout& L, const int* keys, double2* near_uv, Rows rows,
                     const int* leaf_starts, const Counters* ctr, int kernel, bool sym_fused,
                     cudaStream_t s) {
    const int64_t threads = std::max<int64_t>((int64_t)L.nleaves * 32, L.n);  // sym: warp per leaf; generic: thread per particle
    launch_k(k_near_sum, (unsigned)((threads + 255) / 256), 256, 0, s, keys, near_uv, L.n, L.levels,
             rows, leaf_starts, ctr, kernel == VFMM_KERNEL_GAUSSIAN, sym_disabled() ? 0 : 1,
             p2p_sym_split_from(L, rows), (rows.lo > 0 ? rows.lo - 1 : 0) << L.levels, sym_fused ? 1 : 0);
    note_launches(1);
}

void launch_eval_at(const Layout& L, const Tables* T, const double* tx, const double* ty,
                    int64_t m, const Src* src, const int* leaf_starts, const double2* loc,
                    double xmin, double ymin, double side, int kernel, double* u, double* v,
                    Counters* ctr, cudaStream_t s) {
    const double2* leaf_loc = loc;
    const unsigned g = (unsigned)((m + 255) / 256);
    if (kernel == VFMM_KERNEL_GAUSSIAN)
        launch_k(k_eval_at<true>, g, 256, 0, s, tx, ty, m, src, leaf_starts, leaf_loc, L.levels, L.P,
                                          xmin, ymin, side, T, u, v, ctr);
    else
        launch_k(k_eval_at<false>, g, 256, 0, s, tx, ty, m, src, leaf_starts, leaf_loc, L.levels, L.P,
                                           xmin, ymin, side, T, u, v, ctr);
    note_launches(1);
}

}  // namespace vfmm
