// Multipole exchange of the sharded evaluate (north_star:
// "coarse-level multipole coefficients are exchanged by NCCL allgather over
// NVLink and neighbour-leaf particles by halo exchange").
//
// Leaves are sharded in row strips [lo, hi) of the 2^l x 2^l leaf grid.
// PHASE_UP is strip-local: P2M visits the owned leaves, M2M the subtrees
// whose leaf rows touch the strip, and a coarse cell that straddles strips
// holds this rank's PARTIAL multipole (the multipoles are linear in Gamma).
// The M2L of a destination reaches source cells at most two cell rows away
// (dy in [-2-py, 3-py] around iy = 2 jy + py: rows 2 jy - 2 .. 2 jy + 3, i.e.
// the children of the parent's neighbours, engine._il_offsets,
// engine.py:77-89), so per level k:
//   * FINE levels (every strip starts and ends on an even cell row of level k
//     and is >= 2 cell rows tall): a rank needs the two cell rows below its
//     first row and the two above its last one, all owned by the neighbour
//     strips -- ONE row of each parity plane of the planar layout, sent by
//     grouped NCCL send / recv (the halo buffers below);
//   * COARSE levels (2 .. kc): the level is small (4^k cells) and every rank
//     needs most of it: each rank contributes its partials of the cells that
//     touch its strip (zero elsewhere), an NCCL allgather collects the world's
//     contributions and the unpack adds them in rank order (deterministic).
// The occupancy pyramid (owned rows only, tree.cu k_counts_tasks) travels the
// same way: the M2L skips empty sources and counts (destination, nonempty
// source) pairs (engine.py:173-180).
//
// Buffers (caller-owned device memory, vfmm_shard_exchange_size):
//   coarse : [mult cells of levels 2..kc, planar prefix of `mult`][counts of
//            levels 0..kc, prefix of `counts`]                (kc >= 2 only)
//   halo   : [per fine level k: P x 4 planes x half double2][per fine level:
//            2 cell rows x 2^k int32]
#include <cstring>

#include "vfmm_internal.cuh"

namespace vfmm {

namespace {

struct ExchangePlan {
    int levels, P, kc, kf;  // fine levels kf .. levels (kf = max(2, kc + 1))
    int lo, hi;             // owned leaf rows
    int64_t coarse_mult;    // double2 elements of the coarse mult section
    int64_t coarse_cnt;     // int32 elements of the coarse counts section
    size_t coarse_cnt_off;  // byte offset of the counts section in the coarse buffer
    int64_t halo_mult;      // double2 elements of the halo mult section
    int64_t halo_cnt;       // int32 elements of the halo counts section
    size_t halo_cnt_off;    // byte offset of the counts section in a halo buffer
    int64_t lvl_mult_off[VFMM_LEVELS_CAP + 2];  // halo mult element offset of fine level k
    int64_t lvl_cnt_off[VFMM_LEVELS_CAP + 2];   // halo counts element offset of fine level k
    size_t mult_off[VFMM_LEVELS_CAP + 2];       // Layout::level_cell_off (cells)
    size_t count_off[VFMM_LEVELS_CAP + 2];      // Layout::count_off
};

inline size_t align16(size_t b) { return (b + 15) / 16 * 16; }

bool make_plan(const Layout& L, int row_lo, int row_hi, int kc, ExchangePlan* e) {
    if (kc < 1 || kc > L.levels) return false;
    std::memset(e, 0, sizeof(*e));
    e->levels = L.levels;
    e->P = L.P;
    e->kc = kc;
    e->kf = kc + 1 > 2 ? kc + 1 : 2;
    e->lo = row_lo;
    e->hi = row_hi;
    for (int k = 0; k <= L.levels + 1; ++k) {
        e->mult_off[k] = k >= 2 ? L.level_cell_off[k] : 0;
        e->count_off[k] = L.count_off[k];
    }
    if (kc >= 2) {
        e->coarse_mult = (int64_t)L.level_cell_off[kc + 1] * L.P;
        e->coarse_cnt = (int64_t)L.count_off[kc + 1];
    }
    e->coarse_cnt_off = align16(sizeof(double2) * (size_t)e->coarse_mult);
    int64_t hm = 0, hc = 0;
    for (int k = e->kf; k <= L.levels; ++k) {
        e->lvl_mult_off[k] = hm;
        e->lvl_cnt_off[k] = hc;
        hm += (int64_t)L.P * 4 * (1ll << (k - 1));
        hc += 2ll << k;
    }
    e->halo_mult = hm;
    e->halo_cnt = hc;
    e->halo_cnt_off = align16(sizeof(double2) * (size_t)hm);
    // fine levels: strips start / end on even cell rows and hold >= 2 rows
    if (row_hi > row_lo)
        for (int k = e->kf; k <= L.levels; ++k) {
            const int s = L.levels - k;
            const int mask = (1 << (s + 1)) - 1;
            if ((row_lo & mask) != 0 || (row_hi & mask) != 0 || ((row_hi - row_lo) >> s) < 2)
                return false;
        }
    return true;
}

size_t coarse_bytes(const ExchangePlan& e) {
    return e.coarse_mult ? e.coarse_cnt_off + align16(sizeof(int) * (size_t)e.coarse_cnt) : 0;
}
size_t halo_bytes(const ExchangePlan& e) {
    return e.halo_mult ? e.halo_cnt_off + align16(sizeof(int) * (size_t)e.halo_cnt) : 0;
}

// fine level of halo element i (levels ascending)
__device__ __forceinline__ int level_of(const int64_t* off, int kf, int levels, int64_t i) {
    int k = kf;
    while (k < levels && i >= off[k + 1]) ++k;
    return k;
}

// coarse mult element e (planar prefix of mult): does its cell touch the strip?
__device__ __forceinline__ bool coarse_touch(const ExchangePlan& p, int64_t e) {
    int k = 2;
    while (k < p.kc && e >= (int64_t)p.mult_off[k + 1] * p.P) ++k;
    const int64_t r = e - (int64_t)p.mult_off[k] * p.P;
    const int64_t psz = coef_plane_size(k);
    const int plane = (int)((r / psz) & 3);
    const int jy = (int)((r % psz) >> (k - 1));
    const int iy = 2 * jy + (plane >> 1);
    return rows_touch(Rows{p.lo, p.hi}, iy, p.levels - k);
}

// Halo element -> workspace element.  dir 0: rows of the boundary BELOW the
// strip (first owned rows when packing, rows lo_k - 2, lo_k - 1 when
// unpacking); dir 1: ABOVE (last owned rows / rows hi_k, hi_k + 1).
__device__ __forceinline__ int64_t halo_mult_elem(const ExchangePlan& p, int64_t i, bool pack, int dir) {
    const int k = level_of(p.lvl_mult_off, p.kf, p.levels, i);
    const int half = 1 << (k - 1);
    const int64_t r = i - p.lvl_mult_off[k];
    const int coef = (int)(r / (4 * half)), plane = (int)((r / half) & 3), jx = (int)(r % half);
    const int s = p.levels - k;
    const int lo2 = (p.lo >> s) >> 1, hi2 = (p.hi >> s) >> 1;  // plane rows of the strip
    const int jy = dir == 0 ? (pack ? lo2 : lo2 - 1) : (pack ? hi2 - 1 : hi2);
    VCHECK(jy >= 0 && jy < half && coef < p.P);
    const int64_t psz = (int64_t)half * half;
    return (int64_t)p.mult_off[k] * p.P + coef * 4 * psz + plane * psz + (int64_t)jy * half + jx;
}
__device__ __forceinline__ int64_t halo_cnt_elem(const ExchangePlan& p, int64_t i, bool pack, int dir) {
    const int k = level_of(p.lvl_cnt_off, p.kf, p.levels, i);
    const int mk = 1 << k;
    const int64_t r = i - p.lvl_cnt_off[k];
    const int row = (int)(r / mk), ix = (int)(r % mk);
    const int s = p.levels - k;
    const int lo = p.lo >> s, hi = p.hi >> s;
    const int iy = dir == 0 ? (pack ? lo : lo - 2) + row : (pack ? hi - 2 : hi) + row;
    VCHECK(iy >= 0 && iy < mk && row < 2);
    return (int64_t)p.count_off[k] + (int64_t)iy * mk + ix;
}

__global__ void k_shard_pack(const __grid_constant__ ExchangePlan p, const double2* __restrict__ mult,
                             const int* __restrict__ counts, char* __restrict__ coarse,
                             char* __restrict__ down, char* __restrict__ up) {
    pdl_enter();
    const int64_t n1 = coarse ? p.coarse_mult : 0, n2 = coarse ? p.coarse_cnt : 0;
    const int64_t n3 = p.halo_mult, n4 = p.halo_cnt;
    const bool empty = p.hi <= p.lo;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n1 + n2 + n3 + n4;
         t += (int64_t)gridDim.x * blockDim.x) {
        if (t < n1) {
            ((double2*)coarse)[t] = !empty && coarse_touch(p, t) ? mult[t] : make_double2(0.0, 0.0);
        } else if (t < n1 + n2) {
            const int64_t i = t - n1;
            ((int*)(coarse + p.coarse_cnt_off))[i] = empty ? 0 : counts[i];
        } else if (t < n1 + n2 + n3) {
            if (empty) continue;
            const int64_t i = t - n1 - n2;
            if (down) ((double2*)down)[i] = mult[halo_mult_elem(p, i, true, 0)];
            if (up) ((double2*)up)[i] = mult[halo_mult_elem(p, i, true, 1)];
        } else {
            if (empty) continue;
            const int64_t i = t - n1 - n2 - n3;
            if (down) ((int*)(down + p.halo_cnt_off))[i] = counts[halo_cnt_elem(p, i, true, 0)];
            if (up) ((int*)(up + p.halo_cnt_off))[i] = counts[halo_cnt_elem(p, i, true, 1)];
        }
    }
}

__global__ void k_shard_unpack(const __grid_constant__ ExchangePlan p, double2* __restrict__ mult,
                               int* __restrict__ counts, const char* __restrict__ coarse_all, int world,
                               size_t coarse_stride, const char* __restrict__ below,
                               const char* __restrict__ above) {
    pdl_enter();
    const int64_t n1 = coarse_all ? p.coarse_mult : 0, n2 = coarse_all ? p.coarse_cnt : 0;
    const int64_t n3 = p.halo_mult, n4 = p.halo_cnt;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n1 + n2 + n3 + n4;
         t += (int64_t)gridDim.x * blockDim.x) {
        if (t < n1) {  // sum of the world's partials, rank order
            double sx = 0.0, sy = 0.0;
            for (int r = 0; r < world; ++r) {
                const double2 v = ((const double2*)(coarse_all + r * coarse_stride))[t];
                sx += v.x;
                sy += v.y;
            }
            mult[t] = make_double2(sx, sy);
        } else if (t < n1 + n2) {
            const int64_t i = t - n1;
            int c = 0;
            for (int r = 0; r < world; ++r)
                c += ((const int*)(coarse_all + r * coarse_stride + p.coarse_cnt_off))[i];
            counts[i] = c;
        } else if (t < n1 + n2 + n3) {
            const int64_t i = t - n1 - n2;
            if (below) mult[halo_mult_elem(p, i, false, 0)] = ((const double2*)below)[i];
            if (above) mult[halo_mult_elem(p, i, false, 1)] = ((const double2*)above)[i];
        } else {
            const int64_t i = t - n1 - n2 - n3;
            if (below) counts[halo_cnt_elem(p, i, false, 0)] = ((const int*)(below + p.halo_cnt_off))[i];
            if (above) counts[halo_cnt_elem(p, i, false, 1)] = ((const int*)(above + p.halo_cnt_off))[i];
        }
    }
}

unsigned exchange_grid(const ExchangePlan& e) {
    const int64_t total = e.coarse_mult + e.coarse_cnt + e.halo_mult + e.halo_cnt;
    const int64_t b = (total + 255) / 256;
    return (unsigned)(b < 1 ? 1 : (b > 148 * 8 ? 148 * 8 : b));
}

}  // namespace

}  // namespace vfmm

using namespace vfmm;

extern "C" {

int vfmm_shard_exchange_size(int64_t n, int levels, int order, int row_lo, int row_hi, int kc,
                             size_t* coarse, size_t* halo) {
    Layout L;
    ExchangePlan e;
    if (!coarse || !halo || !make_layout(n, levels, order, &L)) return VFMM_EINVAL;
    if (row_lo < 0 || row_hi > (1 << levels) || row_lo > row_hi) return VFMM_EINVAL;
    if (!make_plan(L, row_lo, row_hi, kc, &e)) return VFMM_EINVAL;
    *coarse = coarse_bytes(e);
    *halo = halo_bytes(e);
    return VFMM_OK;
}

int vfmm_shard_pack(int64_t n, int levels, int order, int row_lo, int row_hi, int kc,
                    const void* workspace, void* coarse, void* halo_down, void* halo_up, void* stream) {
    Layout L;
    ExchangePlan e;
    if (!workspace || !make_layout(n, levels, order, &L)) return VFMM_EINVAL;
    if (row_lo < 0 || row_hi > (1 << levels) || row_lo > row_hi) return VFMM_EINVAL;
    if (!make_plan(L, row_lo, row_hi, kc, &e)) return VFMM_EINVAL;
    if (coarse_bytes(e) && !coarse) return VFMM_EINVAL;
    if (!halo_bytes(e)) halo_down = halo_up = nullptr;
    if (!coarse_bytes(e) && !halo_down && !halo_up) return VFMM_OK;
    const char* ws = (const char*)workspace;
    launch_k(k_shard_pack, exchange_grid(e), 256, 0, (cudaStream_t)stream, e,
             (const double2*)(ws + L.mult), (const int*)(ws + L.counts), (char*)coarse,
             (char*)halo_down, (char*)halo_up);
    note_launches(1);
    return cudaGetLastError() == cudaSuccess ? VFMM_OK : VFMM_ECUDA;
}

int vfmm_shard_unpack(int64_t n, int levels, int order, int row_lo, int row_hi, int kc, void* workspace,
                      const void* coarse_all, int world, const void* halo_below, const void* halo_above,
                      void* stream) {
    Layout L;
    ExchangePlan e;
    if (!workspace || world < 1 || !make_layout(n, levels, order, &L)) return VFMM_EINVAL;
    if (row_lo < 0 || row_hi > (1 << levels) || row_lo > row_hi) return VFMM_EINVAL;
    if (!make_plan(L, row_lo, row_hi, kc, &e)) return VFMM_EINVAL;
    if (coarse_bytes(e) && !coarse_all) return VFMM_EINVAL;
    if (!halo_bytes(e)) halo_below = halo_above = nullptr;
    if (!coarse_bytes(e) && !halo_below && !halo_above) return VFMM_OK;
    char* ws = (char*)workspace;
    launch_k(k_shard_unpack, exchange_grid(e), 256, 0, (cudaStream_t)stream, e,
             (double2*)(ws + L.mult), (int*)(ws + L.counts), (const char*)coarse_all, world,
             coarse_bytes(e), (const char*)halo_below, (const char*)halo_above);
    note_launches(1);
    return cudaGetLastError() == cudaSuccess ? VFMM_OK : VFMM_ECUDA;
}

}  // extern "C"
