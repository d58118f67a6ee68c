// Internal declarations shared by the vfmm CUDA translation units.
//
// Representation: every expansion is stored in a
// level-independent scaled form so that all translation operators are the
// same at every level and fit in a few KB of tables:
//   multipole  M_n = a_n / (r^{n+1} n!)          a_n as in expansions.py:88-101
//   local      Lh_m = (-1)^m m! r^m L_m           L_m as in expansions.py:148-155
// with r the cell side of the level.  Then (derivation in DESIGN.md):
//   M2M  P_m  = 2^{-(m+1)} sum_{k<=m} M_k  E_q[m-k],   E_q[j] = d_q^j / j!
//   M2L  Lh_m = sum_n H_o[m+n] M_n,                    H_o[q] = q! tau_o^{-(q+1)}
//   L2L  Lh'_n += sum_{m>=n} 2^{-m} Lh_m F_q[m-n],     F_q[j] = (-d_q)^j / j!
//   L2P  f(z)  = sum_m Lh_m / m! (-w)^m,               w = (z - c) / r
// d_q = (cx-1/2) + i(cy-1/2) for child quadrant q = 2*cy + cx and
// tau_o = -(dx + i dy) for the interaction-list offset o = (dx, dy).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "../../include/vfmm.h"

namespace vfmm {

constexpr int kOrderCap = VFMM_ORDER_CAP;
constexpr int kQMax = 2 * kOrderCap + 16;  // H table length (padded for m-chunks)
constexpr int kOffsets = 49;               // 7x7 offset grid (dy+3)*7 + (dx+3)
constexpr int kExpSteps = 64;              // exp table resolution: 2^(n/64)
constexpr int kExpTabN = 60 * kExpSteps + 1;  // exp table entries, n = -3840..0
constexpr int kExpSteps2 = 128;            // symmetric P2P table: 2^(n/128)
constexpr int kExpTab2N = 60 * kExpSteps2 + 1;  // n = -7680..0 (60 KB)
constexpr int kNearRows = 3;               // generic P2P: one partial sum per neighbourhood row
constexpr int kNearSlots = 5;              // symmetric P2P: own blocks + 4 reactions
constexpr int kSplitSlot = 5;              // split items: the leaf's sums from its second item
constexpr int kNearSlotsAlloc = 6;         // near_uv slots allocated per particle
constexpr int kSymMaxLeaf = 128;           // symmetric P2P needs leaves of <= 128 particles

// Packed per-particle source record in leaf-sorted order: x, y, gamma and
// q2 = -1 / (2 sigma^2 ln 2) so that exp(-r^2/(2 sigma^2)) = 2^(r^2 q2).
struct __align__(16) Src {
    double x, y, g, q2;
};

// Device-side counters (one struct at a fixed workspace offset).  Every field
// is zero-initialised (a memset node) and reduced with max/add atomics.
struct Counters {
    unsigned long long m2l_count;
    unsigned long long near_pairs;
    unsigned long long sigma_max_bits;  // ordered-bits encoding of max sigma
    unsigned long long sigma_min_neg;   // ~(ordered bits) of min sigma, max-reduced (0 = none)
    int bad_count;
    int first_bad_neg;  // INT_MAX - smallest out-of-domain index, max-reduced
    int ntasks;
    int task_cursor;  // dynamic P2P work distribution
    int max_leaf;     // largest leaf occupancy (owned rows)
    int sort_fallback;  // 1: a leaf exceeds kFastLeafMax, the LSD radix path builds the tree
};

// Translation tables (device globals, uploaded once per device).
struct Tables {
    double2 H[kOffsets][kQMax];      // M2L Hankel generators
    double2 E[4][kOrderCap + 16];    // M2M
    double2 F[4][kOrderCap + 16];    // L2L
    double invfact[kOrderCap + 16];
    double pow2neg[2 * kOrderCap + 16];  // 2^-k
    double exp2tab[kExpTabN];        // 2^(n/64), n = -3840..0
    // 2^(n/128), n = -7680..0 (symmetric P2P); 16-byte aligned and padded to
    // an even count so one bulk copy (cp.async.bulk) stages it
    alignas(16) double exp2tab2[kExpTab2N + 1];
};

const Tables* device_tables();   // device pointer (uploaded on first use)

struct Layout {
    int64_t n;
    int levels, order, P;  // P = order + 1
    int digit_bits, passes, wc, nchunks;
    size_t nleaves;
    size_t unperm_cursor;
    size_t key_a, key_b, val_a, val_b, hist, task_scratch, fill, near_done, scan_state, src, near_uv, leaf_starts, anc,
        counts, mult, loc, leaf_loc, tasks, stage, counters, total;
    size_t scan_state_tiles, scan_state_bytes, hist_bytes;  // per scan instance: 1 ticket + tiles
    size_t level_cell_off[VFMM_LEVELS_CAP + 2];  // cells before level k (k>=2) in mult/loc
    size_t count_off[VFMM_LEVELS_CAP + 2];       // cells before level k in counts
    size_t max_tasks;
};

bool make_layout(int64_t n, int levels, int order, Layout* L);

// Leaf rows [lo, hi) owned by this call (a row strip of the leaf grid; the
// full grid for a single-GPU evaluate).  Coarser cells are processed when
// their leaf-row span intersects [lo, hi).
struct Rows {
    int lo, hi;
};
__host__ __device__ __forceinline__ bool rows_touch(Rows r, int level_row, int shift) {
    return (level_row << shift) < r.hi && ((level_row + 1) << shift) > r.lo;
}

// Host-side count of kernel launches issued by the library (bench evidence).
void note_launches(int k);

// Programmatic dependent launch (PDL).  Every library kernel starts with
// pdl_enter(): griddepcontrol.wait blocks until the preceding kernel of the
// stream has completed and its memory is visible (a no-op without a
// programmatic dependency), then launch_dependents lets the NEXT kernel's
// CTAs be scheduled as soon as every CTA of this grid has started.  Kernels
// are launched with launch_k (cudaLaunchAttributeProgrammaticStreamSerialization),
// so the launch latency and ramp of a kernel overlap the tail of its
// predecessor instead of adding to the chain (CUDA graphs keep the
// programmatic edges).  Because every kernel waits before touching memory,
// stream order semantics are unchanged.
// Checked / jittered builds (compute-sanitizer is closed on this pool; the
// substitutes, tools/build_variant.sh + tests/test_checked_build.py):
//   -DVFMM_CHECKED  VCHECK(cond) traps on a failed bounds / invariant check
//                   at the kernels' indexing points (a memcheck substitute);
//   -DVFMM_JITTER   every warp sleeps a pseudo-random 0..2 us at kernel entry
//                   and at VJITTER() points inside the work loops, reshuffling
//                   the warp interleaving (a racecheck / synccheck substitute:
//                   results must stay bitwise identical to the plain build).
#ifdef VFMM_CHECKED
#define VCHECK(cond)         \
    do {                     \
        if (!(cond)) __trap(); \
    } while (0)
#else
#define VCHECK(cond) \
    do {             \
    } while (0)
#endif
__device__ __forceinline__ void vjitter_impl() {
#ifdef VFMM_JITTER
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    unsigned h = (unsigned)(t ^ (t >> 17)) * 2654435761u ^ (blockIdx.x * 40503u + (threadIdx.x >> 5) * 977u);
    h ^= h >> 13;
    __nanosleep(h & 2047u);
#endif
}
#define VJITTER() vjitter_impl()

__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    vjitter_impl();
}
bool pdl_enabled();  // VFMM_PDL=0 disables the attribute (A/B measurement)
template <typename... K, typename... A>
inline void launch_k(void (*kern)(K...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     A&&... args) {
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...);
}

// ---- CUDA-graph conditional nodes (device-side path choice) ----
// The build picks its sort path and the near field its kernel on the device
// (k_bin_scatter / k_counts_tasks decide, no host sync).  Stream launches run
// the untaken path's kernels, which return at once; when the call is being
// CAPTURED into a graph, the untaken path is instead put in the body of an IF
// conditional node whose condition a kernel of the taken path sets with
// cudaGraphSetConditional, so a replay launches only the kernels it needs.
struct GraphCond {
    bool on = false;                       // capturing, handle valid
    cudaGraphConditionalHandle h = 0;
};
// A handle on the graph being captured on s (on = false when s is not capturing).
GraphCond graph_cond_create(cudaStream_t s);
bool graph_cond_enabled();  // VFMM_GRAPH_COND=0 disables (A/B)
// Append an IF node on `h` to the capture of s and start capturing its body on
// the library's body stream (returned); graph_cond_end closes the body and
// makes the node the capture dependency of s.
cudaStream_t graph_cond_begin(cudaStream_t s, const GraphCond& c, cudaGraphNode_t* node);
void graph_cond_end(cudaStream_t s, cudaStream_t body, cudaGraphNode_t node);
__device__ __forceinline__ void graph_cond_set(const GraphCond& c, unsigned value) {
    if (c.on && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(c.h, value);
}

// ---- kernels launchers (each enqueues on `s`) ----
void launch_build(const Layout& L, const double* x, const double* y, const double* g,
                  const double* sigma, double xmin, double ymin, double side, char* ws,
                  Counters* ctr, cudaStream_t s, int** keys_out, int** perm_out,
                  cudaEvent_t gs_ready = nullptr, int sigma_stride = 1,
                  // leaf rows owned (occupancy pyramid and task counts, computed in the build)
                  Rows rows = Rows{0, 1 << 30},
                  // optional: the LSD radix kernels as a parallel branch (fork / join events)
                  cudaStream_t lsd_stream = nullptr, cudaEvent_t lsd_fork = nullptr,
                  cudaEvent_t lsd_join = nullptr);
void launch_scan_i32(int* data, int64_t n, unsigned long long* state, cudaStream_t s,
                     const Counters* sym_skip, bool gauss, const int* skip_flag = nullptr,
                     int skip_val = 0);
size_t scan_tiles(int64_t n);
void launch_leaf_starts(const int* sorted_keys, int64_t n, int nleaves, int* leaf_starts,
                        cudaStream_t s);
void launch_tasks(const Layout& L, char* ws, Counters* ctr, Rows rows, bool gauss, cudaStream_t s);
void launch_p2m(const Layout& L, const Src* src, const int* leaf_starts, double xmin, double ymin,
                double side, double2* mult_leaf, const Tables* T, Rows rows, cudaStream_t s);
void launch_init_counters(Counters* ctr, cudaStream_t s);
void launch_m2m(const Layout& L, const Tables* T, double2* mult, Rows rows, cudaStream_t s);  // subtree.cu
void launch_leaf_locals_copy(const Layout& L, const double2* loc, double2* leaf_loc, cudaStream_t s);
void launch_m2l(const Layout& L, const Tables* T, const double2* mult, const int* counts,
                double2* loc, double2* anc, Counters* ctr, Rows rows, cudaStream_t s);
// L2L split level: CTA roots of the fused downward kernel (subtree.cu); the
// M2L parts of levels 3 .. split-1 are also kept in the `anc` region
int l2l_split_level(int levels, int P);
// L2P + combine fused into the finest L2L level (single-GPU evaluates): the
// near-field totals must be complete when the L2L runs.
// One staged output record: 32 bytes, one full sector per store.
struct __align__(16) UnpermRec {
    double u, v;
    int dest;
    int pad[3];
};
constexpr int kUnpermCursorStride = 32;  // ints: a cursor per 128-byte line
constexpr int kSortPathLsdProbe = 1;     // Counters::sort_fallback: random input order (tree.cu)
struct FusedOut {
    const Src* src;
    const int* keys;
    const int* perm;
    const int* ls;
    const double2* near;  // slot 0: near-field total per sorted particle
    double* u;            // null: not fused (leaf_loc only)
    double* v;            // null: interleaved (N, 2) output
    double xmin, ymin, side;
    // staged un-permute (large random-order inputs, see k_unpermute): records go to
    // buckets of 2^stage_shift destination indices first; null = write straight to u / v
    UnpermRec* stage = nullptr;
    int* stage_cursor = nullptr;  // one cursor per bucket, kUnpermCursorStride ints apart
    int stage_shift = 0;
    int64_t n_total = 0;
    const Counters* ctr = nullptr;
};
void launch_l2l(const Layout& L, const Tables* T, double2* loc, double2* leaf_loc,
                const double2* anc, Rows rows, const FusedOut& fo, cudaStream_t s);
// Second pass of the staged un-permute (after launch_l2l with fo.stage set).
void launch_unpermute(const Layout& L, const FusedOut& fo, cudaStream_t s);
// Zero the bucket cursors (enqueued before the fused L2L of a staged call).
void launch_unpermute_prepare(const Layout& L, const FusedOut& fo, cudaStream_t s);
bool l2l_stageable(const Layout& L);
int unperm_shift(int64_t n);  // log2 of the bucket size: 2^16 destinations, <= 1024 buckets
int p2p_targets_per_lane();  // 1 or 2 (env VFMM_P2P_TPT, default 1)
// the near field: P2P kernels and the per-particle near-field totals (slot 0)
void launch_p2p(const Layout& L, const Tables* T, const Src* src, const int* leaf_starts,
                char* ws, Counters* ctr, int kernel, double2* near_uv, Rows rows, const int* keys,
                cudaStream_t s);
bool sym_disabled();  // env VFMM_P2P_SYM=0 forces the generic near-field kernel
// symmetric P2P: leaves [item_base + split_from, ...) get two work items
// (the forward stream split in two, the leaf's own sums of the second in slot
// kSplitSlot), the leaves before them one (same choice in k_near_sum)
int p2p_sym_split_from(const Layout& L, Rows rows);
__host__ __device__ __forceinline__ int sym_leaf_split(int leaf, int item_base, int split_from) {
    return leaf - item_base >= split_from ? 2 : 1;
}
void launch_l2p_combine(const Layout& L, const Tables* T, const Src* src, const int* keys,
                        const int* perm, const double2* loc, const double2* near_uv, double xmin,
                        double ymin, double side, double* u, double* v, Rows rows,
                        cudaStream_t s);
// near-field total per particle into slot 0 (after the near-field kernels)
// sym_fused: the symmetric kernel sums its slots itself (k_near_sum then
// only serves the generic kernel)
void launch_near_sum(const Layout& L, const int* keys, double2* near_uv, Rows rows,
                     const int* leaf_starts, const Counters* ctr, int kernel, bool sym_fused,
                     cudaStream_t s);
void launch_eval_at(const Layout& L, const Tables* T, const double* tx, const double* ty,
                    int64_t m, const Src* src, const int* leaf_starts, const double2* loc,
                    double xmin, double ymin, double side, int kernel, double* u, double* v,
                    Counters* ctr, cudaStream_t s);
int direct_nsplit(int64_t m, int64_t n);
void launch_direct(const double* tx, const double* ty, int64_t m, const double* x,
                   const double* y, const double* g, const double* sigma, int64_t n, int kernel,
                   double* pu, double* pv, int nsplit, double* u, double* v, const Tables* T,
                   cudaStream_t s);

// Cell centre exactly as Tree.centers (quadtree.py:146-152): xmin + (i + 0.5) * s
// with two roundings (no FMA contraction).
__device__ __forceinline__ double cell_center(double lo, int i, double s) {
    return __dadd_rn(lo, __dmul_rn((double)i + 0.5, s));
}

// Planar coefficient layout of one level k >= 2 (2^k cells per side):
//   [P coefficients][4 parity planes][half^2 cells],  half = 2^(k-1),
//   plane = 2*(iy & 1) + (ix & 1),  j = (iy >> 1) * half + (ix >> 1).
// Threads enumerating j within a plane touch consecutive addresses for every
// coefficient, so the M2L / M2M / L2L sweeps are fully coalesced.
__host__ __device__ __forceinline__ int64_t coef_plane_size(int k) {
    return (int64_t)1 << (2 * (k - 1));
}
__host__ __device__ __forceinline__ int64_t coef_base(int k, int ix, int iy) {
    const int64_t half = (int64_t)1 << (k - 1);
    return (int64_t)(((iy & 1) << 1) | (ix & 1)) * half * half + (int64_t)(iy >> 1) * half + (ix >> 1);
}
__host__ __device__ __forceinline__ int64_t coef_stride(int k) {  // between coefficients
    return (int64_t)4 << (2 * (k - 1));
}

int coef_chunk(int P);  // TN of the chunked coefficient kernels (4..8)

// Near-field mode, decided on the device after the build: the symmetric
// (Newton's third law) block kernel needs one core size for every particle
// (the blob factor uses the SOURCE sigma, engine.py:256) and small leaves.
__device__ __forceinline__ bool p2p_symmetric(const Counters* c, bool gauss) {
    const bool uniform = !gauss || ~c->sigma_min_neg == c->sigma_max_bits;
    return uniform && c->max_leaf <= kSymMaxLeaf;
}

// ---- shared device math ----

// Exponential table: 2^(n/64) for n = -3840..0 (y in [-60, 0]); kernels stage
// it in shared memory (30 KB) and pass a pointer to the n = 0 entry (the last).
constexpr int kExpTab = kExpTabN;

// Clamp y <= 0 to y >= -60 with ONE integer op: for non-positive doubles the
// unsigned high word grows with |y|, so min(hi(y), hi(-60)) caps |y| near 60
// (the low word is kept; the result lies in [-60 - 1e-14, -60] when clamped).
// Below -54, 2^y < 2^-54 and 1 - 2^y rounds to 1.0 exactly, as in the reference.
__device__ __forceinline__ double clamp_neg60(double y) {
    const unsigned hi = min((unsigned)__double2hiint(y), 0xC04E0000u);
    return __hiloint2double((int)hi, __double2loint(y));
}

// Taylor coefficients ln2^k / k!, k = 1..5, in the constant bank so that the
// DFMAs take them as c[][] operands (no per-iteration register moves).
static __constant__ double c_exp2_poly[5] = {6.931471805599453e-1, 2.4022650695910072e-1,
                                             5.550410866482158e-2, 9.618129107628477e-3,
                                             1.3333558146428443e-3};

// e = 2^y for y in [-60, 0]: n = round(64 y) via the 1.5*2^52 shifter,
// r = y - n/64 (exact, |r| <= 1/128), 2^y = T[n] * (1 + r P(r)) with the
// degree-5 Taylor polynomial of 2^r = e^(r ln2).  Truncation error
// (ln2/128)^6/6! < 3.6e-17 relative (0.32 ulp); total error ~1 ulp.
// Returns (T, r P(r)) so the caller can fold 1 - e into one FMA.
__device__ __forceinline__ double exp2_neg_parts(double y, const double* __restrict__ tab_end,
                                                 double& T) {
    const double kShift = 6755399441055744.0;  // 1.5 * 2^52
    const double t = fma(y, (double)kExpSteps, kShift);
    const int n = __double2loint(t);
    const double nf = t - kShift;
    const double r = fma(nf, -1.0 / kExpSteps, y);  // exact
    double p = c_exp2_poly[4];
    p = fma(p, r, c_exp2_poly[3]);
    p = fma(p, r, c_exp2_poly[2]);
    p = fma(p, r, c_exp2_poly[1]);
    p = fma(p, r, c_exp2_poly[0]);
    T = tab_end[n];
    return r * p;
}

__device__ __forceinline__ double exp2_neg(double y, const double* __restrict__ tab_end) {
    double T;
    const double rp = exp2_neg_parts(y, tab_end, T);
    return fma(T, rp, T);
}

// 1/x via the MUFU reciprocal seed and one cubically convergent refinement.
// x = +0 is first raised to 2^-930 (integer max on the high word), so the
// reciprocal stays finite (~1e280); x >= 2^-930 is unchanged.
__device__ __forceinline__ double rcp_fast(double x) {
    const unsigned hi = max((unsigned)__double2hiint(x), 0x05D00000u);
    x = __hiloint2double((int)hi, __double2loint(x));
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    e = fma(e, e, e);
    return fma(y, e, y);
}

// Accumulate the pair interaction of source (sx, sy, g, q2) on target (tx, ty):
// (u, v) += g (1 - exp(-r^2/(2 sigma^2))) / r^2 * (-dy, dx)  [times 1/2pi later]
// Same arithmetic structure as kernels.kernel_eval (kernels.py:39-49) and
// engine._pair_velocity (engine.py:245-257).  A coincident pair (r^2 == 0)
// contributes exactly zero: dx = dy = 0 multiply a finite c (the reference's
// r^2 > 0 mask, without a per-pair select).
template <bool GAUSS>
__device__ __forceinline__ void pair_acc(double tx, double ty, double sx, double sy, double g,
                                         double q2, const double* __restrict__ tab_end, double& u,
                                         double& v) {
    const double dx = tx - sx;
    const double dy = ty - sy;
    const double r2 = fma(dy, dy, dx * dx);
    double c = g * rcp_fast(r2);
    if (GAUSS) c = fma(-c, exp2_neg(clamp_neg60(r2 * q2), tab_end), c);  // c (1 - e)
    u = fma(-c, dy, u);
    v = fma(c, dx, v);
}

// Horner evaluation of the leaf local expansion at z:
//   f(z) = sum_m Lh_m / m! (-w)^m,  w = (z - c) / r
__device__ __forceinline__ double2 eval_local(const double2* __restrict__ Lh, int64_t stride, int P,
                                              double wx, double wy,
                                              const double* __restrict__ invfact) {
    const double nx = -wx, ny = -wy;
    const double2 top = Lh[(P - 1) * stride];
    double ax = top.x * invfact[P - 1], ay = top.y * invfact[P - 1];
#pragma unroll 6
    for (int k = P - 2; k >= 0; --k) {
        const double2 c = Lh[k * stride];
        const double f = invfact[k];
        const double tx = fma(ax, nx, fma(-ay, ny, c.x * f));
        const double ty = fma(ax, ny, fma(ay, nx, c.y * f));
        ax = tx;
        ay = ty;
    }
    return make_double2(ax, ay);
}

// NB independent evaluations of eval_local advanced together (coefficient
// k of every particle, then k - 1, ...): NB Horner chains in flight instead of
// one; each particle's arithmetic and order are eval_local's exactly.
// Lh here holds the coefficients already multiplied by 1/k! (the products
// eval_local forms per particle, formed once per leaf: same values).
template <int NB>
__device__ __forceinline__ void eval_local_multi(const double2* const (&Lh)[NB], int P,
                                                 const double (&wx)[NB], const double (&wy)[NB],
                                                 double2 (&out)[NB]) {
    double ax[NB], ay[NB];
#pragma unroll
    for (int u = 0; u < NB; ++u) {
        const double2 top = Lh[u][P - 1];
        ax[u] = top.x;
        ay[u] = top.y;
    }
#pragma unroll 2
    for (int k = P - 2; k >= 0; --k) {
#pragma unroll
        for (int u = 0; u < NB; ++u) {
            const double2 c = Lh[u][k];
            const double nx = -wx[u], ny = -wy[u];
            const double tx = fma(ax[u], nx, fma(-ay[u], ny, c.x));
            const double ty = fma(ax[u], ny, fma(ay[u], nx, c.y));
            ax[u] = tx;
            ay[u] = ty;
        }
    }
#pragma unroll
    for (int u = 0; u < NB; ++u) out[u] = make_double2(ax[u], ay[u]);
}

// Stage the exponential table in shared memory (all threads of the block).
__device__ __forceinline__ const double* stage_exp_table(double* smem, const double* __restrict__ g) {
    for (int i = threadIdx.x; i < kExpTab; i += blockDim.x) smem[i] = g[i];
    return smem + (kExpTab - 1);
}

constexpr double kInv2Pi = 0.15915494309189535;  // 1 / (2 pi)
constexpr double kTwoPi = 6.283185307179586;

}  // namespace vfmm
