/*
 * vfmm.h — C ABI of the B200-native FMM velocity evaluation for 2-D
 * Gaussian-regularised vortex particles (drop-in for the reference package
 * `vortexfmm`, arXiv 0809.1810).
 *
 * Every entry point takes plain pointers and sizes; all particle / velocity
 * buffers are caller-owned DEVICE memory and all work is enqueued on the
 * caller's CUDA stream (`stream` is a cudaStream_t passed as void*, NULL =
 * legacy default stream).  No torch types cross this boundary.
 *
 * Reference interfaces replaced (paths relative to the reference package
 * `pkg/src/vortexfmm/`):
 *   vfmm_evaluate        <- engine.evaluate            engine.py:335-398
 *   vfmm_evaluate_at     <- engine.evaluate_at         engine.py:401-460
 *   vfmm_direct          <- kernels.velocity_direct    kernels.py:52-94
 *   vfmm_workspace_size  <- (no reference analogue: numpy allocates inside
 *                            engine.upward_pass/translate_pass, engine.py:114-187)
 *   vfmm_layout          <- read-only views that the reference exposes as
 *                           Tree.order / Tree.leaf_starts (quadtree.py:116-134)
 *                           and the per-level multipole / local lists returned
 *                           by upward_pass / translate_pass (engine.py:114-187)
 *   vfmm_stats           <- engine.FmmRunStats         engine.py:58-74
 *
 * Threading: every entry point may be called from any host thread.  Calls on
 * one device serialise their enqueue (the library's internal per-device
 * streams, events and pinned counter staging are shared); a call with
 * VFMM_FLAG_STATS also holds the device until it has synchronised and read
 * its counters.  Concurrent calls must use distinct workspaces (a workspace
 * holds the whole state of one evaluate); the Python layer keys its cached
 * workspaces by thread.  The caller's current device is restored on return.
 *
 * Sizes: 1 <= n < 2^30 (32-bit sorted indices), 2 <= levels <= 13,
 * 0 <= order <= 60.
 *
 * Status codes (return value of every function):
 */
#ifndef VFMM_H
#define VFMM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VFMM_OK 0
#define VFMM_EINVAL 1        /* bad argument: FmmConfig.validate / empty input (engine.py:49-55,346-347) */
#define VFMM_EDOMAIN 2       /* particle or target outside the closed domain square (quadtree.py:191-198) */
#define VFMM_ECUDA 3         /* CUDA runtime error */
#define VFMM_EWORKSPACE 4    /* workspace pointer NULL or smaller than vfmm_workspace_size() */

#define VFMM_KERNEL_POINT 0     /* KernelKind.POINT_VORTEX  (kernels.py:27-29) */
#define VFMM_KERNEL_GAUSSIAN 1  /* KernelKind.GAUSSIAN_BLOB (kernels.py:27-29) */

#define VFMM_ORDER_CAP 60       /* expansions.ORDER_CAP (expansions.py:39) */
#define VFMM_LEVELS_CAP 13      /* 4^13 leaves; int32 leaf keys */

/* Flags for vfmm_evaluate */
#define VFMM_FLAG_STATS 1u      /* synchronise the stream at the end and fill *stats (counters, t_total) */
#define VFMM_FLAG_OVERLAP 2u    /* run the near field (P2P) on a side stream concurrently with the
                                   far-field chain; phase timings then overlap */
#define VFMM_FLAG_FAR_ONLY 4u   /* build the tree and the local expansions only (no near field, no
                                   evaluation at the particles); used before vfmm_evaluate_at */
#define VFMM_FLAG_PHASE_UP 8u   /* vfmm_evaluate_shard: build + P2M + M2M (+ the near field when
                                   VFMM_FLAG_OVERLAP is also set: it then runs on an internal stream
                                   and hides the caller's exchange) */
#define VFMM_FLAG_PHASE_TIMES 64u /* with VFMM_FLAG_STATS: also time every phase (CUDA events between
                                   the phases; costs ~0.1 ms per call) */
#define VFMM_FLAG_SIGMA_SCALAR 128u /* vfmm_evaluate_host: sigma points to ONE core size shared by
                                     all particles (8 bytes copied instead of 8 N) */
#define VFMM_FLAG_UV_PAIRS 32u  /* u is an interleaved (N, 2) array of (u, v) rows -- the reference's
                                   return layout (engine.py:394-398); v is ignored */
#define VFMM_FLAG_PHASE_DOWN 16u /* vfmm_evaluate_shard: M2L + L2L + P2P + L2P on the workspace of a
                                    previous PHASE_UP call (after the caller exchanged the multipoles).
                                    Whether the near field still has to run is taken from what that
                                    PHASE_UP recorded for the workspace, not from this call's
                                    VFMM_FLAG_OVERLAP; PHASE_DOWN without a PHASE_UP -> VFMM_EINVAL */
#define VFMM_FLAG_GRAPH_PHASES 512u /* while the call is captured into a CUDA graph (and without
                                   VFMM_FLAG_STATS): its phase events become event-record nodes of
                                   the graph; after a replay vfmm_graph_phase_times() reads the
                                   phase times as the graph ran them (benchmarks; one such graph per
                                   device at a time) */
#define VFMM_FLAG_GRAPH 256u    /* vfmm_evaluate_host: run the device part as a CUDA graph, captured
                                   on first use and cached per (device, workspace, n, levels, order,
                                   kernel, domain, flags); the copies stay plain async copies on
                                   `stream` around the graph launch.  Not with VFMM_FLAG_PHASE_TIMES
                                   (falls back to stream launches), nor while `stream` is capturing */

/* engine.FmmRunStats (engine.py:58-74).  Times in milliseconds (CUDA events). */
typedef struct vfmm_stats {
    int64_t n;
    int64_t m2l_count;        /* translations performed, engine.py:173-180 */
    int64_t near_pair_count;  /* sum over leaves of n_leaf*(n_nbhd-1), engine.py:284 */
    int32_t levels;
    int32_t order;
    int32_t sigma_guard_ok;   /* engine.py:361-370 (GAUSSIAN only) */
    int32_t bad_count;        /* number of out-of-domain particles (status VFMM_EDOMAIN) */
    int64_t first_bad;        /* smallest out-of-domain index, -1 if none */
    double max_sigma;         /* max core radius seen (sigma guard input) */
    double sigma_guard;       /* leaf half-width / 2 */
    float t_build, t_upward, t_m2l, t_downward, t_eval, t_near, t_total;
    int32_t overlapped;       /* 1 if VFMM_FLAG_OVERLAP was used */
} vfmm_stats;

/* Byte offsets of the internal arrays inside the workspace (debug / parity
 * views).  All arrays are in leaf-sorted particle order unless noted.      */
typedef struct vfmm_layout {
    size_t perm;          /* int32 [n]       Tree.order: sorted -> original index */
    size_t leaf_key;      /* int32 [n]       Tree.sorted_leaf (row-major leaf key) */
    size_t leaf_starts;   /* int32 [4^l+1]   Tree.leaf_starts */
    size_t sources;       /* double4 [n]     (x, y, gamma, -1/(2 sigma^2 ln2)) sorted */
    size_t near_uv;       /* double2 [3][n]  near-field (u, v) partial sums per neighbourhood row, sorted order */
    size_t mult;          /* double2 [sum_{k=2..l} 4^k (p+1)]  scaled multipoles, level 2 first */
    size_t loc;           /* double2 [same]  scaled locals (M2L part at the leaf level), level 2 first */
    size_t leaf_loc;      /* double2 [4^l][p+1] completed leaf locals, cell-major */
    size_t counts;        /* int32  [sum_{k=0..l} 4^k] per-level occupancy, level 0 first */
    size_t total;         /* workspace bytes */
} vfmm_layout;

/* Workspace bytes needed for one evaluate of n particles. */
int vfmm_workspace_size(int64_t n, int levels, int order, size_t* bytes);
int vfmm_layout_of(int64_t n, int levels, int order, vfmm_layout* out);

/* engine.evaluate (engine.py:335-398), device arrays, original particle order.
 *   x, y, gamma, sigma : double[n] device
 *   (xmin, ymin, side) : model.Domain (model.py:39-65); side > 0
 *   u, v               : double[n] device outputs, original particle order
 *   stats              : host pointer, filled when flags has VFMM_FLAG_STATS
 * Without VFMM_FLAG_STATS the call is fully asynchronous and CUDA-graph
 * capturable (no allocation, no synchronisation); the domain check and the
 * counters can then be read with vfmm_read_stats after synchronising.      */
int vfmm_evaluate(const double* x, const double* y, const double* gamma, const double* sigma,
                  int64_t n, double xmin, double ymin, double side, int levels, int order,
                  int kernel, double* u, double* v, void* workspace, size_t workspace_bytes,
                  unsigned flags, vfmm_stats* stats, void* stream);

/* engine.evaluate with HOST buffers (the reference's numpy-in / numpy-out
 * contract, engine.py:335-398): x, y, gamma, sigma and u, v are host arrays
 * (pinned for full speed).  The copies are staged through the workspace and
 * overlapped with the build: positions first (binning / sort need only them),
 * gamma and sigma while the sort runs; u, v are copied back at the end, on
 * `stream`.  Synchronous on `stream` only if VFMM_FLAG_STATS is set.  Without
 * it, calls on distinct streams AND distinct workspaces pipeline: the copies
 * of one call overlap the compute of the previous one (the compute itself is
 * serialised on the library's internal per-device streams).  With
 * VFMM_FLAG_GRAPH the compute is one cached CUDA-graph launch on `stream`
 * after all input copies (no launch gaps; graphs of distinct workspaces may
 * run concurrently).                                                        */
int vfmm_evaluate_host(const double* x, const double* y, const double* gamma, const double* sigma,
                       int64_t n, double xmin, double ymin, double side, int levels, int order,
                       int kernel, double* u, double* v, void* workspace, size_t workspace_bytes,
                       unsigned flags, vfmm_stats* stats, void* stream);

/* vfmm_evaluate_host for a batch of INDEPENDENT evaluations kept in flight
 * (the reference runs them one after another, harness.py:211-267): the same
 * host-buffer contract (engine.py:335-398), with the three stages of a call
 * on three streams of the caller -- the input copies on `h2d_stream`, the
 * cached CUDA graph of the device part on `compute_stream` (VFMM_FLAG_GRAPH is
 * implied), the copy of (u, v) back on `d2h_stream` -- ordered by events
 * inside the library.  The copy streams are meant to be shared by every call
 * of the batch (copies are serialised by the two copy engines anyway) and the
 * compute streams to be few (evaluations on distinct compute streams share
 * the SMs), so input copies run ahead of the compute and results drain behind
 * it, whatever the number of buffers in flight.  The call has completed when
 * `d2h_stream` reaches the point of the call's return (record an event there);
 * ONE call per workspace may be in flight.  No VFMM_FLAG_STATS / phase flags
 * (VFMM_EINVAL); the three streams must be distinct, the copy streams non-NULL. */
int vfmm_evaluate_host_streams(const double* x, const double* y, const double* gamma,
                               const double* sigma, int64_t n, double xmin, double ymin, double side,
                               int levels, int order, int kernel, double* u, double* v,
                               void* workspace, size_t workspace_bytes, unsigned flags,
                               void* compute_stream, void* h2d_stream, void* d2h_stream);

/* Sharded evaluate (one process per GPU; leaves sharded in row strips).
 * The local arrays hold this rank's owned particles (leaf rows [row_lo,
 * row_hi) of the 2^levels x 2^levels leaf grid) plus halo copies of the
 * particles in leaf rows row_lo-1 and row_hi (the P2P of the boundary leaves,
 * engine.py:216-235).  Per evaluate:
 *   PHASE_UP   : tree over the local particles; strip-local upward pass: P2M
 *                of the owned leaves, M2M of the subtrees touching the strip
 *                (a coarse cell straddling strips gets this rank's PARTIAL
 *                multipole); with VFMM_FLAG_OVERLAP the near field starts.
 *   (caller)   : vfmm_shard_pack -> NCCL allgather of the coarse buffers and
 *                grouped send/recv of the halo buffers with the neighbour
 *                strips -> vfmm_shard_unpack (see below).
 *   PHASE_DOWN : M2L / L2L for cells touching the owned strip, P2P for owned
 *                leaves, L2P + combine for owned particles (u, v of halo
 *                particles are left untouched).
 * Counters: m2l_count counts destinations whose first leaf row is owned and
 * near_pair_count owned leaves, so their sums over ranks equal the
 * single-GPU values.  Replaces engine.evaluate (engine.py:335-398) per shard. */
int vfmm_evaluate_shard(const double* x, const double* y, const double* gamma, const double* sigma,
                        int64_t n, double xmin, double ymin, double side, int levels, int order,
                        int kernel, int row_lo, int row_hi, double* u, double* v, void* workspace,
                        size_t workspace_bytes, unsigned flags, vfmm_stats* stats, void* stream);

/* Multipole exchange of the sharded evaluate.  The M2L of a cell reaches two
 * cell rows up and down (engine.py:77-89), so with every strip starting and
 * ending on an even cell row of level k and >= 2 rows tall ("fine" levels
 * kc+1 .. levels) a rank needs one plane row of each parity plane from each
 * neighbour strip; the small "coarse" levels 2 .. kc (kc <= 1: none) are
 * all-gathered (each rank's partials of the cells touching its strip, zero
 * elsewhere) and summed in rank order.  The occupancy pyramid travels along.
 * Buffer sizes depend on (levels, order, kc) only, so they are equal on every
 * rank; VFMM_EINVAL when a level above kc is not fine for this strip.        */
int vfmm_shard_exchange_size(int64_t n, int levels, int order, int row_lo, int row_hi, int kc,
                             size_t* coarse_bytes, size_t* halo_bytes);
/* After PHASE_UP, on `stream`: this rank's coarse contribution, its first
 * owned plane rows (halo_down, for the strip below) and its last ones
 * (halo_up, for the strip above).  NULL halo pointers are skipped.          */
int vfmm_shard_pack(int64_t n, int levels, int order, int row_lo, int row_hi, int kc,
                    const void* workspace, void* coarse, void* halo_down, void* halo_up, void* stream);
/* Before PHASE_DOWN, on `stream`: coarse levels = the sum of the `world`
 * contributions in coarse_all (rank order, coarse_bytes apart); the halo rows
 * received from the strip below / above (NULL: none, e.g. the edge strips). */
int vfmm_shard_unpack(int64_t n, int levels, int order, int row_lo, int row_hi, int kc, void* workspace,
                      const void* coarse_all, int world, const void* halo_below, const void* halo_above,
                      void* stream);

/* Byte ranges of the multipole pyramid (complex128, all levels) and of the
 * occupancy pyramid (int32, levels 0..l) inside the workspace. */
int vfmm_mult_region(int64_t n, int levels, int order, size_t* offset, size_t* bytes);
int vfmm_counts_region(int64_t n, int levels, int order, size_t* offset, size_t* bytes);

/* Read the device counters of the last evaluate that used `workspace`
 * (synchronises `stream`).  Timings are left at 0.                          */
int vfmm_read_stats(int64_t n, int levels, int order, int kernel, double side,
                    const void* workspace, vfmm_stats* stats, void* stream);

/* Enqueue on `stream` a copy of the out-of-domain particle count of the last
 * evaluate on `workspace` into *host_dst (pinned host memory; valid once the
 * stream has reached this point).  The asynchronous host path uses it so that
 * every result is domain-checked like engine.evaluate (quadtree.py:191-198)
 * without an extra synchronisation.                                         */
int vfmm_bad_count_async(int64_t n, int levels, int order, const void* workspace,
                         int32_t* host_dst, void* stream);

/* engine.evaluate_at (engine.py:401-460): velocity at m arbitrary in-domain
 * targets (tx, ty) from the particle set already processed by the LAST
 * vfmm_evaluate on this workspace (same n, levels, order, kernel, domain).  */
int vfmm_evaluate_at(const double* tx, const double* ty, int64_t m, int64_t n,
                     double xmin, double ymin, double side, int levels, int order, int kernel,
                     double* u, double* v, void* workspace, int64_t* bad_count, void* stream);

/* kernels.velocity_direct (kernels.py:52-94): O(m*n) direct sum in ascending
 * source index order.  Self terms excluded by r^2 > 0.                      */
int vfmm_direct_workspace_size(int64_t m, int64_t n, size_t* bytes);
int vfmm_direct(const double* tx, const double* ty, int64_t m,
                const double* x, const double* y, const double* gamma, const double* sigma,
                int64_t n, int kernel, double* u, double* v, void* workspace,
                size_t workspace_bytes, void* stream);

/* Library self-test helpers (benchmarks): peak FP64 FMA throughput probe.
 * Runs `iters` DFMA chains on `blocks` x 256 threads; returns the number of
 * FP64 flops executed via *flops.  Asynchronous on `stream`.              */
int vfmm_fp64_probe(double* sink, int blocks, int iters, double* flops, void* stream);

/* Total kernel launches issued by this library in this process (host-side
 * counter; CUDA-graph replays are not counted).  While a call is captured
 * into a CUDA graph, the untaken path of a device-side choice (the LSD sort,
 * the generic near field) is put in the body of an IF conditional node that
 * a kernel of the taken path sets; those body launches are not counted.    */
int64_t vfmm_launch_count(void);

/* Phase times of the last replay of a graph captured with
 * VFMM_FLAG_GRAPH_PHASES on `device`: ms[0..7] = elapsed from the call's
 * start to: built, upward, m2l, downward, near joined, end, near start, near
 * end (-1 for an event the call did not record).  Synchronise first.       */
int vfmm_graph_phase_times(int device, float* ms);

/* Version / build string. */
const char* vfmm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* VFMM_H */
