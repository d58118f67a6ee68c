// C ABI entry points (include/vfmm.h): argument validation, workspace layout,
// translation tables, phase sequencing / timing, and the FP64 probe.
//
// vfmm_evaluate mirrors engine.evaluate (engine.py:335-398) phase for phase:
// build (quadtree.py:182-201 + engine.py:355-358), upward (engine.py:114-147),
// m2l (engine.py:150-187), downward (engine.py:190-202), near
// (engine.py:260-285), eval = far field + combine (engine.py:205-213, 394-396).
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <mutex>
#include <vector>

#include "vfmm_internal.cuh"

namespace vfmm {

__device__ Tables g_tables;

static std::atomic<long long> g_launches{0};
// launches captured into the body of a graph conditional node run only when
// the node's condition is set; they are not counted as launches of the call
static thread_local int t_cond_depth = 0;
void note_launches(int k) {
    if (t_cond_depth == 0) g_launches.fetch_add(k, std::memory_order_relaxed);
}
bool pdl_enabled() {
    static const bool on = !(getenv("VFMM_PDL") && getenv("VFMM_PDL")[0] == '0');
    return on;
}

namespace {

constexpr int kMaxDevices = 64;
std::mutex g_mu;
bool g_tables_ready[kMaxDevices];

struct Resources {
    bool ready = false;
    cudaStream_t far = nullptr;   // far-field chain
    cudaStream_t far_hi = nullptr;  // high-priority stream (VFMM_PRIO_M2L A/B)
    cudaStream_t near = nullptr;  // near field
    cudaStream_t comp = nullptr;  // compute stream of host-buffer evaluates
    cudaStream_t lsd = nullptr;   // LSD radix branch of the tree build
    cudaEvent_t lsd_fork = nullptr, lsd_join = nullptr;
    cudaEvent_t fork = nullptr, join_far = nullptr, join_near = nullptr;
    cudaEvent_t xy = nullptr, gs = nullptr, done = nullptr;
    cudaEvent_t ev[9] = {};
    cudaEvent_t gev[9] = {};  // VFMM_FLAG_GRAPH_PHASES: event-record nodes of a captured call
    Counters* hctr = nullptr;  // pinned staging of the device counters (stats)
    // Serialises the calls on this device: the internal streams, events and
    // the pinned counter staging above are shared, so one call enqueues (and,
    // with VFMM_FLAG_STATS, synchronises and reads its counters) at a time.
    // Recursive: a graph capture (evaluate_host_graph) holds it around the
    // evaluate_impl it captures, so no other call touches the shared streams
    // while they are part of the capture.
    std::recursive_mutex mu;
};
Resources g_res[kMaxDevices];

inline size_t align_up(size_t v, size_t a = 256) { return (v + a - 1) / a * a; }

// ---- host-side table construction in long double (64-bit mantissa) ----
struct CLD {
    long double re, im;
};
inline CLD cmul(CLD a, CLD b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }

void build_tables(Tables* t) {
    std::memset(t, 0, sizeof(Tables));
    long double fact[kQMax + 1];
    fact[0] = 1.0L;
    for (int q = 1; q <= kQMax; ++q) fact[q] = fact[q - 1] * (long double)q;
    // H_o[q] = q! tau^{-(q+1)}, tau = -(dx + i dy)
    for (int dy = -3; dy <= 3; ++dy)
        for (int dx = -3; dx <= 3; ++dx) {
            const int o = (dy + 3) * 7 + (dx + 3);
            if ((dx < 0 ? -dx : dx) < 2 && (dy < 0 ? -dy : dy) < 2) continue;
            const long double tr = -(long double)dx, ti = -(long double)dy;
            const long double nrm = tr * tr + ti * ti;
            const CLD inv = {tr / nrm, -ti / nrm};
            CLD pw = inv;  // tau^{-(q+1)}
            for (int q = 0; q < kQMax; ++q) {
                t->H[o][q] = make_double2((double)(pw.re * fact[q]), (double)(pw.im * fact[q]));
                pw = cmul(pw, inv);
            }
        }
    // E_q[j] = d^j / j!,  F_q[j] = (-d)^j / j!,  d = (cx - 1/2) + i (cy - 1/2)
    for (int q = 0; q < 4; ++q) {
        const CLD d = {(q & 1) - 0.5L, (q >> 1) - 0.5L};
        const CLD nd = {-d.re, -d.im};
        CLD pe = {1.0L, 0.0L}, pf = {1.0L, 0.0L};
        for (int j = 0; j < kOrderCap + 16; ++j) {
            t->E[q][j] = make_double2((double)(pe.re / fact[j]), (double)(pe.im / fact[j]));
            t->F[q][j] = make_double2((double)(pf.re / fact[j]), (double)(pf.im / fact[j]));
            pe = cmul(pe, d);
            pf = cmul(pf, nd);
        }
    }
    for (int j = 0; j < kOrderCap + 16; ++j) t->invfact[j] = (double)(1.0L / fact[j]);
    for (int j = 0; j < 2 * kOrderCap + 16; ++j) t->pow2neg[j] = std::ldexp(1.0, -j);
    for (int j = 0; j < kExpTabN; ++j)
        t->exp2tab[j] = (double)exp2l((long double)(j - (kExpTabN - 1)) / (long double)kExpSteps);
    for (int j = 0; j < kExpTab2N; ++j)
        t->exp2tab2[j] = (double)exp2l((long double)(j - (kExpTab2N - 1)) / (long double)kExpSteps2);
}

// Makes the device that owns `p` current for the duration of one C-ABI call
// and restores the caller's current device when the call returns (the
// reference has no device state; a call must not move torch's current
// device).  A host / null pointer keeps the current device.
struct DeviceGuard {
    int prev = -1;
    bool switched = false;
    int bind(const void* p, int* dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) return -1;
        *dev = prev;
        cudaPointerAttributes a;
        if (p && cudaPointerGetAttributes(&a, p) == cudaSuccess && a.type == cudaMemoryTypeDevice) {
            *dev = a.device;
            if (a.device != prev) {
                if (cudaSetDevice(a.device) != cudaSuccess) return -1;
                switched = true;
            }
            return 0;
        }
        cudaGetLastError();
        return 0;
    }
    ~DeviceGuard() {
        if (switched) cudaSetDevice(prev);
    }
};

const Tables* tables_for(int dev) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (dev < 0 || dev >= kMaxDevices) return nullptr;
    if (!g_tables_ready[dev]) {
        Tables* host = new Tables;
        build_tables(host);
        cudaError_t e = cudaMemcpyToSymbol(g_tables, host, sizeof(Tables));
        delete host;
        if (e != cudaSuccess) return nullptr;
        g_tables_ready[dev] = true;
    }
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, g_tables) != cudaSuccess) return nullptr;
    return (const Tables*)p;
}

Resources* resources_for(int dev) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (dev < 0 || dev >= kMaxDevices) return nullptr;
    Resources& r = g_res[dev];
    if (!r.ready) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        // Stream priorities of the two overlapped chains.  Measured (config 2,
        // graph replay): equal 0.813 ms, near first 0.814, far first 0.851 --
        // a prioritised far chain takes SM slots from the FP64-bound near
        // field for latency-bound kernels.  VFMM_STREAM_PRIO=far|equal|near
        // overrides (tuning).
        const char* e = getenv("VFMM_STREAM_PRIO");
        int pf = lo, pn = lo;
        if (e && e[0] == 'f') pf = hi;
        if (e && e[0] == 'n') pn = hi;
        if (cudaStreamCreateWithPriority(&r.far_hi, cudaStreamNonBlocking, hi) != cudaSuccess)
            return nullptr;
        if (cudaStreamCreateWithPriority(&r.far, cudaStreamNonBlocking, pf) != cudaSuccess)
            return nullptr;
        if (cudaStreamCreateWithPriority(&r.near, cudaStreamNonBlocking, pn) != cudaSuccess)
            return nullptr;
        if (cudaStreamCreateWithFlags(&r.comp, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
        if (cudaStreamCreateWithFlags(&r.lsd, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
        cudaEventCreateWithFlags(&r.lsd_fork, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&r.lsd_join, cudaEventDisableTiming);
        if (cudaMallocHost((void**)&r.hctr, sizeof(Counters)) != cudaSuccess) return nullptr;
        cudaEventCreateWithFlags(&r.xy, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&r.gs, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&r.done, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&r.fork, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&r.join_far, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&r.join_near, cudaEventDisableTiming);
        for (auto& e : r.ev) cudaEventCreate(&e);
        for (auto& e : r.gev) cudaEventCreate(&e);
        r.ready = true;
    }
    return &r;
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

double decode_sigma(unsigned long long b) {
    if (b == 0ull) return 0.0;
    const unsigned long long raw = (b & 0x8000000000000000ull) ? (b & ~0x8000000000000000ull) : ~b;
    double d;
    std::memcpy(&d, &raw, sizeof d);
    return d;
}

bool args_ok(int64_t n, int levels, int order, double side, int kernel) {
    return n >= 1 && n < (int64_t)1 << 30 && levels >= 2 && levels <= VFMM_LEVELS_CAP &&
           order >= 0 && order <= VFMM_ORDER_CAP && side > 0.0 && std::isfinite(side) &&
           (kernel == VFMM_KERNEL_POINT || kernel == VFMM_KERNEL_GAUSSIAN);
}

void fill_stats(const Layout& L, const Counters& c, int kernel, double side, vfmm_stats* st) {
    st->n = L.n;
    st->levels = L.levels;
    st->order = L.order;
    st->m2l_count = (int64_t)c.m2l_count;
    st->near_pair_count = (int64_t)c.near_pairs;
    st->bad_count = c.bad_count;
    st->first_bad = c.bad_count ? (int64_t)(INT_MAX - c.first_bad_neg) : -1;
    st->max_sigma = decode_sigma(c.sigma_max_bits);
    // engine.py:362: tree.half_width(levels) / 2 = side / 2^(levels+1) / 2
    st->sigma_guard = side / std::ldexp(1.0, L.levels + 1) / 2.0;
    st->sigma_guard_ok = (kernel == VFMM_KERNEL_GAUSSIAN && st->max_sigma > st->sigma_guard) ? 0 : 1;
}

}  // namespace

bool graph_cond_enabled() {
    static const bool off = getenv("VFMM_GRAPH_COND") && getenv("VFMM_GRAPH_COND")[0] == '0';
    return !off;
}

GraphCond graph_cond_create(cudaStream_t s) {
    GraphCond c;
    if (!graph_cond_enabled()) return c;
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    cudaGraph_t g = nullptr;
    if (cudaStreamGetCaptureInfo(s, &st, nullptr, &g, nullptr, nullptr) != cudaSuccess ||
        st != cudaStreamCaptureStatusActive || !g) {
        cudaGetLastError();
        return c;
    }
    if (cudaGraphConditionalHandleCreate(&c.h, g, 0, cudaGraphCondAssignDefault) != cudaSuccess) {
        cudaGetLastError();
        return c;
    }
    c.on = true;
    return c;
}

namespace {
cudaStream_t g_body_stream[64];
std::mutex g_body_mu;
}  // namespace

cudaStream_t graph_cond_begin(cudaStream_t s, const GraphCond& c, cudaGraphNode_t* node) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaStream_t bs = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_body_mu);
        if (!g_body_stream[dev]) cudaStreamCreateWithFlags(&g_body_stream[dev], cudaStreamNonBlocking);
        bs = g_body_stream[dev];
    }
    cudaStreamCaptureStatus st;
    cudaGraph_t g = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    cudaStreamGetCaptureInfo(s, &st, nullptr, &g, &deps, &nd);
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = c.h;
    p.conditional.type = cudaGraphCondTypeIf;
    p.conditional.size = 1;
    cudaGraphAddNode(node, g, deps, nd, &p);
    cudaStreamBeginCaptureToGraph(bs, p.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                  cudaStreamCaptureModeRelaxed);
    ++t_cond_depth;
    return bs;
}

void graph_cond_end(cudaStream_t s, cudaStream_t body, cudaGraphNode_t node) {
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(body, &g);
    cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies);
    --t_cond_depth;
}

const Tables* device_tables() {
    int dev = 0;
    cudaGetDevice(&dev);
    return tables_for(dev);
}

bool make_layout(int64_t n, int levels, int order, Layout* L) {
    // n < 2^30: 32-bit indices, 30-bit look-back counts in the LSD sort
    if (n < 1 || n >= (1ll << 30) || levels < 2 || levels > VFMM_LEVELS_CAP || order < 0 ||
        order > VFMM_ORDER_CAP)
        return false;
    std::memset(L, 0, sizeof(Layout));
    L->n = n;
    L->levels = levels;
    L->order = order;
    L->P = order + 1;
    L->nleaves = (size_t)1 << (2 * levels);
    const int bits = 2 * levels;
    L->passes = (bits + 7) / 8;
    L->digit_bits = (bits + L->passes - 1) / L->passes;
    const int64_t wc = 2048;  // keys per LSD tile (k_onesweep)
    L->wc = (int)wc;
    L->nchunks = (int)((n + wc - 1) / wc);
    const size_t B = (size_t)1 << L->digit_bits;
    size_t cells = 0;
    for (int k = 2; k <= levels; ++k) {
        L->level_cell_off[k] = cells;
        cells += (size_t)1 << (2 * k);
    }
    L->level_cell_off[levels + 1] = cells;
    size_t cc = 0;
    for (int k = 0; k <= levels; ++k) {
        L->count_off[k] = cc;
        cc += (size_t)1 << (2 * k);
    }
    L->count_off[levels + 1] = cc;
    L->max_tasks = (size_t)((n + 31) / 32) + ((size_t)n < L->nleaves ? (size_t)n : L->nleaves);
    // LSD scratch: global digit histograms, tile tickets, per-pass look-back words
    L->hist_bytes = sizeof(int) * (L->passes * B + 8 + (size_t)L->passes * L->nchunks * B);
    L->scan_state_tiles = scan_tiles((int64_t)L->nleaves + 1);
    // one look-back state per radix pass + the task scan + the leaf-count scan
    L->scan_state_bytes = sizeof(unsigned long long) * (L->scan_state_tiles + 1) * (L->passes + 2);

    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = align_up(off + bytes);
        return o;
    };
    L->counters = take(sizeof(Counters));
    L->key_a = take(sizeof(int) * n);
    L->key_b = take(sizeof(int) * n);
    L->val_a = take(sizeof(int) * n);
    L->val_b = take(sizeof(int) * n);
    L->hist = take(L->hist_bytes);
    L->task_scratch = take(sizeof(int) * L->nleaves);
    L->fill = take(sizeof(int) * L->nleaves);
    L->near_done = take(sizeof(int) * L->nleaves);  // symmetric P2P: writers done per leaf
    L->unperm_cursor = take(sizeof(int) * kUnpermCursorStride * 1025);  // staged un-permute
    L->scan_state = take(L->scan_state_bytes);
    L->src = take(sizeof(Src) * n);
    L->near_uv = take(sizeof(double2) * n * kNearSlotsAlloc);
    L->leaf_starts = take(sizeof(int) * (L->nleaves + 1));
    L->counts = take(sizeof(int) * cc);
    L->mult = take(sizeof(double2) * cells * L->P);
    L->loc = take(sizeof(double2) * cells * L->P);
    L->leaf_loc = take(sizeof(double2) * L->nleaves * L->P);
    L->anc = take(sizeof(double2) * L->level_cell_off[l2l_split_level(levels, L->P)] * L->P);
    L->tasks = take(sizeof(int2) * L->max_tasks);
    L->stage = take(sizeof(double) * 6 * n);  // host-mode staging: x, y, gamma, sigma, u, v
    L->total = off;
    return true;
}

}  // namespace vfmm

namespace vfmm {

__global__ void k_fp64_probe(double* sink, int iters) {
    pdl_enter();
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-3, a2 = a0 + 2e-3, a3 = a0 + 3e-3;
    double a4 = a0 + 4e-3, a5 = a0 + 5e-3, a6 = a0 + 6e-3, a7 = a0 + 7e-3;
    const double b = 0.999999, c = 1e-7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
            a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
        }
    }
    const double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 12345.678) sink[0] = s;  // never true; keeps the chains live
}

}  // namespace vfmm

using namespace vfmm;

extern "C" {

const char* vfmm_version(void) { return "vfmm 0.1.0 sm_100a fp64"; }

int vfmm_workspace_size(int64_t n, int levels, int order, size_t* bytes) {
    Layout L;
    if (!bytes || !make_layout(n, levels, order, &L)) return VFMM_EINVAL;
    *bytes = L.total;
    return VFMM_OK;
}

int vfmm_layout_of(int64_t n, int levels, int order, vfmm_layout* out) {
    Layout L;
    if (!out || !make_layout(n, levels, order, &L)) return VFMM_EINVAL;
    // perm / leaf_key live in whichever ping-pong buffer the last radix pass wrote
    const bool odd = (L.passes & 1) != 0;
    out->perm = odd ? L.val_b : L.val_a;
    out->leaf_key = odd ? L.key_b : L.key_a;
    out->leaf_starts = L.leaf_starts;
    out->sources = L.src;
    out->near_uv = L.near_uv;
    out->mult = L.mult;
    out->loc = L.loc;
    out->leaf_loc = L.leaf_loc;
    out->counts = L.counts;
    out->total = L.total;
    return VFMM_OK;
}

namespace {

// One evaluate (or one phase of a sharded evaluate) over leaf rows [row_lo, row_hi).
// Host-buffer I/O of vfmm_evaluate_host: staged through the workspace.
struct HostIO {
    const double *hx, *hy, *hg, *hs;
    double *hu, *hv;
};

// What PHASE_UP did on a workspace, read by the PHASE_DOWN that follows it.
struct PhaseRecord {
    bool up_done = false;       // a PHASE_UP ran and its PHASE_DOWN has not
    bool near_started = false;  // that PHASE_UP launched the near field (OVERLAP)
    cudaEvent_t join_near = nullptr;
};
std::mutex g_phase_mu;
std::vector<std::pair<const void*, PhaseRecord*>> g_phase;

PhaseRecord* phase_record(const void* ws) {
    std::lock_guard<std::mutex> lk(g_phase_mu);
    for (auto& e : g_phase)
        if (e.first == ws) return e.second;
    PhaseRecord* r = new PhaseRecord;
    if (cudaEventCreateWithFlags(&r->join_near, cudaEventDisableTiming) != cudaSuccess) {
        delete r;
        return nullptr;
    }
    g_phase.emplace_back(ws, r);
    return r;
}

// One evaluate (or one phase of a sharded evaluate) over leaf rows [row_lo, row_hi).
int evaluate_impl(const double* x, const double* y, const double* gamma, const double* sigma,
                  int64_t n, double xmin, double ymin, double side, int levels, int order,
                  int kernel, double* u, double* v, void* workspace, size_t workspace_bytes,
                  unsigned flags, Rows rows, vfmm_stats* stats, void* stream,
                  const HostIO* hio = nullptr, bool sigma_one = false) {
    const bool timed = (flags & VFMM_FLAG_STATS) != 0;
    // one core size for all particles: host mode (VFMM_FLAG_SIGMA_SCALAR) or
    // the device part of a graph-replayed host call (sigma_one)
    const bool sigma_scalar = ((flags & VFMM_FLAG_SIGMA_SCALAR) != 0 && hio != nullptr) || sigma_one;
    const bool far_only = (flags & VFMM_FLAG_FAR_ONLY) != 0;
    bool up = (flags & VFMM_FLAG_PHASE_UP) != 0, down = (flags & VFMM_FLAG_PHASE_DOWN) != 0;
    if (!up && !down) up = down = true;
    // Overlap: the near field runs on a side stream concurrently with the
    // far-field chain.  In a sharded run (separate phases) the near field is
    // launched at the end of PHASE_UP -- it needs only the local tree -- so it
    // also hides the caller's multipole all-reduce; PHASE_DOWN joins it.
    bool overlap = (flags & VFMM_FLAG_OVERLAP) != 0 && !far_only;
    const bool pairs = (flags & VFMM_FLAG_UV_PAIRS) != 0;
    if (pairs) v = nullptr;  // u is an interleaved (N, 2) array
    if (!x || !y || !gamma || (down && !far_only && (!u || (!pairs && !v)))) return VFMM_EINVAL;
    if (kernel == VFMM_KERNEL_GAUSSIAN && !sigma) return VFMM_EINVAL;
    if (timed && !stats) return VFMM_EINVAL;
    if (!args_ok(n, levels, order, side, kernel) || !std::isfinite(xmin) || !std::isfinite(ymin))
        return VFMM_EINVAL;
    if (rows.lo < 0 || rows.hi > (1 << levels) || rows.lo > rows.hi) return VFMM_EINVAL;
    Layout L;
    if (!make_layout(n, levels, order, &L)) return VFMM_EINVAL;
    if (!workspace || workspace_bytes < L.total) return VFMM_EWORKSPACE;
    int dev = 0;
    DeviceGuard dg;
    if (dg.bind(hio ? workspace : (const void*)x, &dev) != 0) return VFMM_ECUDA;
    const Tables* T = tables_for(dev);
    Resources* R = resources_for(dev);
    if (!T || !R) return VFMM_ECUDA;
    std::lock_guard<std::recursive_mutex> call_lock(R->mu);
    // Sharded phases: PHASE_DOWN joins the near field only if PHASE_UP on
    // this workspace started it (recorded per workspace), whatever its own
    // OVERLAP flag says; PHASE_DOWN without a preceding PHASE_UP is invalid.
    PhaseRecord* rec_up = nullptr;
    if (up != down) {
        rec_up = phase_record(workspace);
        if (!rec_up) return VFMM_ECUDA;
        if (down && !rec_up->up_done) return VFMM_EINVAL;
        if (down) overlap = rec_up->near_started;
    }
    cudaStream_t s = (cudaStream_t)stream;
    char* ws = (char*)workspace;
    Counters* ctr = (Counters*)(ws + L.counters);
    Src* src = (Src*)(ws + L.src);
    int* ls = (int*)(ws + L.leaf_starts);
    int* counts = (int*)(ws + L.counts);
    double2* mult = (double2*)(ws + L.mult);
    double2* loc = (double2*)(ws + L.loc);
    double2* near_uv = (double2*)(ws + L.near_uv);
    const bool odd = (L.passes & 1) != 0;
    int* keys = (int*)(ws + (odd ? L.key_b : L.key_a));
    int* perm = (int*)(ws + (odd ? L.val_b : L.val_a));
    // per-phase events only on request; plain stats time the whole call (ev 0 -> 6)
    const bool phases = timed && (flags & VFMM_FLAG_PHASE_TIMES) != 0;
    auto near_field = [&](cudaStream_t st) {  // P2P, then the per-particle near total
        launch_p2p(L, T, src, ls, ws, ctr, kernel, near_uv, rows, keys, st);
    };
    // VFMM_FLAG_GRAPH_PHASES while captured: the phase events become
    // event-record nodes of the graph (read after a replay by
    // vfmm_graph_phase_times), so the phases are timed as the graph runs them
    bool gphases = false;
    if ((flags & VFMM_FLAG_GRAPH_PHASES) && !timed) {
        cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
        gphases = cudaStreamIsCapturing((cudaStream_t)stream, &cst) == cudaSuccess &&
                  cst == cudaStreamCaptureStatusActive;
        cudaGetLastError();
    }
    auto rec = [&](int i, cudaStream_t st) {
        if (gphases)
            cudaEventRecordWithFlags(R->gev[i], st, cudaEventRecordExternal);
        else if (phases || (timed && (i == 0 || i == 6)))
            cudaEventRecord(R->ev[i], st);
    };
    for (int i = 0; i < 9; ++i) rec(i, s);  // every event defined even for a single phase

    // Host mode: x, y are copied first (the keys only need positions); gamma
    // and sigma follow on the copy engine while the sort runs, and only the
    // last radix pass waits for them.  Compute runs on an internal stream.
    cudaStream_t cs = s;
    cudaEvent_t gs_ready = nullptr;
    if (hio) {
        double* st = (double*)(ws + L.stage);
        const size_t b = sizeof(double) * (size_t)n;
        double *dx = st, *dy = st + n, *dg = st + 2 * n, *dsg = st + 3 * n;
        cudaMemcpyAsync(dx, hio->hx, b, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(dy, hio->hy, b, cudaMemcpyHostToDevice, s);
        cudaEventRecord(R->xy, s);
        cudaMemcpyAsync(dg, hio->hg, b, cudaMemcpyHostToDevice, s);
        // VFMM_FLAG_SIGMA_SCALAR: one core size for all (8 bytes instead of 8 N)
        if (hio->hs) cudaMemcpyAsync(dsg, hio->hs, sigma_scalar ? sizeof(double) : b,
                                     cudaMemcpyHostToDevice, s);
        cudaEventRecord(R->gs, s);
        cudaStreamWaitEvent(R->comp, R->xy, 0);
        cs = R->comp;
        gs_ready = R->gs;
        x = dx;
        y = dy;
        gamma = dg;
        sigma = hio->hs ? dsg : nullptr;
        u = st + 4 * n;
        v = pairs ? nullptr : st + 5 * n;
    }

    cudaStream_t fs = cs;
    // VFMM_LSD_BRANCH=1: the LSD radix kernels as a parallel branch of the build
    // (off by default: measured no gain -- config 2 0.7313 vs 0.7317 ms in line)
    static const bool lsd_branch = getenv("VFMM_LSD_BRANCH") && getenv("VFMM_LSD_BRANCH")[0] == '1';
    if (up) {
        if (!hio) rec(0, cs);
        // ---- build: binning, stable sort, pack, leaf starts, occupancy, tasks ----
        // (the counters are zeroed by the build's first kernel)
        launch_build(L, x, y, gamma, kernel == VFMM_KERNEL_GAUSSIAN ? sigma : nullptr, xmin, ymin,
                     side, ws, ctr, cs, &keys, &perm, gs_ready, sigma_scalar ? 0 : 1, rows,
                     lsd_branch ? R->lsd : nullptr, R->lsd_fork, R->lsd_join);
        rec(1, cs);
        // Overlap: the far-field chain and the near field run on two streams
        // (equal priority, see resources_for); P2P CTAs are short-lived, so
        // far-field CTAs are scheduled as soon as SM slots free up.
        if (overlap) {
            cudaEventRecord(R->fork, cs);
            cudaStreamWaitEvent(R->far, R->fork, 0);
            cudaStreamWaitEvent(R->near, R->fork, 0);
            fs = R->far;
        }
        // Head start of the far chain: the near field waits for P2M when the
        // call is captured into a graph, where the generic near-field chain
        // (whose idle launches gave P2M that head start in stream mode) sits
        // in a conditional node.  Measured (config 2, graph replay): no
        // conditional nodes 0.7315 ms (21 launches); conditional nodes 0.7498
        // (13); conditional nodes + near after P2M 0.7334 (13); near after M2M
        // 0.7796.  VFMM_NEAR_AFTER=none|p2m|m2m overrides (A/B).
        static const int near_after_env = [] {
            const char* e = getenv("VFMM_NEAR_AFTER");
            return e ? (e[0] == 'p' ? 1 : (e[0] == 'm' ? 2 : 0)) : -1;
        }();
        int near_after = near_after_env;
        if (near_after < 0) {
            cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
            const bool cap = cudaStreamIsCapturing(cs, &cst) == cudaSuccess && cst == cudaStreamCaptureStatusActive;
            cudaGetLastError();
            near_after = cap && graph_cond_enabled() ? 1 : 0;
        }
        if (overlap && !down) {  // sharded PHASE_UP: start the near field now
            rec(7, R->near);
            near_field(R->near);
            rec(8, R->near);
            cudaEventRecord(rec_up->join_near, R->near);
            fs = cs;  // the far chain stays on the caller's stream (the all-reduce follows it)
        }
        if (rec_up) {
            rec_up->up_done = true;
            rec_up->near_started = overlap;
        }
        // ---- upward ----
        launch_p2m(L, src, ls, xmin, ymin, side, mult + L.level_cell_off[levels] * L.P, T, rows, fs);
        if (overlap && down && near_after == 1) {
            cudaEventRecord(R->lsd_fork, fs);
            cudaStreamWaitEvent(R->near, R->lsd_fork, 0);
        }
        launch_m2m(L, T, mult, rows, fs);
        if (overlap && down && near_after == 2) {
            cudaEventRecord(R->lsd_fork, fs);
            cudaStreamWaitEvent(R->near, R->lsd_fork, 0);
        }
        rec(2, fs);
    }
    bool fuse = false;  // L2P + combine inside the L2L launch (see below)
    // VFMM_PRIO_M2L=1 (A/B): M2L and L2L on a high-priority stream, so they
    // take SM slots as soon as near-field CTAs retire and finish before the
    // near field; the L2P + combine then runs alone after the join
    static const bool prio_m2l = getenv("VFMM_PRIO_M2L") && getenv("VFMM_PRIO_M2L")[0] == '1';
    const bool hp = prio_m2l && overlap && up && down && !far_only;
    if (hp) {
        cudaEventRecord(R->lsd_join, fs);
        cudaStreamWaitEvent(R->far_hi, R->lsd_join, 0);
        fs = R->far_hi;
    }
    if (down) {
        if (!up) rec(2, cs);
        // ---- M2L (all levels, one launch) ----
        launch_m2l(L, T, mult, counts, loc, (double2*)(ws + L.anc), ctr, rows, fs);
        rec(3, fs);
        // ---- downward ----
        // The L2P + combine is fused into the finest L2L level (the
        // near-field totals must be complete first): one launch and one pass
        // over the leaf locals fewer on the critical path.  A sharded
        // PHASE_DOWN joins the near field PHASE_UP started (or runs it now).
        static const bool fuse_env = !(getenv("VFMM_FUSE_L2P") && getenv("VFMM_FUSE_L2P")[0] == '0');
        fuse = fuse_env && !hp && !far_only && levels > 2;
        FusedOut fo{};
        if (fuse && !up) {
            if (overlap) {
                cudaStreamWaitEvent(fs, rec_up->join_near, 0);
            } else {
                rec(7, cs);
                near_field(cs);
                rec(8, cs);
            }
            fo = FusedOut{src, keys, perm, ls, near_uv, u, v, xmin, ymin, side};
        } else if (fuse) {
            if (overlap) {
                rec(7, R->near);
                near_field(R->near);
                rec(8, R->near);
                cudaEventRecord(R->join_near, R->near);
                cudaStreamWaitEvent(fs, R->join_near, 0);
            } else {
                rec(7, cs);
                near_field(cs);
                rec(8, cs);
            }
            fo = FusedOut{src, keys, perm, ls, near_uv, u, v, xmin, ymin, side};
        }
        rec(5, fs);
        // Staged un-permute for large whole-domain calls: decided on the device by the
        // sort path (random input order), see k_unpermute; the records live in the
        // near-field reaction slots 1-2, free once the slot sums are in slot 0.
        static const bool unperm_env = !(getenv("VFMM_UNPERM_STAGED") && getenv("VFMM_UNPERM_STAGED")[0] == '0');
        const bool stage_out = unperm_env && fuse && fo.u && n >= ((int64_t)1 << 22) && rows.lo == 0 &&
                               rows.hi == (1 << levels) && n <= INT32_MAX && l2l_stageable(L);
        if (stage_out) {
            fo.stage = (UnpermRec*)(near_uv + n);
            fo.stage_cursor = (int*)(ws + L.unperm_cursor);
            fo.stage_shift = unperm_shift(n);
            fo.n_total = n;
            fo.ctr = ctr;
            launch_unpermute_prepare(L, fo, fs);
        }
        launch_l2l(L, T, loc, (double2*)(ws + L.leaf_loc), (const double2*)(ws + L.anc), rows, fo,
                   fs);
        if (stage_out) launch_unpermute(L, fo, fs);
        rec(4, fs);
        if (fuse) {
            if (overlap && up) {
                cudaEventRecord(R->join_far, fs);
                cudaStreamWaitEvent(cs, R->join_far, 0);
            }
        } else if (overlap && up) {
            cudaEventRecord(R->join_far, fs);
            rec(7, R->near);
            near_field(R->near);
            rec(8, R->near);
            cudaEventRecord(R->join_near, R->near);
            cudaStreamWaitEvent(cs, R->join_far, 0);
            cudaStreamWaitEvent(cs, R->join_near, 0);
        } else if (overlap) {  // sharded PHASE_DOWN: join the near field started in PHASE_UP
            cudaStreamWaitEvent(cs, rec_up->join_near, 0);
        }
        if (rec_up) rec_up->up_done = false;  // one PHASE_DOWN per PHASE_UP
        if (!far_only && !fuse) {
            if (!overlap) near_field(cs);
            rec(5, cs);
            launch_l2p_combine(L, T, src, keys, perm, (const double2*)(ws + L.leaf_loc), near_uv,
                               xmin, ymin, side, u, v, rows, cs);
        }
    }
    if (hio) {
        // results go back on the CALLER's stream: the internal compute stream
        // is free for the next call at once (pipelined host-buffer calls on
        // distinct streams and workspaces overlap D2H(k) and H2D(k+1) with
        // the compute of k+1)
        cudaEventRecord(R->done, cs);
        cudaStreamWaitEvent(s, R->done, 0);
        const size_t b = sizeof(double) * (size_t)n;
        if (pairs) {
            cudaMemcpyAsync(hio->hu, u, 2 * b, cudaMemcpyDeviceToHost, s);
        } else {
            cudaMemcpyAsync(hio->hu, u, b, cudaMemcpyDeviceToHost, s);
            cudaMemcpyAsync(hio->hv, v, b, cudaMemcpyDeviceToHost, s);
        }
    }
    // the counters ride along on the caller's stream: one synchronisation in all
    if (timed) cudaMemcpyAsync(R->hctr, ctr, sizeof(Counters), cudaMemcpyDeviceToHost, s);
    rec(6, s);
    if (cudaGetLastError() != cudaSuccess) return VFMM_ECUDA;
    if (!timed) return VFMM_OK;

    if (cudaStreamSynchronize(s) != cudaSuccess) return VFMM_ECUDA;
    const Counters c = *R->hctr;
    std::memset(stats, 0, sizeof(*stats));
    fill_stats(L, c, kernel, side, stats);
    stats->overlapped = overlap ? 1 : 0;
    stats->t_total = elapsed(R->ev[0], R->ev[6]);
    if (!phases) return c.bad_count ? VFMM_EDOMAIN : VFMM_OK;
    if (up) {
        stats->t_build = elapsed(R->ev[0], R->ev[1]);
        stats->t_upward = elapsed(R->ev[1], R->ev[2]);
        if (!down && overlap) {  // sharded PHASE_UP: the near field it started
            cudaEventSynchronize(R->ev[8]);
            stats->t_near = elapsed(R->ev[7], R->ev[8]);
        }
    }
    if (down) {
        stats->t_m2l = elapsed(R->ev[2], R->ev[3]);
        stats->t_downward = elapsed(R->ev[3], R->ev[4]);
        if (fuse) {  // t_downward covers L2L + L2P + combine (after the near field)
            stats->t_downward = elapsed(R->ev[5], R->ev[4]);
            stats->t_near = elapsed(R->ev[7], R->ev[8]);
            stats->t_eval = 0.f;
            stats->overlapped = overlap ? 1 : 0;
        } else if (far_only) {
            stats->t_near = 0.f;
            stats->t_eval = 0.f;
        } else if (overlap) {
            stats->t_near = elapsed(R->ev[7], R->ev[8]);
            stats->t_eval = elapsed(R->ev[5], R->ev[6]);
            stats->overlapped = 1;
        } else {
            stats->t_near = elapsed(R->ev[4], R->ev[5]);
            stats->t_eval = elapsed(R->ev[5], R->ev[6]);
        }
    }
    stats->t_total = elapsed(R->ev[up ? 0 : 2], R->ev[6]);
    static const bool tl = getenv("VFMM_DEBUG_TIMELINE") != nullptr;  // tuning aid
    if (tl) {
        static const char* names[9] = {"start", "built", "upward", "m2l", "downward",
                                       "near joined", "end", "near start", "near end"};
        for (int i = 1; i < 9; ++i)
            fprintf(stderr, "vfmm timeline: %-12s %8.4f ms\n", names[i], elapsed(R->ev[0], R->ev[i]));
    }
    return c.bad_count ? VFMM_EDOMAIN : VFMM_OK;
}

}  // namespace

int vfmm_evaluate(const double* x, const double* y, const double* gamma, const double* sigma,
                  int64_t n, double xmin, double ymin, double side, int levels, int order,
                  int kernel, double* u, double* v, void* workspace, size_t workspace_bytes,
                  unsigned flags, vfmm_stats* stats, void* stream) {
    if (levels < 2 || levels > VFMM_LEVELS_CAP) return VFMM_EINVAL;
    return evaluate_impl(x, y, gamma, sigma, n, xmin, ymin, side, levels, order, kernel, u, v,
                         workspace, workspace_bytes, flags & ~(VFMM_FLAG_PHASE_UP | VFMM_FLAG_PHASE_DOWN),
                         Rows{0, 1 << levels}, stats, stream);
}

namespace {

// Cached CUDA graphs of the device part of vfmm_evaluate_host
// (VFMM_FLAG_GRAPH): staged inputs -> staged (u, v).  Everything a graph
// bakes in is part of the key; the graph reads / writes only the workspace.
struct HostGraph {
    int dev;
    const void* ws;
    int64_t n;
    int levels, order, kernel;
    unsigned flags;
    double xmin, ymin, side;
    cudaGraphExec_t exec;
    long long launches;  // kernels per replay
    unsigned long long used;
    // vfmm_evaluate_host_streams: inputs staged (copy stream -> compute stream) and
    // velocities ready (compute stream -> copy stream); one call per workspace in flight
    cudaEvent_t ev_in = nullptr, ev_done = nullptr;
};
std::mutex g_graph_mu;
std::vector<HostGraph> g_graphs;
// Keys seen once: a graph is captured on the SECOND call of a key, so one-off
// shapes (parameter sweeps) do not pay the capture + instantiation (~1 ms).
std::vector<HostGraph> g_graph_seen;
unsigned long long g_graph_tick = 0;
constexpr size_t kMaxGraphs = 32;

// Returns VFMM_OK after enqueueing copies + graph + copies on `s`, or -1 when
// the graph path does not apply (the caller falls back to stream launches).
int evaluate_host_graph(const HostIO& io, int64_t n, double xmin, double ymin, double side,
                        int levels, int order, int kernel, void* workspace,
                        size_t workspace_bytes, unsigned flags, vfmm_stats* stats, void* stream,
                        void* h2d_stream = nullptr, void* d2h_stream = nullptr) {
    const bool timed = (flags & VFMM_FLAG_STATS) != 0;
    if (flags & (VFMM_FLAG_PHASE_TIMES | VFMM_FLAG_PHASE_UP | VFMM_FLAG_PHASE_DOWN |
                 VFMM_FLAG_FAR_ONLY))
        return -1;
    if (!args_ok(n, levels, order, side, kernel) || !std::isfinite(xmin) || !std::isfinite(ymin))
        return VFMM_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cst) != cudaSuccess || cst != cudaStreamCaptureStatusNone) {
        cudaGetLastError();
        return -1;
    }
    Layout L;
    if (!make_layout(n, levels, order, &L)) return VFMM_EINVAL;
    if (!workspace || workspace_bytes < L.total) return VFMM_EWORKSPACE;
    int dev = 0;
    DeviceGuard guard;
    if (guard.bind(workspace, &dev) != 0) return VFMM_ECUDA;
    Resources* R = resources_for(dev);
    if (!R || !tables_for(dev)) return VFMM_ECUDA;
    std::lock_guard<std::recursive_mutex> call_lock(R->mu);  // capture, ev[], hctr
    char* ws = (char*)workspace;
    double* st = (double*)(ws + L.stage);
    double *dx = st, *dy = st + n, *dg = st + 2 * n, *dsg = st + 3 * n, *du = st + 4 * n,
           *dv = st + 5 * n;
    const bool gauss = kernel == VFMM_KERNEL_GAUSSIAN;
    const bool one = gauss && (flags & VFMM_FLAG_SIGMA_SCALAR) != 0;
    const bool pairs = (flags & VFMM_FLAG_UV_PAIRS) != 0;
    // flags of the captured device evaluate (no stats: counters are read after the replay)
    const unsigned dflags = flags & (VFMM_FLAG_OVERLAP | VFMM_FLAG_UV_PAIRS);
    const unsigned kflags = dflags | (one ? VFMM_FLAG_SIGMA_SCALAR : 0u);

    cudaGraphExec_t exec = nullptr;
    cudaEvent_t ev_in = nullptr, ev_done = nullptr;
    long long nl = 0;
    {
        std::lock_guard<std::mutex> lk(g_graph_mu);
        for (auto& g : g_graphs)
            if (g.dev == dev && g.ws == workspace && g.n == n && g.levels == levels &&
                g.order == order && g.kernel == kernel && g.flags == kflags && g.xmin == xmin &&
                g.ymin == ymin && g.side == side) {
                g.used = ++g_graph_tick;
                exec = g.exec;
                nl = g.launches;
                ev_in = g.ev_in;
                ev_done = g.ev_done;
                break;
            }
        if (!exec) {
            bool seen = false;
            for (auto& g : g_graph_seen)
                if (g.dev == dev && g.ws == workspace && g.n == n && g.levels == levels &&
                    g.order == order && g.kernel == kernel && g.flags == kflags && g.xmin == xmin &&
                    g.ymin == ymin && g.side == side)
                    seen = true;
            if (!seen) {
                if (g_graph_seen.size() >= 64) g_graph_seen.erase(g_graph_seen.begin());
                g_graph_seen.push_back(HostGraph{dev, workspace, n, levels, order, kernel, kflags, xmin,
                                                 ymin, side, nullptr, 0, 0});
                return -1;  // stream launches this time
            }
        }
        if (!exec) {
            // capture on the library's compute stream (thread-local mode: other
            // threads' unrelated CUDA calls do not invalidate the capture)
            cudaStream_t cap = R->comp;
            const long long before = g_launches.load();
            if (cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
                cudaGetLastError();
                return -1;
            }
            const int rc = evaluate_impl(dx, dy, dg, gauss ? dsg : nullptr, n, xmin, ymin, side,
                                         levels, order, kernel, du, pairs ? nullptr : dv, workspace,
                                         workspace_bytes, dflags, Rows{0, 1 << levels}, nullptr,
                                         cap, nullptr, one);
            cudaGraph_t graph = nullptr;
            const cudaError_t ec = cudaStreamEndCapture(cap, &graph);
            nl = g_launches.load() - before;
            g_launches.fetch_sub(nl);  // counted per replay instead
            if (rc != VFMM_OK || ec != cudaSuccess || !graph) {
                if (graph) cudaGraphDestroy(graph);
                cudaGetLastError();
                return rc != VFMM_OK ? rc : -1;
            }
            const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
            cudaGraphDestroy(graph);
            if (ei != cudaSuccess) {
                cudaGetLastError();
                return -1;
            }
            if (g_graphs.size() >= kMaxGraphs) {  // evict the least recently used
                size_t lru = 0;
                for (size_t i = 1; i < g_graphs.size(); ++i)
                    if (g_graphs[i].used < g_graphs[lru].used) lru = i;
                cudaGraphExecDestroy(g_graphs[lru].exec);
                if (g_graphs[lru].ev_in) cudaEventDestroy(g_graphs[lru].ev_in);
                if (g_graphs[lru].ev_done) cudaEventDestroy(g_graphs[lru].ev_done);
                g_graphs.erase(g_graphs.begin() + (long)lru);
            }
            if (cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming) != cudaSuccess) {
                cudaGetLastError();
                cudaGraphExecDestroy(exec);
                return -1;
            }
            HostGraph hg{dev, workspace, n, levels, order, kernel, kflags, xmin, ymin, side, exec, nl,
                         ++g_graph_tick};
            hg.ev_in = ev_in;
            hg.ev_done = ev_done;
            g_graphs.push_back(hg);
        }
    }
    // copies on the caller's copy streams when given (vfmm_evaluate_host_streams)
    cudaStream_t sin = h2d_stream ? (cudaStream_t)h2d_stream : s;
    cudaStream_t sout = d2h_stream ? (cudaStream_t)d2h_stream : s;
    if (timed) cudaEventRecord(R->ev[0], s);
    const size_t b = sizeof(double) * (size_t)n;
    cudaMemcpyAsync(dx, io.hx, b, cudaMemcpyHostToDevice, sin);
    cudaMemcpyAsync(dy, io.hy, b, cudaMemcpyHostToDevice, sin);
    cudaMemcpyAsync(dg, io.hg, b, cudaMemcpyHostToDevice, sin);
    if (gauss) cudaMemcpyAsync(dsg, io.hs, one ? sizeof(double) : b, cudaMemcpyHostToDevice, sin);
    if (sin != s) {
        cudaEventRecord(ev_in, sin);
        cudaStreamWaitEvent(s, ev_in, 0);
    }
    if (cudaGraphLaunch(exec, s) != cudaSuccess) return VFMM_ECUDA;
    note_launches((int)nl);
    if (sout != s) {
        cudaEventRecord(ev_done, s);
        cudaStreamWaitEvent(sout, ev_done, 0);
    }
    if (pairs) {
        cudaMemcpyAsync(io.hu, du, 2 * b, cudaMemcpyDeviceToHost, sout);
    } else {
        cudaMemcpyAsync(io.hu, du, b, cudaMemcpyDeviceToHost, sout);
        cudaMemcpyAsync(io.hv, dv, b, cudaMemcpyDeviceToHost, sout);
    }
    if (!timed) return cudaGetLastError() == cudaSuccess ? VFMM_OK : VFMM_ECUDA;
    if (!stats) return VFMM_EINVAL;
    Counters* ctr = (Counters*)(ws + L.counters);
    cudaMemcpyAsync(R->hctr, ctr, sizeof(Counters), cudaMemcpyDeviceToHost, s);
    cudaEventRecord(R->ev[6], s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return VFMM_ECUDA;
    const Counters c = *R->hctr;
    std::memset(stats, 0, sizeof(*stats));
    fill_stats(L, c, kernel, side, stats);
    stats->overlapped = (dflags & VFMM_FLAG_OVERLAP) ? 1 : 0;
    stats->t_total = elapsed(R->ev[0], R->ev[6]);
    return c.bad_count ? VFMM_EDOMAIN : VFMM_OK;
}

}  // namespace

int vfmm_evaluate_host(const double* x, const double* y, const double* gamma, const double* sigma,
                       int64_t n, double xmin, double ymin, double side, int levels, int order,
                       int kernel, double* u, double* v, void* workspace, size_t workspace_bytes,
                       unsigned flags, vfmm_stats* stats, void* stream) {
    if (levels < 2 || levels > VFMM_LEVELS_CAP) return VFMM_EINVAL;
    if (!x || !y || !gamma || !u || (!v && !(flags & VFMM_FLAG_UV_PAIRS)) ||
        (kernel == VFMM_KERNEL_GAUSSIAN && !sigma))
        return VFMM_EINVAL;
    const HostIO io{x, y, gamma, kernel == VFMM_KERNEL_GAUSSIAN ? sigma : nullptr, u, v};
    if (flags & VFMM_FLAG_GRAPH) {
        const int rc = evaluate_host_graph(io, n, xmin, ymin, side, levels, order, kernel,
                                           workspace, workspace_bytes, flags, stats, stream);
        if (rc >= 0) return rc;
    }
    // staging pointers are substituted inside; pass the host ones for the argument checks
    return evaluate_impl(x, y, gamma, sigma, n, xmin, ymin, side, levels, order, kernel, u, v,
                         workspace, workspace_bytes,
                         flags & ~(VFMM_FLAG_PHASE_UP | VFMM_FLAG_PHASE_DOWN | VFMM_FLAG_FAR_ONLY),
                         Rows{0, 1 << levels}, stats, stream, &io);
}

int vfmm_evaluate_host_streams(const double* x, const double* y, const double* gamma,
                               const double* sigma, int64_t n, double xmin, double ymin, double side,
                               int levels, int order, int kernel, double* u, double* v,
                               void* workspace, size_t workspace_bytes, unsigned flags,
                               void* compute_stream, void* h2d_stream, void* d2h_stream) {
    if (levels < 2 || levels > VFMM_LEVELS_CAP) return VFMM_EINVAL;
    if (!x || !y || !gamma || !u || (!v && !(flags & VFMM_FLAG_UV_PAIRS)) ||
        (kernel == VFMM_KERNEL_GAUSSIAN && !sigma))
        return VFMM_EINVAL;
    if ((flags & (VFMM_FLAG_STATS | VFMM_FLAG_PHASE_TIMES | VFMM_FLAG_PHASE_UP | VFMM_FLAG_PHASE_DOWN |
                  VFMM_FLAG_FAR_ONLY)) ||
        !h2d_stream || !d2h_stream || h2d_stream == compute_stream || d2h_stream == compute_stream)
        return VFMM_EINVAL;
    const HostIO io{x, y, gamma, kernel == VFMM_KERNEL_GAUSSIAN ? sigma : nullptr, u, v};
    const int rc = evaluate_host_graph(io, n, xmin, ymin, side, levels, order, kernel, workspace,
                                       workspace_bytes, flags | VFMM_FLAG_GRAPH, nullptr,
                                       compute_stream, h2d_stream, d2h_stream);
    if (rc >= 0) return rc;
    // no graph for this key yet (first sighting) or capture unavailable: the whole call on
    // the compute stream, in stream order with what the copy streams hold; the caller's
    // "complete when d2h_stream reaches this point" still holds
    cudaStream_t cs = (cudaStream_t)compute_stream;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (cudaEventCreateWithFlags(&e0, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&e1, cudaEventDisableTiming) != cudaSuccess) {
        if (e0) cudaEventDestroy(e0);
        cudaGetLastError();
        return VFMM_ECUDA;
    }
    cudaEventRecord(e0, (cudaStream_t)h2d_stream);
    cudaStreamWaitEvent(cs, e0, 0);
    const int rs = evaluate_impl(x, y, gamma, sigma, n, xmin, ymin, side, levels, order, kernel, u, v,
                                 workspace, workspace_bytes, flags & ~VFMM_FLAG_GRAPH,
                                 Rows{0, 1 << levels}, nullptr, compute_stream, &io);
    cudaEventRecord(e1, cs);
    cudaStreamWaitEvent((cudaStream_t)d2h_stream, e1, 0);
    cudaEventDestroy(e0);  // released by the runtime once the recorded work has completed
    cudaEventDestroy(e1);
    return rs;
}

int vfmm_evaluate_shard(const double* x, const double* y, const double* gamma, const double* sigma,
                        int64_t n, double xmin, double ymin, double side, int levels, int order,
                        int kernel, int row_lo, int row_hi, double* u, double* v, void* workspace,
                        size_t workspace_bytes, unsigned flags, vfmm_stats* stats, void* stream) {
    if (levels < 2 || levels > VFMM_LEVELS_CAP) return VFMM_EINVAL;
    return evaluate_impl(x, y, gamma, sigma, n, xmin, ymin, side, levels, order, kernel, u, v,
                         workspace, workspace_bytes, flags, Rows{row_lo, row_hi}, stats, stream);
}

int vfmm_counts_region(int64_t n, int levels, int order, size_t* offset, size_t* bytes) {
    Layout L;
    if (!offset || !bytes || !make_layout(n, levels, order, &L)) return VFMM_EINVAL;
    *offset = L.counts;
    *bytes = sizeof(int) * L.count_off[levels + 1];
    return VFMM_OK;
}

int vfmm_mult_region(int64_t n, int levels, int order, size_t* offset, size_t* bytes) {
    Layout L;
    if (!offset || !bytes || !make_layout(n, levels, order, &L)) return VFMM_EINVAL;
    *offset = L.mult;
    *bytes = sizeof(double2) * L.level_cell_off[levels + 1] * L.P;
    return VFMM_OK;
}

int vfmm_read_stats(int64_t n, int levels, int order, int kernel, double side,
                    const void* workspace, vfmm_stats* stats, void* stream) {
    Layout L;
    if (!stats || !workspace || !make_layout(n, levels, order, &L)) return VFMM_EINVAL;
    int dev = 0;
    DeviceGuard dg;
    if (dg.bind(workspace, &dev) != 0) return VFMM_ECUDA;
    if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) return VFMM_ECUDA;
    Counters c;
    if (cudaMemcpy(&c, (const char*)workspace + L.counters, sizeof c, cudaMemcpyDeviceToHost) !=
        cudaSuccess)
        return VFMM_ECUDA;
    std::memset(stats, 0, sizeof(*stats));
    fill_stats(L, c, kernel, side, stats);
    return c.bad_count ? VFMM_EDOMAIN : VFMM_OK;
}

int vfmm_bad_count_async(int64_t n, int levels, int order, const void* workspace,
                         int32_t* host_dst, void* stream) {
    Layout L;
    if (!workspace || !host_dst || !make_layout(n, levels, order, &L)) return VFMM_EINVAL;
    int dev = 0;
    DeviceGuard dg;
    if (dg.bind(workspace, &dev) != 0) return VFMM_ECUDA;
    const Counters* ctr = (const Counters*)((const char*)workspace + L.counters);
    cudaMemcpyAsync(host_dst, &ctr->bad_count, sizeof(int32_t), cudaMemcpyDeviceToHost,
                    (cudaStream_t)stream);
    return cudaGetLastError() == cudaSuccess ? VFMM_OK : VFMM_ECUDA;
}

int vfmm_evaluate_at(const double* tx, const double* ty, int64_t m, int64_t n, double xmin,
                     double ymin, double side, int levels, int order, int kernel, double* u,
                     double* v, void* workspace, int64_t* bad_count, void* stream) {
    if (!tx || !ty || !u || !v || !workspace || m < 0) return VFMM_EINVAL;
    if (!args_ok(n, levels, order, side, kernel)) return VFMM_EINVAL;
    if (m == 0) {
        if (bad_count) *bad_count = 0;
        return VFMM_OK;
    }
    Layout L;
    if (!make_layout(n, levels, order, &L)) return VFMM_EINVAL;
    int dev = 0;
    DeviceGuard dg;
    if (dg.bind(tx, &dev) != 0) return VFMM_ECUDA;
    const Tables* T = tables_for(dev);
    if (!T) return VFMM_ECUDA;
    cudaStream_t s = (cudaStream_t)stream;
    char* ws = (char*)workspace;
    Counters* ctr = (Counters*)(ws + L.counters);
    launch_init_counters(ctr, s);
    launch_eval_at(L, T, tx, ty, m, (const Src*)(ws + L.src), (const int*)(ws + L.leaf_starts),
                   (const double2*)(ws + L.leaf_loc), xmin, ymin, side, kernel, u, v, ctr, s);
    if (cudaGetLastError() != cudaSuccess) return VFMM_ECUDA;
    if (bad_count) {
        if (cudaStreamSynchronize(s) != cudaSuccess) return VFMM_ECUDA;
        Counters c;
        if (cudaMemcpy(&c, ctr, sizeof c, cudaMemcpyDeviceToHost) != cudaSuccess) return VFMM_ECUDA;
        *bad_count = c.bad_count;
        if (c.bad_count) return VFMM_EDOMAIN;
    }
    return VFMM_OK;
}

int vfmm_direct_workspace_size(int64_t m, int64_t n, size_t* bytes) {
    if (!bytes || m < 0 || n < 0) return VFMM_EINVAL;
    *bytes = (size_t)direct_nsplit(m, n) * (size_t)(m > 0 ? m : 1) * 2 * sizeof(double);
    return VFMM_OK;
}

int vfmm_direct(const double* tx, const double* ty, int64_t m, const double* x, const double* y,
                const double* gamma, const double* sigma, int64_t n, int kernel, double* u,
                double* v, void* workspace, size_t workspace_bytes, void* stream) {
    if (m < 0 || n < 0) return VFMM_EINVAL;
    if (kernel != VFMM_KERNEL_POINT && kernel != VFMM_KERNEL_GAUSSIAN) return VFMM_EINVAL;
    if (m == 0) return VFMM_OK;
    if (!tx || !ty || !u || !v) return VFMM_EINVAL;
    if (n > 0 && (!x || !y || !gamma || (kernel == VFMM_KERNEL_GAUSSIAN && !sigma)))
        return VFMM_EINVAL;
    size_t need = 0;
    vfmm_direct_workspace_size(m, n, &need);
    if (!workspace || workspace_bytes < need) return VFMM_EWORKSPACE;
    int dev = 0;
    DeviceGuard dg;
    if (dg.bind(tx, &dev) != 0) return VFMM_ECUDA;
    const Tables* T = tables_for(dev);
    if (!T) return VFMM_ECUDA;
    const int ns = direct_nsplit(m, n);
    double* pu = (double*)workspace;
    double* pv = pu + (size_t)ns * m;
    launch_direct(tx, ty, m, x, y, gamma, sigma, n, kernel, pu, pv, ns, u, v, T,
                  (cudaStream_t)stream);
    return cudaGetLastError() == cudaSuccess ? VFMM_OK : VFMM_ECUDA;
}

int64_t vfmm_launch_count(void) { return (int64_t)g_launches.load(); }

int vfmm_graph_phase_times(int device, float* ms) {
    if (!ms || device < 0 || device >= kMaxDevices) return VFMM_EINVAL;
    Resources* R = &g_res[device];
    if (!R->ready) return VFMM_EINVAL;
    std::lock_guard<std::recursive_mutex> lk(R->mu);
    for (int i = 1; i < 9; ++i) {
        float t = 0.f;
        if (cudaEventElapsedTime(&t, R->gev[0], R->gev[i]) != cudaSuccess) {
            cudaGetLastError();
            t = -1.f;  // not recorded by the captured call (e.g. a phase it did not run)
        }
        ms[i - 1] = t;
    }
    return VFMM_OK;
}

int vfmm_fp64_probe(double* sink, int blocks, int iters, double* flops, void* stream) {
    if (!sink || blocks < 1 || iters < 1) return VFMM_EINVAL;
    int dev = 0;
    DeviceGuard dg;
    if (dg.bind(sink, &dev) != 0) return VFMM_ECUDA;
    launch_k(k_fp64_probe, blocks, 256, 0, (cudaStream_t)stream, sink, iters);
    note_launches(1);
    if (flops) *flops = (double)blocks * 256.0 * (double)iters * 32.0 * 2.0;
    return cudaGetLastError() == cudaSuccess ? VFMM_OK : VFMM_ECUDA;
}

}  // extern "C"
