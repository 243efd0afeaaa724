// cg_api.cu -- extern "C" entry points of libcodegemm_b200.so (include/codegemm_b200.h).
//
// The layer handle owns the device-resident prepacked weights (uploaded once,
// weights are static), a split-K workspace and pinned staging buffers for the
// host-buffer entry point.  Validation mirrors the reference exactly:
//   QuantConfig / validate_shape  (quantizer.py:35-84)      -> CG_ERR_CONFIG
//   code range                    (quantizer.py:181-182)    -> CG_ERR_INTEGRITY
//   q.cols != x.rows              (engines.py:184-186)      -> CG_ERR_SHAPE (n < 1 here)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/codegemm_b200.h"
#include "cg_batch.h"
#include "cg_internal.h"

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(CG_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

#define CG_CUDA(call, what)                                 \
    do {                                                    \
        cudaError_t _e = (call);                            \
        if (_e != cudaSuccess) return cuda_fail(_e, what);  \
    } while (0)

int sm_count_of(int device) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || n < 1)
        return 148;
    return n;
}

bool pow2(int64_t x) { return x > 0 && (x & (x - 1)) == 0; }

int ilog2(int64_t x) {
    int r = 0;
    while ((1LL << r) < x) ++r;
    return r;
}

// Scale-group constraint of the fused kernel for segments-per-lane u: returns
// lg = log2(lanes sharing one scale group) or -1 when a lane's u segments
// would straddle groups / slices would straddle groups.
int scale_lg(const cg::Plan& p, int u) {
    if (p.g_row) return 5;
    const int64_t lane_elems = (int64_t)u * p.v, slice_elems = 32 * lane_elems;
    if (p.g_eff >= slice_elems) return (p.g_eff % slice_elems == 0) ? 5 : -1;
    if (p.g_eff % lane_elems != 0 || slice_elems % p.g_eff != 0) return -1;
    const int64_t lanes = p.g_eff / lane_elems;
    if (!pow2(lanes)) return -1;
    // >= 8 lanes: the gather scales two slots after three halvings; 1, 2 or 4
    // lanes: all 16 slots of a lane before the reduction
    return ilog2(lanes);
}

// Raw task inputs staged by bulk copy: binary16 codebooks, then (16-byte
// aligned) the binary16 x slice of one task.
int raw_books_bytes(const cg::Plan& p) { return (p.m * p.kcount * p.v * 2 + 15) / 16 * 16; }
// raw task-input buffer: codebooks, then the x slice (binary16, or binary32 for a
// staged-chain input read by bulk copy)
int raw_input_bytes(const cg::Plan& p, int u, int x_elem_bytes = 2) {
    return raw_books_bytes(p) + 32 * u * p.v * x_elem_bytes;
}
// fix-up list entries (deterministic) or the split-K staging rows (reduce-add)
int list_bytes_for(int64_t rg_per_task, int n) {
    // (>= 512: the kernel prologue lists the CTA's tasks through 128 ints of it)
    return (int)std::max<int64_t>(std::max((rg_per_task * n + 16) * 16, rg_per_task * 16 * n * 4), 512);
}

// Planner: pick u (segments per lane) and rows per task for the fused kernel.
// Cost model per SM, in shared-memory wavefronts (the co-bound with HBM):
//   gather  = rows/16 * 16*(u*m + 1)   (one LDS per lookup + SHFL reduction)
//   build   = m*u*2**kb                (STS.128 of the slice tables)
// with tasks = n_slices * n_rb spread over the SMs (1 CTA/SM at >=114 KB smem).
void plan_fast(cg::Plan& p, int force_u, int force_rg, int sms, int reserved) {
    p.fast = false;
    if (p.b > 8 || p.m > 4 || !(p.v == 2 || p.v == 4 || p.v == 8 || p.v == 16)) return;
    // table / code-stream class: 16 entries + nibbles (b <= 4); 64 entries + 6-bit
    // stream (b = 5, 6 where instantiated: v = 4, m = 1, u = 4); else 256 + bytes
    p.kbits = p.b <= 4 ? 4 : 8;
    if ((p.b == 5 || p.b == 6) && (force_u == 0 || force_u == 4) && cg::fused_instantiated(p.v, p.m, 4, 6) &&
        scale_lg(p, 4) >= 0)
        p.kbits = 6;
    double best = 1e300;
    const int us[3] = {4, 2, 1};
    for (int ui = 0; ui < 3; ++ui) {
        const int u = us[ui];
        if (force_u && u != force_u) continue;
        if (!cg::fused_instantiated(p.v, p.m, u, p.kbits)) continue;
        const int lg = scale_lg(p, u);
        if (lg < 0) continue;
        const int64_t slice_segs = 32LL * u;
        const int64_t n_slices = (p.segs + slice_segs - 1) / slice_segs;
        const int64_t n_rg = (p.rows + 15) / 16;
        cg::FusedSizes z;
        if (!cg::fused_sizes(p.v, p.m, u, p.kbits, &z)) continue;
        const int n_gs = 32 >> lg;
        const int raw_bytes = raw_input_bytes(p, u);
        // rows per task are capped by the smem left for the task's scale tiles;
        // the cap holds for staged launches too, whose x may be binary32
        const int raw_cap_bytes = raw_input_bytes(p, u, 4);
        int64_t rg_cap = 0;
        {
            cg::SmemLayout lay;
            int64_t lo = 0, hi = 1 << 16;
            while (lo < hi) {  // largest rg count whose layout fits
                const int64_t mid = (lo + hi + 1) / 2;
                if (cg::smem_layout(z, (int)(mid * n_gs * 32), raw_cap_bytes,
                                    list_bytes_for(mid, 1), reserved, &lay, (int)(mid * 64)))
                    lo = mid;
                else hi = mid - 1;
            }
            rg_cap = lo;
        }
        if (rg_cap < 1) continue;
        const int occ = 1;  // 512 threads x 128 registers: one CTA per SM
        int64_t rg_per_task;
        if (force_rg) {
            rg_per_task = force_rg;
        } else {
            // fill exactly one wave: tasks = n_slices * n_rb <= sms * occ
            const int64_t want_tasks = (int64_t)sms * occ;
            int64_t n_rb = std::max<int64_t>(1, want_tasks / n_slices);
            rg_per_task = std::max<int64_t>(1, (n_rg + n_rb - 1) / n_rb);
        }
        if (rg_per_task > rg_cap) {
            if (force_rg) continue;
            rg_per_task = rg_cap;
        }
        const int64_t n_rb = (n_rg + rg_per_task - 1) / rg_per_task;
        const int64_t tasks = n_slices * n_rb;
        cg::SmemLayout lay;
        cg::smem_layout(z, (int)(rg_per_task * n_gs * 32), raw_bytes,
                        list_bytes_for(rg_per_task, 1), reserved, &lay, (int)(rg_per_task * 64));
        const double per_task = (double)rg_per_task * 16.0 * (u * p.m + 1) +
                                (double)p.m * u * (1 << p.kbits) + 600.0;
        const double waves = std::ceil((double)tasks / ((double)sms * occ));
        const double cost = waves * per_task * occ;
        if (cost < best) {
            best = cost;
            p.fast = true;
            p.rg_cap = (int)rg_cap;
            p.u = u;
            p.lg = lg;
            p.n_gs = 32 >> lg;
            p.slice_segs = slice_segs;
            p.n_slices = n_slices;
            p.rows_pad = n_rg * 16;
            p.n_rg = n_rg;
            p.rg_per_task = (int)rg_per_task;
            p.n_rb = n_rb;
            p.smem = lay;
            p.smem_bytes = lay.total;
        }
    }
    if (p.fast) {
        // one byte per code, or two per byte for 16-entry tables (b <= 4)
        p.code_bytes = p.n_slices * p.n_rg * (int64_t)p.m * 16 * p.slice_segs * p.kbits / 8;
        p.scale_bytes = p.n_slices * p.n_rg * (int64_t)p.n_gs * 16 * 2;
    }
}

}  // namespace

struct cg_layer {
    cg::Plan plan;
    int device = 0;
    uint8_t* codes = nullptr;       // fast layout (plan.fast)
    uint16_t* raw16 = nullptr;      // (m, rows, segs) when no fast layout
    uint16_t* scl = nullptr;        // prepacked scale tiles (fast)
    uint16_t* scales = nullptr;     // (rows, groups) binary16
    uint16_t* books = nullptr;      // (m, 2**b, v) binary16
    float* ws = nullptr;            // split-K workspace (n_slices, rows, ws_cols)
    unsigned long long* tickets = nullptr;  // split-K tickets (n_rg, ws_cols), monotonic
    unsigned long long* grid_flags = nullptr;  // per-CTA barrier flags of launches led by this layer
    unsigned long long* rg_cnt = nullptr;      // row-group readiness counters (producer layer)
    int ws_cols = 0;
    int reserved = 1024;            // driver-reserved smem at the start of the CTA window
    uint16_t* x_dev = nullptr;      // staging for the host entry point
    float* y_dev = nullptr;
    int stage_cols = 0;
    uint16_t* x_pin = nullptr;
    float* y_pin = nullptr;
    int flags = 0;
    int pf_dist = 2;  // L2 prefetch window in rounds of row groups (measured best: 2)
    int sms = 148;
    bool rg_forced = false;  // rg_per_task given at creation: launches keep the task split
    int rg_cap = 0;          // largest rows-per-task whose task buffers fit shared memory (n=1)
    unsigned long long* stamps = nullptr;  // diagnostics (CG_STAMPS=1)
    int64_t device_bytes = 0;
    float2* llp = nullptr;          // LL-chain partials (n_slices, rows) of this layer's y
    int64_t llp_bytes = 0;
    // batch path (K4, n >= 2): its code stream, built on first use, and the
    // split-K partial planes
    bool batch_ok = false;          // config has a batch kernel
    uint8_t* bcodes = nullptr;
    uint16_t* bscl = nullptr;
    float* bws = nullptr;
    int64_t bws_bytes = 0;
};

// One rank's row-shard exchange region (cg_comm_*): a header of counters and
// barrier flags (cg::kXc*), then `bytes` of gathered buffers; the peers' regions
// mapped into this process (CUDA IPC) or, for ranks of one process, given directly.
struct cg_comm {
    int world = 1, rank = 0, ctas = 0, device = 0;
    unsigned char* base = nullptr;  // cudaMalloc: header + data
    int64_t bytes = 0;              // data bytes after the header
    unsigned char* peer[cg::kMaxRanks] = {nullptr};
    bool ipc[cg::kMaxRanks] = {false};  // peer[r] opened with cudaIpcOpenMemHandle
    bool linked = false;
    unsigned long long timeout_ns = 0;
};

namespace {

template <typename T>
int dev_alloc(cg_layer* L, T** p, size_t bytes, const char* what) {
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), bytes);
    if (e != cudaSuccess) return cuda_fail(e, what);
    L->device_bytes += (int64_t)bytes;
    return CG_OK;
}

void free_layer(cg_layer* L) {
    if (!L) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(L->device);
    cudaFree(L->codes);
    cudaFree(L->raw16);
    cudaFree(L->scl);
    cudaFree(L->scales);
    cudaFree(L->books);
    cudaFree(L->ws);
    cudaFree(L->tickets);
    cudaFree(L->grid_flags);
    cudaFree(L->rg_cnt);
    cudaFree(L->stamps);
    cudaFree(L->llp);
    cudaFree(L->bcodes);
    cudaFree(L->bscl);
    cudaFree(L->bws);
    cudaFree(L->x_dev);
    cudaFree(L->y_dev);
    cudaFreeHost(L->x_pin);
    cudaFreeHost(L->y_pin);
    cudaSetDevice(prev);
    delete L;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

int ensure_ws(cg_layer* L, int n) {
    const cg::Plan& p = L->plan;
    if (!p.fast || p.n_slices <= 1 || n <= L->ws_cols) return CG_OK;
    if (L->ws) {
        cudaFree(L->ws);
        cudaFree(L->tickets);
        L->device_bytes -= (int64_t)p.n_slices * p.rows * L->ws_cols * 4 + p.n_rg * L->ws_cols * 8;
        L->ws = nullptr;
        L->tickets = nullptr;
        L->ws_cols = 0;  // (a failed reallocation below must not leave a stale width)
    }
    int rc = dev_alloc(L, &L->ws, (size_t)p.n_slices * p.rows * n * 4, "workspace alloc");
    if (rc) return rc;
    // one monotonic ticket per (row group, column): +n_slices per call
    rc = dev_alloc(L, &L->tickets, (size_t)p.n_rg * n * 8, "ticket alloc");
    if (rc) return rc;
    cudaError_t e = cudaMemset(L->tickets, 0, (size_t)p.n_rg * n * 8);
    if (e != cudaSuccess) return cuda_fail(e, "ticket init");
    L->ws_cols = n;
    return CG_OK;
}

cg::LayerTask task_of(const cg_layer* L, const uint16_t* x, float* y) {
    const cg::Plan& p = L->plan;
    cg::LayerTask t{};
    t.codes = L->codes;
    t.scl = L->scl;
    t.books = L->books;
    t.x = x;
    t.y = y;
    t.ws = L->ws;
    t.tickets = L->tickets;
    t.rows = p.rows;
    t.cols = p.cols;
    t.n_rg = p.n_rg;
    t.n_slices = p.n_slices;
    t.n_rb = p.n_rb;
    t.u = p.u;
    t.rg_per_task = p.rg_per_task;
    t.lg = p.lg;
    t.n_gs = p.n_gs;
    t.kcount = p.kcount;
    t.n_tasks = (int)(p.n_slices * p.n_rb);
    return t;
}

// One launch of the fused kernel for `count` layers (all fast, same v/m/kbits/device),
// stages[i] = dependency stage of layer i (non-decreasing; NULL = all stage 0).
// A planned staged launch: the kernel parameters and launch configuration.
struct StagedPlan {
    cg::GroupParams gp;
    int grid = 0, smem = 0;
    bool pdl = true;
    int v = 0, m = 0, u = 0, kbits = 0;
};

int plan_stages(cg_layer* const* layers, const uint16_t* const* xs, float* const* ys,
                const int* stages, int count, int n, const int* x_dtypes, const int* xchg,
                cg_comm* comm, StagedPlan* out, bool allow_llc = true) {
    if (count < 1 || count > cg::kMaxGroup)
        return fail(CG_ERR_ARG, "group size %d outside 1..%d", count, cg::kMaxGroup);
    const cg::Plan& p0 = layers[0]->plan;
    cg::GroupParams gp{};
    gp.n_layers = count;
    gp.n = n;
    gp.flags = (layers[0]->flags & CG_OPT_NO_L2_PREFETCH) ? cg::kFlagNoPrefetch : 0;
    gp.pf_dist = layers[0]->pf_dist;
    if (const char* e = std::getenv("CG_PF_DIST")) gp.pf_dist = std::atoi(e);  // tuning knob
    gp.stamps = layers[0]->stamps;
    cg::FusedSizes zmax{0, 0, 0};
    int scl_max = 0, rg_max = 0, grid = 1, raw_bytes = 0, books_raw = 0;
    bool x_copy = (n == 1) && !std::getenv("CG_X_REGS");
    int prev_stage = 0;
    for (int i = 0; i < count; ++i) {
        cg_layer* L = layers[i];
        const cg::Plan& p = L->plan;
        if (!p.fast) return fail(CG_ERR_UNSUPPORTED, "layer %d has no fused kernel", i);
        if (p.v != p0.v || p.m != p0.m || p.kbits != p0.kbits || p.u != p0.u ||
            L->device != layers[0]->device)
            return fail(CG_ERR_CONFIG, "staged launch layers must share v, m, u, code width and device");
        const int st = stages ? stages[i] : 0;
        if (st < prev_stage || st > prev_stage + 1 || (i == 0 && st != 0))
            return fail(CG_ERR_ARG, "stages must start at 0 and grow by at most 1 (layer %d: %d)",
                        i, st);
        prev_stage = st;
        int rc = ensure_ws(L, n);
        if (rc) return rc;
        // the split-K flush is a bulk reduce-add into y: 16-byte aligned rows
        if (reinterpret_cast<uintptr_t>(ys[i]) & 15)
            return fail(CG_ERR_ARG, "y of layer %d is not 16-byte aligned", i);
        gp.layer[i] = task_of(L, xs[i], ys[i]);
        gp.layer[i].stage = st;
        if (x_dtypes && x_dtypes[i] == CG_X_F32) {
            gp.layer[i].x = nullptr;
            gp.layer[i].x32 = reinterpret_cast<const float*>(xs[i]);
        } else if (x_dtypes && x_dtypes[i] != CG_X_F16) {
            return fail(CG_ERR_ARG, "x_dtypes[%d] = %d is not CG_X_F16 / CG_X_F32", i, x_dtypes[i]);
        }
        cg::FusedSizes z;
        cg::fused_sizes(p.v, p.m, p.u, p.kbits, &z);
        zmax.psum = std::max(zmax.psum, z.psum);
        zmax.books = std::max(zmax.books, z.books);
        zmax.x = std::max(zmax.x, z.x);
        raw_bytes = std::max(raw_bytes, raw_input_bytes(p, p.u, (x_dtypes && x_dtypes[i] == CG_X_F32) ? 4 : 2));
        books_raw = std::max(books_raw, raw_books_bytes(p));
        // x travels by bulk copy only if every slice of it is a 16-byte multiple
        if ((reinterpret_cast<uintptr_t>(xs[i]) & 15) || (p.cols % 8)) x_copy = false;
    }
    gp.n_stages = prev_stage + 1;
    // An x must not overlap a y written in its own stage or later: split-K outputs
    // are zeroed by every CTA at launch start (before stage 0 reads its x) and a
    // same-stage y is written while x is read.  Only an earlier stage's y may be
    // read (the staged chain).
    for (int i = 0; i < count; ++i) {
        const int64_t xe = (x_dtypes && x_dtypes[i] == CG_X_F32) ? 4 : 2;
        const uintptr_t x0 = reinterpret_cast<uintptr_t>(xs[i]);
        const uintptr_t x1 = x0 + (uintptr_t)(layers[i]->plan.cols * n * xe);
        for (int j = 0; j < count; ++j) {
            const uintptr_t y0 = reinterpret_cast<uintptr_t>(ys[j]);
            const uintptr_t y1 = y0 + (uintptr_t)(layers[j]->plan.rows * n * 4);
            if (x0 < y1 && y0 < x1 && gp.layer[j].stage >= gp.layer[i].stage)
                return fail(CG_ERR_ARG,
                            "x of layer %d overlaps y of layer %d, which is written in the same or "
                            "a later stage (outputs are zeroed at launch start)", i, j);
        }
    }
    // ---- row-shard exchange: pushed y / gathered x must lie in the comm region
    if (comm) {
        if (!comm->linked) return fail(CG_ERR_ARG, "comm peers not opened / set");
        if (comm->device != layers[0]->device)
            return fail(CG_ERR_ARG, "comm and layers are on different devices");
        const uintptr_t lo = reinterpret_cast<uintptr_t>(comm->base) + cg::kXcHeader;
        const uintptr_t hi = lo + (uintptr_t)comm->bytes;
        for (int i = 0; i < count; ++i) {
            const int f = xchg ? xchg[i] : 0;
            if (f & ~(cg::kXchgPush | cg::kXchgWait))
                return fail(CG_ERR_ARG, "xchg[%d] = %d: unknown bits", i, f);
            cg::LayerTask& t = gp.layer[i];
            t.xchg = f;
            if (f & cg::kXchgPush) {
                const uintptr_t a = reinterpret_cast<uintptr_t>(t.y);
                if (a < lo || a + (uintptr_t)(t.rows * n * 4) > hi)
                    return fail(CG_ERR_ARG, "layer %d: pushed y is not inside the comm buffer", i);
            }
            if (f & cg::kXchgWait) {
                const uintptr_t a = reinterpret_cast<uintptr_t>(t.x32);
                if (!t.x32 || a < lo || a + (uintptr_t)(t.cols * n * 4) > hi)
                    return fail(CG_ERR_ARG,
                                "layer %d: gathered x must be CG_X_F32 inside the comm buffer", i);
            }
        }
        // LL stage exchange: every later-stage x inside the gathered buffers must be
        // the gathered y of a layer pushed in an earlier stage of this launch (its
        // range contains that layer's local rows); else the fenced per-stage protocol
        {
            bool ll = !std::getenv("CG_XC_LL") || std::atoi(std::getenv("CG_XC_LL")) != 0;
            for (int i = 0; i < count; ++i) {
                cg::LayerTask& t = gp.layer[i];
                t.xll = 0;
                const uintptr_t xa = reinterpret_cast<uintptr_t>(t.x32);
                if (!t.x32 || (t.xchg & cg::kXchgWait) || xa < lo || xa >= hi) continue;
                const uintptr_t xe = xa + (uintptr_t)(t.cols * n * 4);
                bool found = false;
                for (int j = 0; j < count && !found; ++j) {
                    const cg::LayerTask& u = gp.layer[j];
                    const uintptr_t ya = reinterpret_cast<uintptr_t>(u.y);
                    found = (u.xchg & cg::kXchgPush) && u.stage < t.stage && ya >= xa &&
                            ya + (uintptr_t)(u.rows * n * 4) <= xe;
                }
                if (found) t.xll = 1;
                else ll = false;
            }
            if (ll) {
                gp.flags |= cg::kFlagXcLL;
            } else {
                for (int i = 0; i < count; ++i) gp.layer[i].xll = 0;
            }
            gp.xc_gbase = comm->base + cg::kXcHeader;
            gp.xc_ll = comm->base + cg::kXcHeader + comm->bytes;
        }
        gp.xc_local = comm->base;
        gp.xc_world = comm->world;
        gp.xc_rank = comm->rank;
        gp.xc_timeout_ns = comm->timeout_ns;
        for (int r = 0; r < comm->world; ++r) {
            gp.xc_peer[r] = comm->peer[r];
            gp.xc_delta[r] = (long long)(reinterpret_cast<intptr_t>(comm->peer[r]) -
                                         reinterpret_cast<intptr_t>(comm->base));
        }
    } else if (xchg) {
        for (int i = 0; i < count; ++i)
            if (xchg[i]) return fail(CG_ERR_ARG, "xchg[%d] set without a comm", i);
    }
    // ---- dependencies (optional): a layer whose x IS an earlier stage's y (same
    //      pointer, float32, matching shape) waits for the row groups it reads
    //      instead of a grid barrier.  Only when every later-stage layer's x is either
    //      such a y or not written in this launch; never in deterministic mode
    //      (the owner sums complete rows later than the tasks).
    {
        // (opt-in, CG_ROW_DEPS=1: measured slower than the grid barrier on the 8B
        // block -- 44.8 vs 41.5 us -- the per-dependency fence and polling cost
        // more than one barrier; kept for the row-local chains of later rounds)
        const char* rd = std::getenv("CG_ROW_DEPS");
        bool ok = gp.n_stages > 1 && !(layers[0]->flags & CG_OPT_DETERMINISTIC) && rd &&
                  std::atoi(rd) != 0 && !comm;
        for (int i = 0; i < count; ++i) gp.layer[i].dep = -1;
        for (int i = 0; ok && i < count; ++i) {
            cg::LayerTask& t = gp.layer[i];
            const void* xp = t.x32 ? (const void*)t.x32 : (const void*)t.x;
            for (int j = 0; j < count; ++j) {
                const bool alias = (const void*)gp.layer[j].y == xp;
                if (!alias) continue;
                if (j < i && gp.layer[j].stage < t.stage && t.x32 && gp.layer[j].rows == t.cols)
                    t.dep = j;
                else
                    ok = false;  // an aliasing we do not track: keep the barriers
            }
        }
        for (int i = 0; ok && i < count; ++i)
            for (int j = i + 1; ok && j < count; ++j)
                if (layers[i] == layers[j] || gp.layer[i].y == gp.layer[j].y) ok = false;
        if (ok) {
            gp.flags |= cg::kFlagRowDeps;
            for (int i = 0; i < count; ++i)
                if (gp.layer[i].dep >= 0) gp.layer[gp.layer[i].dep].rg_cnt = layers[gp.layer[i].dep]->rg_cnt;
        } else {
            for (int i = 0; i < count; ++i) gp.layer[i].dep = -1;
        }
    }
    // ---- LL chain (single GPU, batch 1, non-deterministic launches; CG_LL_CHAIN=0
    //      disables): a later-stage x that is an earlier stage's y (same pointer
    //      and length), produced in at most CG_LL_MAX_SLICES (32) K-slices, is read
    //      as the sum of the producer's (value, epoch) partials -- the zeroing and
    //      reduce-add of that y go away, and so does the grid barrier before the
    //      consumer's stage when all its aliased inputs come this way.  (Wider
    //      producers cost the consumer more spinning loads than a barrier.  A/B on
    //      one box: limit 8 -> 32 takes the 8B down -> next q,k,v (28 slices) and
    //      every 70B stage (16 slices) off the barrier: 8B block 38.72 -> 38.36 us,
    //      70B 91.3 -> 88.9 us; 64 (the 70B down too) gains nothing more.)  Any
    //      other alias of an output keeps the barriers.
    for (int i = 0; i < count; ++i) {
        gp.layer[i].llx = -1;
        gp.layer[i].llw = 0;
        gp.layer[i].llp = nullptr;
    }
    {
        const char* ev = std::getenv("CG_LL_CHAIN");
        const char* em = std::getenv("CG_LL_MAX_SLICES");
        const int64_t max_slices = em ? std::atoi(em) : 32;
        bool llc = allow_llc && !comm && n == 1 && gp.n_stages > 1 &&
                   !(layers[0]->flags & CG_OPT_DETERMINISTIC) && !(gp.flags & cg::kFlagRowDeps) &&
                   !(ev && std::atoi(ev) == 0);
        int nprod = 0;
        for (int i = 0; llc && i < count; ++i) {
            cg::LayerTask& t = gp.layer[i];
            int src = -1;
            for (int j = 0; t.x32 && j < count; ++j)
                if (gp.layer[j].y == t.x32 && gp.layer[j].stage < t.stage && gp.layer[j].rows == t.cols)
                    src = j;
            if (src >= 0 && gp.layer[src].n_slices > max_slices) src = -2;  // barrier path
            if (src == -2) continue;
            if (src < 0) {  // an x that is not an earlier stage's whole y must not touch any y
                const uintptr_t xa = t.x32 ? reinterpret_cast<uintptr_t>(t.x32)
                                           : reinterpret_cast<uintptr_t>(t.x);
                const uintptr_t xb = xa + (uintptr_t)(t.cols * (t.x32 ? 4 : 2));
                for (int j = 0; j < count; ++j) {
                    const uintptr_t ya = reinterpret_cast<uintptr_t>(gp.layer[j].y);
                    if (xa < ya + (uintptr_t)(gp.layer[j].rows * 4) && ya < xb) llc = false;
                }
                continue;
            }
            t.llx = src;
            ++nprod;
        }
        // a producer's partial planes and epoch live in its cg_layer: one use per launch
        for (int i = 0; llc && i < count; ++i)
            for (int j = 0; j < count; ++j)
                if (j != i && gp.layer[j].llx >= 0 && layers[i] == layers[gp.layer[j].llx] &&
                    i != gp.layer[j].llx)
                    llc = false;
        if (llc && nprod > 0) {
            for (int i = 0; i < count; ++i) {
                cg::LayerTask& t = gp.layer[i];
                if (t.llx < 0) continue;
                cg::LayerTask& P = gp.layer[t.llx];
                cg_layer* PL = layers[t.llx];
                if (!P.llp) {
                    // the producer's partial planes, zero-filled once (epoch 0 never matches)
                    const int64_t bytes = PL->plan.n_slices * PL->plan.rows * 8;
                    if (bytes > PL->llp_bytes) {
                        cudaFree(PL->llp);
                        PL->device_bytes -= PL->llp_bytes;
                        PL->llp = nullptr;
                        PL->llp_bytes = 0;
                        int rc = dev_alloc(PL, &PL->llp, (size_t)bytes, "LL-chain partials alloc");
                        if (rc) return rc;
                        cudaMemset(PL->llp, 0, (size_t)bytes);
                        PL->llp_bytes = bytes;
                    }
                    P.llp = PL->llp;
                    P.rg_cnt = PL->rg_cnt;  // its launch generation: the epoch
                    t.llw = 1;              // the first consumer writes the reduced y
                }
            }
            gp.flags |= cg::kFlagLLChain;
            // the barrier before stage t stays if a stage-t layer reads an earlier
            // stage's y the ordinary way (every alias is a whole earlier y here)
            unsigned skip = 0;
            for (int st = 0; st + 1 < gp.n_stages; ++st) {
                bool need = false;
                for (int i = 0; i < count; ++i) {
                    const cg::LayerTask& t = gp.layer[i];
                    if (t.stage != st + 1 || t.llx >= 0 || !t.x32) continue;
                    for (int j = 0; j < count; ++j)
                        if (gp.layer[j].y == t.x32 && gp.layer[j].stage <= st) need = true;
                }
                if (!need) skip |= 1u << st;
            }
            gp.bar_skip = skip;
        } else {
            for (int i = 0; i < count; ++i) gp.layer[i].llx = -1;
        }
    }
    // ---- per-stage task split.  A layer's plan fills the GPU on its own
    //      (~1 task per SM); a stage of several layers would then run several
    //      tasks -- several Psumbook builds -- per CTA.  Re-split the rows of
    //      the stage's layers jointly (the prepacked layout does not depend on
    //      it): minimise waves x (per-task cost + rows per task), the per-task
    //      cost (table build, input round trip, flush) expressed in row groups
    //      of gather work.  Layers created with an explicit rg_per_task keep it.
    // (a comm launch runs the comm's grid on every rank: its barrier flags and
    // exchange counters count arrivals of exactly that many CTAs)
    const int sms = comm ? comm->ctas : layers[0]->sms;
    // contiguous per-CTA task ranges with Psumbook reuse (reduce-add split-K, one column)
    bool contig = !(layers[0]->flags & CG_OPT_DETERMINISTIC) && n == 1 &&
                  std::getenv("CG_NO_CONTIG") == nullptr &&
                  cg::fused_contig_instantiated(p0.v, p0.m, p0.u, p0.kbits);
    {
        bool forced = false;
        // columns the per-task smem buffers scale with: reduce-add mode adds the
        // partials of several columns straight into y (no staging)
        const int n_stage = (layers[0]->flags & CG_OPT_DETERMINISTIC) ? n : 1;
        int64_t cap = 1 << 30;
        for (int i = 0; i < count; ++i) {
            forced |= layers[i]->rg_forced;
            cap = std::min<int64_t>(cap, layers[i]->rg_cap / n_stage);
        }
        if (!forced) {
            for (int st = 0; st < gp.n_stages; ++st) {
                int64_t max_rg = 1;
                for (int i = 0; i < count; ++i)
                    if (gp.layer[i].stage == st) max_rg = std::max(max_rg, gp.layer[i].n_rg);
                const double f_rg = 2.0 / (0.019 * p0.u * p0.m);  // ~2 us of fixed cost per task
                auto stage_tasks = [&](int64_t rg) {
                    int64_t tasks = 0;
                    for (int i = 0; i < count; ++i)
                        if (gp.layer[i].stage == st)
                            tasks += gp.layer[i].n_slices * ((gp.layer[i].n_rg + rg - 1) / rg);
                    return tasks;
                };
                double best = 1e300;
                int64_t best_rg = 0;
                for (int64_t rg = 1; rg <= max_rg; ++rg) {
                    if (rg > cap) break;
                    const int64_t tasks = stage_tasks(rg);
                    const double waves = (double)((tasks + sms - 1) / sms);
                    const double cost = waves * (f_rg + (double)rg) + 1e-6 * (double)rg;
                    if (cost < best) {
                        best = cost;
                        best_rg = rg;
                    }
                }
                if (contig && best_rg > 0) {
                    // contiguous task ranges: a CTA rebuilds the Psumbook only when its
                    // range enters another (layer, K-slice); a task that reuses the table
                    // costs ~1/2 of the fixed cost (input wait, flush).  Candidates: the
                    // smallest rg that fits the stage in k tasks per CTA, k = 1..24; cost
                    // = the slowest CTA's rows + per-task and per-build costs.
                    auto contig_cost = [&](int64_t rg) {
                        const int64_t T = stage_tasks(rg);
                        if (T <= sms) return f_rg + (double)rg;
                        double worst = 0.0;
                        for (int64_t c = 0; c < sms; ++c) {
                            const int64_t lo = c * T / sms, hi = (c + 1) * T / sms;
                            if (hi <= lo) continue;
                            // (layer, slice) column of stage task g: columns numbered in order
                            auto column = [&](int64_t g) {
                                int64_t col0 = 0;
                                for (int i = 0; i < count; ++i) {
                                    const cg::LayerTask& t = gp.layer[i];
                                    if (t.stage != st) continue;
                                    const int64_t nrb = (t.n_rg + rg - 1) / rg;
                                    const int64_t nt = t.n_slices * nrb;
                                    if (g < nt) return col0 + g / nrb;
                                    g -= nt;
                                    col0 += t.n_slices;
                                }
                                return col0;
                            };
                            const double builds = (double)(column(hi - 1) - column(lo) + 1);
                            const double cost =
                                (double)(hi - lo) * ((double)rg + 0.5 * f_rg) + 0.5 * f_rg * builds;
                            worst = std::max(worst, cost);
                        }
                        return worst;
                    };
                    double cbest = contig_cost(best_rg);
                    for (int64_t k = 1; k <= 24; ++k) {
                        int64_t lo = 1, hi = std::min<int64_t>(max_rg, cap);
                        if (stage_tasks(hi) > k * sms) continue;
                        while (lo < hi) {  // smallest rg with at most k tasks per CTA
                            const int64_t mid = (lo + hi) / 2;
                            if (stage_tasks(mid) <= k * sms) hi = mid;
                            else lo = mid + 1;
                        }
                        const double cst = contig_cost(lo);
                        if (cst < cbest) {
                            cbest = cst;
                            best_rg = lo;
                        }
                    }
                }
                if (best_rg < 1) continue;
                for (int i = 0; i < count; ++i) {
                    cg::LayerTask& t = gp.layer[i];
                    if (t.stage != st) continue;
                    const int64_t rg = std::min<int64_t>(best_rg, t.n_rg);
                    t.rg_per_task = (int)rg;
                    t.n_rb = (t.n_rg + rg - 1) / rg;
                    t.n_tasks = (int)(t.n_slices * t.n_rb);
                }
            }
        }
        for (int i = 0; i < count; ++i) {
            const cg::Plan& p = layers[i]->plan;
            scl_max = std::max(scl_max, gp.layer[i].rg_per_task * p.n_gs * 32);
            rg_max = std::max(rg_max, gp.layer[i].rg_per_task);
            grid = std::max(grid, gp.layer[i].n_tasks);
        }
    }
    // persistent grid: one CTA per SM, always the full grid (the per-CTA grid
    // barrier flags rely on every launch making the same arrivals on every
    // CTA); if a layer has more tasks than CTAs, a CTA runs several tasks of it
    // and deterministic split-K falls back to last-arriver sums
    if (grid > sms) gp.flags |= cg::kFlagLastArriver;
    grid = sms;
    for (int i = 0; i < count; ++i) {
        const int64_t elems = gp.layer[i].rows * n;
        if (elems >= (int64_t(1) << 31))
            return fail(CG_ERR_SHAPE, "layer %d: rows * n = %lld exceeds 2^31", i, (long long)elems);
        gp.layer[i].zero_per =
            gp.layer[i].llp ? 0 : (int)((((elems + grid - 1) / grid) + 3) & ~int64_t(3));
    }
    // fix-up list / owned-ticket targets (deterministic) or the staging buffer
    // of a task's partial rows (reduce-add): the larger of the two
    const int cap = rg_max * n + 16;
    const int n_buf = (layers[0]->flags & CG_OPT_DETERMINISTIC) ? n : 1;
    const int list_bytes = (int)list_bytes_for(rg_max, n_buf);
    cg::SmemLayout lay;
    if (!cg::smem_layout(zmax, scl_max, raw_bytes, list_bytes, layers[0]->reserved, &lay,
                         rg_max * 16 * n_buf * 4))
        return fail(CG_ERR_CONFIG,
                    "fused kernel does not fit in shared memory at n=%d (rows per task %d); "
                    "use fewer columns per call or CG_MODE_STRICT", n, rg_max);
    gp.off_psum = lay.off_psum;
    gp.off_books = lay.off_books;
    gp.off_x = lay.off_x;
    gp.off_scl[0] = lay.off_scl[0];
    gp.off_scl[1] = lay.off_scl[1];
    gp.off_raw[0] = lay.off_raw[0];
    gp.off_raw[1] = lay.off_raw[1];
    gp.raw_x_off = books_raw;
    gp.off_bar = lay.off_bar;
    gp.off_list = lay.off_list;
    gp.off_stage[0] = lay.off_list;
    gp.off_stage[1] = lay.off_stage1;
    gp.list_cap = cap;
    gp.grid_flags = comm ? reinterpret_cast<unsigned long long*>(comm->base + cg::kXcFlags)
                         : layers[0]->grid_flags;
    if (!x_copy) gp.flags |= cg::kFlagXRegs;
    // ranks sharing one GPU (comm->ctas < SMs) must run concurrently: no
    // cooperative attribute (it may serialise their grids); each grid fits
    if (comm && comm->ctas < layers[0]->sms) gp.flags |= cg::kFlagDbgNoCoop;
    if (layers[0]->flags & CG_OPT_DETERMINISTIC) gp.flags |= cg::kFlagDeterministic;
    if (contig) {  // the contiguous instance only where a CTA runs several tasks of a stage
        bool multi = false;
        for (int st = 0; st < gp.n_stages; ++st) {
            int64_t tasks = 0;
            for (int i = 0; i < count; ++i)
                if (gp.layer[i].stage == st) tasks += gp.layer[i].n_tasks;
            multi |= tasks > sms;
        }
        if (multi) gp.flags |= cg::kFlagContig;
    }
    if (const char* e = std::getenv("CG_DEBUG_FLAGS")) gp.flags |= std::atoi(e);
    out->gp = gp;
    out->grid = grid;
    out->smem = lay.total;
    out->pdl = !(layers[0]->flags & CG_OPT_NO_PDL) && !(gp.flags & cg::kFlagDbgNoPdl);
    out->v = p0.v;
    out->m = p0.m;
    out->u = p0.u;
    out->kbits = p0.kbits;
    return CG_OK;
}

int launch_plan(const StagedPlan& sp, cudaStream_t s) {
    CG_CUDA(cg::launch_group_gemv(sp.v, sp.m, sp.u, sp.kbits, sp.gp, sp.grid, sp.smem, sp.pdl, s),
            "fused gemv launch");
    return CG_OK;
}

int launch_stages(cg_layer* const* layers, const uint16_t* const* xs, float* const* ys,
                  const int* stages, int count, int n, cudaStream_t s,
                  const int* x_dtypes = nullptr, const int* xchg = nullptr,
                  cg_comm* comm = nullptr) {
    StagedPlan sp;
    const int rc = plan_stages(layers, xs, ys, stages, count, n, x_dtypes, xchg, comm, &sp);
    return rc ? rc : launch_plan(sp, s);
}

// Group launch: layers are partitioned by their tiling u (one kernel
// instantiation per u); each partition is one launch, in first-seen order.
int launch_group(cg_layer* const* layers, const uint16_t* const* xs, float* const* ys, int count,
                 int n, cudaStream_t s) {
    bool done[cg::kMaxGroup] = {false};
    for (int i = 0; i < count; ++i) {
        if (done[i]) continue;
        cg_layer* part[cg::kMaxGroup];
        const uint16_t* px[cg::kMaxGroup];
        float* py[cg::kMaxGroup];
        int k = 0;
        for (int j = i; j < count; ++j) {
            if (done[j] || layers[j]->plan.u != layers[i]->plan.u) continue;
            part[k] = layers[j];
            px[k] = xs[j];
            py[k] = ys[j];
            ++k;
            done[j] = true;
        }
        int rc = launch_stages(part, px, py, nullptr, k, n, s);
        if (rc) return rc;
    }
    return CG_OK;
}

// ---- batch path (K4) ----
unsigned long long* g_batch_stamps = nullptr;  // diagnostics (CG_STAMPS=1)

// The config has a batch kernel: v in {4, 8}, m in {1, 2}, b <= 8, and scale
// groups that close at k16-step granularity without straddling a 128-element
// chunk: g in {16, 32, 64} or a multiple of 128, or one group per row.
bool batch_config_ok(const cg::Plan& p) {
    if (!cg::batch_supported_vm(p.v, p.m) || p.b > 8) return false;
    if (p.g_row || p.g_eff >= p.cols) return true;
    return p.g_eff == 16 || p.g_eff == 32 || p.g_eff == 64 || p.g_eff % 128 == 0;
}

// Task geometry of one layer at batch width n: 32 rows x a K-slice of at most
// 4096/NT elements (equal slices), shrunk until it fits shared memory and
// never straddling a scale group.
bool plan_batch(const cg::Plan& p, int n, cg::BatchLayer* out, int* smem_out) {
    if (!batch_config_ok(p)) return false;
    const int nt = cg::batch_nt_for(n);
    const int n_rt = (int)((p.rows + 15) / 16);
    const int n_chunks = (int)((p.cols + 127) / 128);
    const int rsets = (n_rt + 1) / 2;
    const bool one_group = p.g_row || p.g_eff >= p.cols;
    // slices of at most 4096/NT elements (measured: one slice of a larger x^T tile
    // costs more in staging and occupancy than the extra partial plane), all
    // slices the same width
    int ks = std::min(n_chunks, 32 / nt);
    ks = (n_chunks + ((n_chunks + ks - 1) / ks) - 1) / ((n_chunks + ks - 1) / ks);
    for (; ks >= 1; --ks) {
        const int64_t kslice = (int64_t)ks * 128;
        if (!one_group && ks < n_chunks && p.g_eff > kslice && p.g_eff % kslice != 0) continue;
        const int gis = one_group ? 1 : (int)std::max<int64_t>(1, kslice / p.g_eff);
        if (cg::batch_layout(p.v, p.m, p.kcount, nt, ks, gis, nullptr) <= 225 * 1024) break;  // (+ the static layer table)
    }
    if (ks < 1) return false;
    cg::BatchLayer b{};
    b.rows = p.rows;
    b.cols = p.cols;
    b.groups = one_group ? 1 : p.groups;
    b.g_eff = one_group ? ((int64_t)1 << 62) : p.g_eff;
    b.g_row = one_group ? 1 : 0;
    b.kcount = p.kcount;
    b.n_rt = n_rt;
    b.n_chunks = n_chunks;
    b.ks_chunks = ks;
    b.n_slices = (n_chunks + ks - 1) / ks;
    b.n_rsets = rsets;
    b.n_tasks = rsets * b.n_slices;
    const int64_t kslice = (int64_t)ks * 128;
    if (one_group || p.g_eff >= kslice) {
        b.spg = ks * 8;  // the whole slice lies in one scale group
        b.gis = 1;
    } else {
        b.spg = (int)(p.g_eff / 16);
        b.gis = (int)(kslice / p.g_eff);
    }
    *out = b;
    *smem_out = cg::batch_layout(p.v, p.m, p.kcount, nt, ks, b.gis, nullptr);
    return true;
}

// the batch code stream and scale tiles, from the uint16 planes recovered on the device
int ensure_batch_codes(cg_layer* L, cudaStream_t s) {
    if (L->bcodes) return CG_OK;
    const cg::Plan& p = L->plan;
    const bool one_group = p.g_row || p.g_eff >= p.cols;
    const int64_t bytes = cg::batch_code_bytes(p.rows, p.cols, p.v, p.m);
    const int64_t groups = one_group ? 1 : p.groups;
    int rc = dev_alloc(L, &L->bcodes, (size_t)bytes, "batch code stream alloc");
    if (rc) return rc;
    rc = dev_alloc(L, &L->bscl, (size_t)cg::batch_scale_bytes(p.rows, groups), "batch scales alloc");
    if (rc) return rc;
    uint16_t* raw = L->raw16;
    bool tmp = false;
    if (!raw) {
        CG_CUDA(cudaMalloc(&raw, (size_t)p.m * p.rows * p.segs * 2), "batch prepack staging");
        tmp = true;
        cudaError_t e = cg::launch_unpack_codes(p, L->codes, nullptr, raw, s);
        if (e != cudaSuccess) {
            cudaFree(raw);
            return cuda_fail(e, "batch prepack (unpack)");
        }
    }
    // one scale per row: the (rows, 1) plane; else the (rows, groups) plane
    cudaError_t e = cg::launch_prepack_batch(raw, L->bcodes, p.rows, p.segs, p.m, p.v, L->scales,
                                             groups, L->bscl, s);
    if (e == cudaSuccess && tmp) e = cudaStreamSynchronize(s);
    if (tmp) cudaFree(raw);
    if (e != cudaSuccess) return cuda_fail(e, "batch prepack");
    return CG_OK;
}

int ensure_batch_ws(cg_layer* L, int64_t bytes) {
    if (bytes <= L->bws_bytes) return CG_OK;
    cudaFree(L->bws);
    L->device_bytes -= L->bws_bytes;
    L->bws = nullptr;
    L->bws_bytes = 0;
    int rc = dev_alloc(L, &L->bws, (size_t)bytes, "batch workspace alloc");
    if (rc) return rc;
    L->bws_bytes = bytes;
    return CG_OK;
}

// One persistent launch of K4 (+ the ordered split-K sum) for `count` layers
// sharing v and m, over columns [c0, c0 + nb) of x / y (row stride ld).
int launch_batch(cg_layer* const* layers, const uint16_t* const* xs, float* const* ys, int count,
                 int ld, int c0, int nb, cudaStream_t s) {
    cg::BatchParams bp{};
    bp.n_layers = count;
    bp.n = nb;
    bp.ld = ld;
    const cg::Plan& p0 = layers[0]->plan;
    const int nt = cg::batch_nt_for(nb);
    int kc_max = 0, ks_max = 0, gis_max = 0, tasks = 0;
    for (int i = 0; i < count; ++i) {
        cg_layer* L = layers[i];
        int sm = 0;
        if (!plan_batch(L->plan, nb, &bp.layer[i], &sm))
            return fail(CG_ERR_UNSUPPORTED, "layer %d has no batch kernel", i);
        if (reinterpret_cast<uintptr_t>(xs[i]) & 15)
            return fail(CG_ERR_ARG, "x of layer %d is not 16-byte aligned", i);
        int rc = ensure_batch_codes(L, s);
        if (rc) return rc;
        cg::BatchLayer& b = bp.layer[i];
        if (b.n_slices > 1) {
            rc = ensure_batch_ws(L, (int64_t)b.n_slices * L->plan.rows * nb * 4);
            if (rc) return rc;
        }
        b.codes = L->bcodes;
        b.scl = L->bscl;
        b.books = L->books;
        b.x = xs[i] + c0;
        b.y = ys[i] + c0;
        b.ws = L->bws;
        b.x0 = xs[i];
        kc_max = std::max(kc_max, b.kcount);
        ks_max = std::max(ks_max, b.ks_chunks);
        gis_max = std::max(gis_max, b.gis);
        tasks += b.n_tasks;
    }
    bp.total_tasks = tasks;
    if (std::getenv("CG_STAMPS")) {  // diagnostics: one stamp buffer per process
        if (!g_batch_stamps && cudaMalloc(&g_batch_stamps, 64 * 1024 * 8) == cudaSuccess)
            cudaMemset(g_batch_stamps, 0, 64 * 1024 * 8);
        bp.stamps = g_batch_stamps;
    }
    const int smem = cg::batch_layout(p0.v, p0.m, kc_max, nt, ks_max, gis_max, &bp);
    if (smem > 225 * 1024)
        return fail(CG_ERR_CONFIG, "batch launch does not fit in shared memory (%d bytes)", smem);
    // every layer's code tiles must fit the buffer stride of the largest slice
    const int grid = std::min(tasks, layers[0]->sms);
    CG_CUDA(cg::launch_batch_gemm(p0.v, p0.m, nt, bp, grid, smem, s,
                                  !(layers[0]->flags & CG_OPT_NO_PDL)),
            "batch gemm launch");
    return CG_OK;
}

// n >= 2 through K4 in column blocks of <= 32
int run_batch(cg_layer* const* layers, const uint16_t* const* xs, float* const* ys, int count,
              int n, cudaStream_t s) {
    for (int c0 = 0; c0 < n; c0 += 32) {
        const int nb = std::min(32, n - c0);
        int rc = launch_batch(layers, xs, ys, count, n, c0, nb, s);
        if (rc) return rc;
    }
    return CG_OK;
}

bool use_batch(const cg_layer* L, int n) {
    return n >= 2 && L->batch_ok && !(L->flags & CG_OPT_NO_BATCH);
}

int run_gemm(cg_layer* L, const uint16_t* x, int n, float* y, int mode, cudaStream_t s) {
    const cg::Plan& p = L->plan;
    if (mode == CG_MODE_AUTO) mode = (p.fast || use_batch(L, n)) ? CG_MODE_FAST : CG_MODE_STRICT;
    if (mode == CG_MODE_FAST && !p.fast && !use_batch(L, n))
        return fail(CG_ERR_UNSUPPORTED,
                    "no fused kernel for v=%d m=%d b=%d g=%lld at cols=%lld; use CG_MODE_STRICT",
                    p.v, p.m, p.b, (long long)p.g, (long long)p.cols);
    if (mode == CG_MODE_STRICT) {
        CG_CUDA(cg::launch_strict_gemm(p, L->codes, L->raw16, L->books, L->scales, x, n, y, s),
                "strict kernel launch");
        return CG_OK;
    }
    if (mode != CG_MODE_FAST) return fail(CG_ERR_ARG, "unknown mode %d", mode);
    cg_layer* one[1] = {L};
    const uint16_t* xs[1] = {x};
    float* ys[1] = {y};
    if (use_batch(L, n)) return run_batch(one, xs, ys, 1, n, s);
    return launch_group(one, xs, ys, 1, n, s);
}

}  // namespace

extern "C" {

int cg_abi_version(void) { return CG_ABI_VERSION; }

const char* cg_last_error(void) { return g_last_error.c_str(); }

int cg_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

}  // extern "C"

namespace {
// codes: uint16 planes (host), or packed: b-bit packed planes (host, CGMM layout)
int create_layer(const uint16_t* const* codes, const uint8_t* const* packed,
                 const uint16_t* const* books, const uint16_t* scales, int64_t rows, int64_t cols,
                 int v, int m, int b, int64_t g, const cg_layer_options* opts, cg_layer** out) {
    if (!out) return fail(CG_ERR_ARG, "out is NULL");
    *out = nullptr;
    if ((!codes && !packed) || !books || !scales)
        return fail(CG_ERR_ARG, "NULL codes/books/scales");
    // QuantConfig.__post_init__ / validate_shape (quantizer.py:55-84)
    if (v < 1) return fail(CG_ERR_CONFIG, "v must be >= 1, got %d", v);
    if (m < 1) return fail(CG_ERR_CONFIG, "m must be >= 1, got %d", m);
    if (b < 1 || b > 16) return fail(CG_ERR_CONFIG, "b must be in [1, 16], got %d", b);
    if (g != -1) {
        if (g < v) return fail(CG_ERR_CONFIG, "g must be >= v (got g=%lld, v=%d)", (long long)g, v);
        if (g % v) return fail(CG_ERR_CONFIG, "g must be a multiple of v (got g=%lld, v=%d)",
                               (long long)g, v);
    }
    if (rows < 1 || cols < 1)
        return fail(CG_ERR_CONFIG, "matrix dims must be >= 1, got %lldx%lld", (long long)rows,
                    (long long)cols);
    if (cols % v) return fail(CG_ERR_CONFIG, "cols=%lld not divisible by v=%d", (long long)cols, v);
    const int64_t g_eff = g == -1 ? cols : g;
    if (cols % g_eff)
        return fail(CG_ERR_CONFIG, "cols=%lld not divisible by g=%lld", (long long)cols,
                    (long long)g);
    for (int t = 0; t < m; ++t)
        if (!(codes ? (const void*)codes[t] : (const void*)packed[t]) || !books[t])
            return fail(CG_ERR_ARG, "NULL plane/book %d", t);

    int device = 0;
    if (opts && opts->device >= 0) device = opts->device;
    else if (cudaGetDevice(&device) != cudaSuccess) device = 0;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return fail(CG_ERR_CUDA, "no CUDA device available (%s); this library has no CPU path",
                    cudaGetErrorString(e));
    if (device >= ndev) return fail(CG_ERR_ARG, "device %d out of range (%d)", device, ndev);
    DeviceGuard guard(device);

    cg_layer* L = new cg_layer();
    L->device = device;
    L->flags = opts ? opts->flags : 0;
    L->sms = sm_count_of(device);
    if (const char* e = std::getenv("CG_PF_DIST")) L->pf_dist = std::atoi(e);  // tuning knob
    cg::Plan& p = L->plan;
    p.rows = rows;
    p.cols = cols;
    p.v = v;
    p.m = m;
    p.b = b;
    p.g = g;
    p.g_row = (g == -1);
    p.g_eff = g_eff;
    p.kcount = 1 << b;
    p.segs = cols / v;
    p.groups = cols / g_eff;
    int reserved = 1024;
    if (cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, device) !=
        cudaSuccess)
        reserved = 1024;
    L->reserved = reserved;
    plan_fast(p, opts ? opts->u : 0, opts ? opts->rg_per_task : 0, sm_count_of(device), reserved);
    L->rg_forced = opts && opts->rg_per_task > 0;
    L->rg_cap = p.fast ? p.rg_cap : 0;
    // a tiling the fused kernel never has (u not in {1,2,4} or m*u > 4) is a
    // config error; a valid u the fused kernel cannot use for this group size
    // (scale group < 8 lanes) leaves a strict-mode-only layer
    if (opts && opts->u && !p.fast &&
        (!(opts->u == 1 || opts->u == 2 || opts->u == 4) || m * opts->u > 4)) {
        free_layer(L);
        return fail(CG_ERR_CONFIG, "u=%d is not valid for v=%d m=%d b=%d g=%lld", opts->u, v, m,
                    b, (long long)g);
    }

    const size_t plane_elems = (size_t)rows * p.segs;
    const size_t raw_bytes = plane_elems * m * 2;
    const size_t scale_elems = (size_t)rows * p.groups;
    const size_t book_elems = (size_t)p.kcount * v;
    int rc = CG_OK;
    uint16_t* raw = nullptr;
    unsigned* bad = nullptr;
    cudaStream_t s = nullptr;
    auto bail = [&](int code) {
        cudaFree(raw);
        cudaFree(bad);
        free_layer(L);
        return code;
    };
    if ((rc = dev_alloc(L, &L->scales, scale_elems * 2, "scales alloc"))) return bail(rc);
    if ((rc = dev_alloc(L, &L->books, book_elems * m * 2, "books alloc"))) return bail(rc);
    e = cudaMemcpy(L->scales, scales, scale_elems * 2, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return bail(cuda_fail(e, "scales upload"));
    for (int t = 0; t < m; ++t) {
        e = cudaMemcpy(L->books + t * book_elems, books[t], book_elems * 2, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return bail(cuda_fail(e, "books upload"));
    }
    e = cudaMalloc(&raw, raw_bytes ? raw_bytes : 16);
    if (e != cudaSuccess) return bail(cuda_fail(e, "plane staging alloc"));
    e = cudaMalloc(&bad, sizeof(unsigned));
    if (e != cudaSuccess) return bail(cuda_fail(e, "flag alloc"));
    cudaMemset(bad, 0, sizeof(unsigned));
    if (codes) {
        for (int t = 0; t < m; ++t) {
            e = cudaMemcpy(raw + t * plane_elems, codes[t], plane_elems * 2, cudaMemcpyHostToDevice);
            if (e != cudaSuccess) return bail(cuda_fail(e, "plane upload"));
        }
    } else {
        // b bits per code on the wire; unpacked to uint16 planes on the device
        const int64_t plane_bytes = ((int64_t)plane_elems * b + 7) / 8;
        uint8_t* pk = nullptr;
        e = cudaMalloc(&pk, (size_t)(plane_bytes * m + 16));
        if (e != cudaSuccess) return bail(cuda_fail(e, "packed plane staging alloc"));
        for (int t = 0; t < m && e == cudaSuccess; ++t)
            e = cudaMemcpy(pk + t * plane_bytes, packed[t], (size_t)plane_bytes,
                           cudaMemcpyHostToDevice);
        if (e == cudaSuccess)
            e = cg::launch_unpack_packed(pk, plane_bytes, m, (int64_t)plane_elems, b, raw, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        cudaFree(pk);
        if (e != cudaSuccess) return bail(cuda_fail(e, "packed plane upload"));
    }
    if (p.fast) {
        if ((rc = dev_alloc(L, &L->codes, (size_t)p.code_bytes, "code stream alloc")))
            return bail(rc);
        if ((rc = dev_alloc(L, &L->scl, (size_t)p.scale_bytes, "scale tiles alloc")))
            return bail(rc);
        e = cg::launch_prepack_codes(p, raw, L->codes, bad, s);
        if (e != cudaSuccess) return bail(cuda_fail(e, "prepack codes"));
        e = cg::launch_prepack_scales(p, L->scales, L->scl, s);
        if (e != cudaSuccess) return bail(cuda_fail(e, "prepack scales"));
    } else {
        e = cg::launch_check_codes(p, raw, bad, s);
        if (e != cudaSuccess) return bail(cuda_fail(e, "check codes"));
    }
    unsigned bad_h = 0;
    e = cudaMemcpy(&bad_h, bad, sizeof bad_h, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return bail(cuda_fail(e, "prepack"));
    if (bad_h) return bail(fail(CG_ERR_INTEGRITY, "code out of range for b=%d", b));
    if (p.fast) {
        cudaFree(raw);
    } else {
        L->raw16 = raw;  // strict kernel reads the uint16 planes directly
        L->device_bytes += (int64_t)raw_bytes;
    }
    raw = nullptr;
    cudaFree(bad);
    bad = nullptr;
    if (p.fast && p.n_slices > 1) {
        if ((rc = ensure_ws(L, 1))) return bail(rc);
    }
    if (p.fast) {
        const size_t cb = (size_t)(1 + p.n_rg) * sizeof(unsigned long long);
        if ((rc = dev_alloc(L, &L->rg_cnt, cb, "row-group counters"))) return bail(rc);
        cudaMemset(L->rg_cnt, 0, cb);
        const size_t fb = (size_t)(16 + L->sms) * sizeof(unsigned long long);
        if ((rc = dev_alloc(L, &L->grid_flags, fb, "grid barrier flags"))) return bail(rc);
        cudaMemset(L->grid_flags, 0, fb);
    }
    L->batch_ok = batch_config_ok(p) && (p.fast || L->raw16);
    if (L->batch_ok && (L->flags & CG_OPT_BATCH_EAGER)) {
        if ((rc = ensure_batch_codes(L, s))) return bail(rc);
        if (cudaStreamSynchronize(s) != cudaSuccess) return bail(fail(CG_ERR_CUDA, "batch prepack"));
    }
    if (p.fast && std::getenv("CG_STAMPS")) {
        if ((rc = dev_alloc(L, &L->stamps, (size_t)L->sms * 1024, "stamps"))) return bail(rc);
        cudaMemset(L->stamps, 0, (size_t)L->sms * 1024);
    }
    *out = L;
    return CG_OK;
}

}  // namespace

extern "C" {

int cg_layer_create(const uint16_t* const* codes, const uint16_t* const* books,
                    const uint16_t* scales, int64_t rows, int64_t cols, int v, int m, int b,
                    int64_t g, const cg_layer_options* opts, cg_layer** out) {
    if (!codes) return fail(CG_ERR_ARG, "NULL codes");
    return create_layer(codes, nullptr, books, scales, rows, cols, v, m, b, g, opts, out);
}

int cg_layer_create_packed(const uint8_t* const* planes, const uint16_t* const* books,
                           const uint16_t* scales, int64_t rows, int64_t cols, int v, int m,
                           int b, int64_t g, const cg_layer_options* opts, cg_layer** out) {
    if (!planes) return fail(CG_ERR_ARG, "NULL planes");
    return create_layer(nullptr, planes, books, scales, rows, cols, v, m, b, g, opts, out);
}

int cg_layer_destroy(cg_layer* layer) {
    free_layer(layer);
    return CG_OK;
}

int cg_layer_query(const cg_layer* L, cg_layer_info* info) {
    if (!L || !info) return fail(CG_ERR_ARG, "NULL layer/info");
    const cg::Plan& p = L->plan;
    std::memset(info, 0, sizeof *info);
    info->rows = p.rows;
    info->cols = p.cols;
    info->v = p.v;
    info->m = p.m;
    info->b = p.b;
    info->g = p.g;
    info->fast_supported = p.fast ? 1 : 0;
    info->u = p.u;
    info->rg_per_task = p.rg_per_task;
    info->n_slices = p.n_slices;
    info->n_tasks = p.fast ? p.n_slices * p.n_rb : 0;
    info->smem_bytes = p.fast ? p.smem.total : 0;
    info->launches_fast = p.fast ? 1 : 0;
    info->device_bytes = L->device_bytes;
    // codes at b bits + binary16 scales + binary16 codebooks
    info->algorithmic_bytes = (p.rows * p.segs * p.m * p.b + 7) / 8 + 2 * p.rows * p.groups +
                              2LL * p.m * p.kcount * p.v;
    info->batch_supported = L->batch_ok && !(L->flags & CG_OPT_NO_BATCH) ? 1 : 0;
    info->batch_ready = L->bcodes ? 1 : 0;
    return CG_OK;
}

int cg_layer_gemm(cg_layer* L, const void* x, int n, float* y, int mode, void* stream) {
    if (!L || !x || !y) return fail(CG_ERR_ARG, "NULL layer/x/y");
    if (n < 1) return fail(CG_ERR_SHAPE, "x must have >= 1 column, got %d", n);
    DeviceGuard guard(L->device);
    return run_gemm(L, static_cast<const uint16_t*>(x), n, y, mode,
                    static_cast<cudaStream_t>(stream));
}

int cg_gemm_group(cg_layer* const* layers, const void* const* xs, float* const* ys, int count,
                  int n, void* stream) {
    if (!layers || !xs || !ys) return fail(CG_ERR_ARG, "NULL layers/xs/ys");
    if (count < 1 || count > cg::kMaxGroup)
        return fail(CG_ERR_ARG, "group size %d outside 1..%d", count, cg::kMaxGroup);
    if (n < 1) return fail(CG_ERR_SHAPE, "x must have >= 1 column, got %d", n);
    for (int i = 0; i < count; ++i)
        if (!layers[i] || !xs[i] || !ys[i]) return fail(CG_ERR_ARG, "NULL entry %d", i);
    DeviceGuard guard(layers[0]->device);
    bool batch = count <= cg::kMaxBatchGroup;
    for (int i = 0; i < count && batch; ++i)
        batch = use_batch(layers[i], n) && layers[i]->plan.v == layers[0]->plan.v &&
                layers[i]->plan.m == layers[0]->plan.m;
    if (batch)
        return run_batch(layers, reinterpret_cast<const uint16_t* const*>(xs), ys, count, n,
                         static_cast<cudaStream_t>(stream));
    return launch_group(layers, reinterpret_cast<const uint16_t* const*>(xs), ys, count, n,
                        static_cast<cudaStream_t>(stream));
}

int cg_gemm_stages(cg_layer* const* layers, const void* const* xs, const int* x_dtypes,
                   float* const* ys, const int* stages, int count, int n, void* stream) {
    if (!layers || !xs || !ys || !stages) return fail(CG_ERR_ARG, "NULL layers/xs/ys/stages");
    if (count < 1 || count > cg::kMaxGroup)
        return fail(CG_ERR_ARG, "launch size %d outside 1..%d", count, cg::kMaxGroup);
    if (n < 1) return fail(CG_ERR_SHAPE, "x must have >= 1 column, got %d", n);
    for (int i = 0; i < count; ++i)
        if (!layers[i] || !xs[i] || !ys[i]) return fail(CG_ERR_ARG, "NULL entry %d", i);
    DeviceGuard guard(layers[0]->device);
    return launch_stages(layers, reinterpret_cast<const uint16_t* const*>(xs), ys, stages, count,
                         n, static_cast<cudaStream_t>(stream), x_dtypes);
}

int cg_gemm_stages_xchg(cg_layer* const* layers, const void* const* xs, const int* x_dtypes,
                        float* const* ys, const int* stages, const int* xchg, int count, int n,
                        cg_comm* comm, void* stream) {
    if (!layers || !xs || !ys || !stages || !xchg || !comm)
        return fail(CG_ERR_ARG, "NULL layers/xs/ys/stages/xchg/comm");
    if (count < 1 || count > cg::kMaxGroup)
        return fail(CG_ERR_ARG, "launch size %d outside 1..%d", count, cg::kMaxGroup);
    if (n < 1) return fail(CG_ERR_SHAPE, "x must have >= 1 column, got %d", n);
    for (int i = 0; i < count; ++i)
        if (!layers[i] || !xs[i] || !ys[i]) return fail(CG_ERR_ARG, "NULL entry %d", i);
    DeviceGuard guard(layers[0]->device);
    return launch_stages(layers, reinterpret_cast<const uint16_t* const*>(xs), ys, stages, count,
                         n, static_cast<cudaStream_t>(stream), x_dtypes, xchg, comm);
}

// ---- prepared staged launches (cg_stages_*): planned once, launched per call
struct cg_stages {
    StagedPlan plan;
    float* mirror[cg::kMaxGroup] = {nullptr};  // host-mapped y copies (cg_stages_set_mirror)
    bool no_llc = false;  // mirrors copy y at stage barriers: plan without the LL chain
    int gen = 0;  // bumped whenever the launch parameters change
    // cg_stages_run_host replays one CUDA graph (H2D, the launch, D2H): a direct
    // cooperative launch costs tens of microseconds of host time per call
    cudaGraphExec_t gexec = nullptr;
    int g_gen = -1;
    const void* g_xh = nullptr;
    void* g_xd = nullptr;
    const void* g_yd = nullptr;
    void* g_yh = nullptr;
    int64_t g_xb = -1, g_yb = -1;
    int count = 0, n = 0, device = 0;
    cg_layer* layers[cg::kMaxGroup] = {nullptr};
    const uint16_t* xs[cg::kMaxGroup] = {nullptr};
    float* ys[cg::kMaxGroup] = {nullptr};
    int stages[cg::kMaxGroup] = {0}, x_dtypes[cg::kMaxGroup] = {0}, xchg[cg::kMaxGroup] = {0};
    float* ws[cg::kMaxGroup] = {nullptr};  // split-K workspaces the plan points at
    cg_comm* comm = nullptr;
};

namespace {
int replan_if_needed(cg_stages* P, bool force = false) {
    bool stale = force;
    for (int i = 0; i < P->count; ++i) stale |= P->layers[i]->ws != P->ws[i];
    if (!stale) return CG_OK;  // (a layer's workspace grew for a wider call since)
    int rc = plan_stages(P->layers, P->xs, P->ys, P->stages, P->count, P->n, P->x_dtypes,
                         P->comm ? P->xchg : nullptr, P->comm, &P->plan, !P->no_llc);
    if (rc) return rc;
    for (int i = 0; i < P->count; ++i) P->ws[i] = P->layers[i]->ws;
    for (int i = 0; i < P->count; ++i) P->plan.gp.layer[i].mirror = P->mirror[i];
    ++P->gen;
    return CG_OK;
}
}  // namespace

int cg_stages_prepare(cg_layer* const* layers, const void* const* xs, const int* x_dtypes,
                      float* const* ys, const int* stages, const int* xchg, int count, int n,
                      cg_comm* comm, cg_stages** out) {
    if (!out) return fail(CG_ERR_ARG, "NULL out");
    *out = nullptr;
    if (!layers || !xs || !ys || !stages) return fail(CG_ERR_ARG, "NULL layers/xs/ys/stages");
    if (count < 1 || count > cg::kMaxGroup)
        return fail(CG_ERR_ARG, "launch size %d outside 1..%d", count, cg::kMaxGroup);
    if (n < 1) return fail(CG_ERR_SHAPE, "x must have >= 1 column, got %d", n);
    if (xchg && !comm) return fail(CG_ERR_ARG, "xchg flags need a comm");
    for (int i = 0; i < count; ++i)
        if (!layers[i] || !xs[i] || !ys[i]) return fail(CG_ERR_ARG, "NULL entry %d", i);
    DeviceGuard guard(layers[0]->device);
    cg_stages* P = new cg_stages;
    P->count = count;
    P->n = n;
    P->device = layers[0]->device;
    P->comm = comm;
    for (int i = 0; i < count; ++i) {
        P->layers[i] = layers[i];
        P->xs[i] = static_cast<const uint16_t*>(xs[i]);
        P->ys[i] = ys[i];
        P->stages[i] = stages[i];
        P->x_dtypes[i] = x_dtypes ? x_dtypes[i] : CG_X_F16;
        P->xchg[i] = xchg ? xchg[i] : 0;
    }
    int rc = plan_stages(P->layers, P->xs, P->ys, P->stages, count, n, P->x_dtypes,
                         comm ? P->xchg : nullptr, comm, &P->plan);
    if (rc) {
        delete P;
        return rc;
    }
    for (int i = 0; i < count; ++i) P->ws[i] = layers[i]->ws;
    *out = P;
    return CG_OK;
}

int cg_stages_launch(cg_stages* P, void* stream) {
    if (!P) return fail(CG_ERR_ARG, "NULL plan");
    DeviceGuard guard(P->device);
    int rc = replan_if_needed(P);
    return rc ? rc : launch_plan(P->plan, static_cast<cudaStream_t>(stream));
}

int cg_stages_run_host(cg_stages* P, const void* x_host, int64_t x_bytes, void* x_dev,
                       const void* y_dev, void* y_host, int64_t y_bytes, void* stream) {
    if (!P) return fail(CG_ERR_ARG, "NULL plan");
    if (x_bytes < 0 || y_bytes < 0 || (x_bytes && (!x_host || !x_dev)) ||
        (y_bytes && (!y_host || !y_dev)))
        return fail(CG_ERR_ARG, "bad host/device copy arguments");
    DeviceGuard guard(P->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int rc = replan_if_needed(P);
    if (rc) return rc;
    const bool same = P->gexec && P->g_gen == P->gen && P->g_xh == x_host && P->g_xb == x_bytes &&
                      P->g_xd == x_dev && P->g_yd == y_dev && P->g_yh == y_host && P->g_yb == y_bytes;
    if (!same && !std::getenv("CG_NO_HOST_GRAPH")) {
        // (re)capture: H2D of the inputs, the launch (no PDL inside a graph of its
        // own), D2H of the outputs -- then every call is one graph launch
        if (P->gexec) cudaGraphExecDestroy(P->gexec);
        P->gexec = nullptr;
        cudaStream_t cs = nullptr;
        cudaGraph_t graph = nullptr;
        bool ok = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) == cudaSuccess &&
                  cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
        if (ok) {
            if (x_bytes)
                ok = cudaMemcpyAsync(x_dev, x_host, (size_t)x_bytes, cudaMemcpyHostToDevice, cs) ==
                     cudaSuccess;
            StagedPlan sp = P->plan;
            sp.pdl = false;
            if (ok) ok = cg::launch_group_gemv(sp.v, sp.m, sp.u, sp.kbits, sp.gp, sp.grid, sp.smem,
                                               false, cs) == cudaSuccess;
            if (ok && y_bytes)
                ok = cudaMemcpyAsync(y_host, y_dev, (size_t)y_bytes, cudaMemcpyDeviceToHost, cs) ==
                     cudaSuccess;
            ok = (cudaStreamEndCapture(cs, &graph) == cudaSuccess) && ok;
            if (ok) ok = cudaGraphInstantiate(&P->gexec, graph, 0) == cudaSuccess;
        }
        if (graph) cudaGraphDestroy(graph);
        if (cs) cudaStreamDestroy(cs);
        if (!ok) {  // (capture unsupported here: direct calls below)
            cudaGetLastError();
            if (P->gexec) cudaGraphExecDestroy(P->gexec);
            P->gexec = nullptr;
        } else {
            P->g_gen = P->gen;
            P->g_xh = x_host;
            P->g_xb = x_bytes;
            P->g_xd = x_dev;
            P->g_yd = y_dev;
            P->g_yh = y_host;
            P->g_yb = y_bytes;
        }
    }
    if (P->gexec && P->g_gen == P->gen && P->g_xh == x_host && P->g_xb == x_bytes &&
        P->g_xd == x_dev && P->g_yd == y_dev && P->g_yh == y_host && P->g_yb == y_bytes) {
        CG_CUDA(cudaGraphLaunch(P->gexec, s), "staged host call (graph)");
    } else {
        if (x_bytes)
            CG_CUDA(cudaMemcpyAsync(x_dev, x_host, (size_t)x_bytes, cudaMemcpyHostToDevice, s),
                    "x H2D");
        if ((rc = launch_plan(P->plan, s))) return rc;
        if (y_bytes)
            CG_CUDA(cudaMemcpyAsync(y_host, y_dev, (size_t)y_bytes, cudaMemcpyDeviceToHost, s),
                    "y D2H");
    }
    CG_CUDA(cudaStreamSynchronize(s), "staged host call");
    return CG_OK;
}

int cg_stages_set_mirror(cg_stages* P, void* const* host_ys) {
    if (!P) return fail(CG_ERR_ARG, "NULL plan");
    if (P->comm && host_ys) return fail(CG_ERR_ARG, "host mirrors are not supported on exchange plans");
    DeviceGuard guard(P->device);
    for (int i = 0; i < P->count; ++i) {
        float* h = host_ys ? static_cast<float*>(host_ys[i]) : nullptr;
        if (h) {
            // pinned (page-locked) host memory, mapped into the device address space
            cudaPointerAttributes a{};
            if (cudaPointerGetAttributes(&a, h) != cudaSuccess || a.type != cudaMemoryTypeHost ||
                !a.devicePointer) {
                cudaGetLastError();
                return fail(CG_ERR_ARG, "host_ys[%d] is not pinned, device-mapped host memory", i);
            }
            h = static_cast<float*>(a.devicePointer);
        }
        P->mirror[i] = h;
        P->plan.gp.layer[i].mirror = h;
    }
    bool any = false;
    for (int i = 0; i < P->count; ++i) any |= P->mirror[i] != nullptr;
    if (any != P->no_llc) {
        P->no_llc = any;
        int rc = replan_if_needed(P, true);
        if (rc) return rc;
    }
    ++P->gen;
    return CG_OK;
}

int cg_stages_destroy(cg_stages* P) {
    if (P && P->gexec) cudaGraphExecDestroy(P->gexec);
    delete P;
    return CG_OK;
}

int cg_comm_create(int world, int rank, int64_t bytes, int ctas, int timeout_ms, int device,
                   cg_comm** out) {
    if (!out) return fail(CG_ERR_ARG, "NULL out");
    *out = nullptr;
    if (world < 1 || world > cg::kMaxRanks)
        return fail(CG_ERR_ARG, "world %d outside 1..%d", world, cg::kMaxRanks);
    if (rank < 0 || rank >= world) return fail(CG_ERR_ARG, "rank %d outside 0..%d", rank, world - 1);
    if (bytes < 0 || timeout_ms < 0) return fail(CG_ERR_ARG, "negative bytes / timeout");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(CG_ERR_CUDA, "no CUDA device available; this library has no CPU path");
    if (device < 0) cudaGetDevice(&device);
    if (device >= ndev) return fail(CG_ERR_ARG, "device %d of %d", device, ndev);
    DeviceGuard guard(device);
    const int sms = sm_count_of(device);
    if (ctas == 0) ctas = sms;
    if (ctas < 1 || ctas > sms || ctas > cg::kMaxCtas)
        return fail(CG_ERR_ARG, "ctas %d outside 1..%d", ctas, std::min(sms, cg::kMaxCtas));
    cg_comm* c = new cg_comm;
    c->world = world;
    c->rank = rank;
    c->ctas = ctas;
    c->device = device;
    c->bytes = (bytes + 255) & ~int64_t(255);
    c->timeout_ns = (unsigned long long)timeout_ms * 1000000ull;
    // header | gathered buffers | their LL copy ((value, epoch) pairs: 2x the bytes)
    cudaError_t e = cudaMalloc(&c->base, (size_t)(cg::kXcHeader + 3 * c->bytes));
    if (e == cudaSuccess) e = cudaMemset(c->base, 0, (size_t)(cg::kXcHeader + 3 * c->bytes));
    if (e != cudaSuccess) {
        cudaFree(c->base);
        delete c;
        return cuda_fail(e, "comm region alloc");
    }
    c->peer[rank] = c->base;
    if (world == 1) c->linked = true;
    *out = c;
    return CG_OK;
}

int cg_comm_buffer(const cg_comm* c, void** out) {
    if (!c || !out) return fail(CG_ERR_ARG, "NULL comm/out");
    *out = c->base + cg::kXcHeader;
    return CG_OK;
}

int cg_comm_ipc_handle(const cg_comm* c, void* out) {
    if (!c || !out) return fail(CG_ERR_ARG, "NULL comm/out");
    static_assert(sizeof(cudaIpcMemHandle_t) == CG_IPC_HANDLE_BYTES, "IPC handle size");
    DeviceGuard guard(c->device);
    cudaIpcMemHandle_t h;
    CG_CUDA(cudaIpcGetMemHandle(&h, c->base), "IPC handle");
    std::memcpy(out, &h, sizeof(h));
    return CG_OK;
}

int cg_comm_open_peers(cg_comm* c, const void* handles) {
    if (!c || !handles) return fail(CG_ERR_ARG, "NULL comm/handles");
    if (c->linked) return fail(CG_ERR_ARG, "comm peers already set");
    DeviceGuard guard(c->device);
    const unsigned char* h = static_cast<const unsigned char*>(handles);
    for (int r = 0; r < c->world; ++r) {
        if (r == c->rank) continue;
        cudaIpcMemHandle_t ih;
        std::memcpy(&ih, h + (size_t)r * CG_IPC_HANDLE_BYTES, sizeof(ih));
        void* ptr = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&ptr, ih, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) return cuda_fail(e, "IPC open of a peer region");
        c->peer[r] = static_cast<unsigned char*>(ptr);
        c->ipc[r] = true;
    }
    c->linked = true;
    return CG_OK;
}

int cg_comm_set_peers(cg_comm* c, cg_comm* const* peers) {
    if (!c || !peers) return fail(CG_ERR_ARG, "NULL comm/peers");
    if (c->linked && c->world > 1) return fail(CG_ERR_ARG, "comm peers already set");
    for (int r = 0; r < c->world; ++r) {
        const cg_comm* q = peers[r];
        if (!q || q->world != c->world || q->rank != r || q->bytes != c->bytes || q->ctas != c->ctas)
            return fail(CG_ERR_ARG, "peers[%d] is not rank %d of a matching comm", r, r);
        if (r == c->rank && q != c) return fail(CG_ERR_ARG, "peers[%d] must be this comm", r);
    }
    for (int r = 0; r < c->world; ++r) c->peer[r] = peers[r]->base;
    c->linked = true;
    return CG_OK;
}

int cg_comm_destroy(cg_comm* c) {
    if (!c) return CG_OK;
    DeviceGuard guard(c->device);
    for (int r = 0; r < c->world; ++r)
        if (c->ipc[r]) cudaIpcCloseMemHandle(c->peer[r]);
    cudaFree(c->base);
    delete c;
    return CG_OK;
}

int cg_layer_gemm_host(cg_layer* L, const uint16_t* x, int n, float* y, int mode, void* stream) {
    if (!L || !x || !y) return fail(CG_ERR_ARG, "NULL layer/x/y");
    if (n < 1) return fail(CG_ERR_SHAPE, "x must have >= 1 column, got %d", n);
    DeviceGuard guard(L->device);
    const cg::Plan& p = L->plan;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t xb = (size_t)p.cols * n * 2, yb = (size_t)p.rows * n * 4;
    if (n > L->stage_cols) {
        cudaFree(L->x_dev);
        cudaFree(L->y_dev);
        cudaFreeHost(L->x_pin);
        cudaFreeHost(L->y_pin);
        L->x_dev = nullptr;
        L->y_dev = nullptr;
        L->x_pin = nullptr;
        L->y_pin = nullptr;
        L->stage_cols = 0;  // (a failed reallocation below must not leave a stale width)
        CG_CUDA(cudaMalloc(&L->x_dev, xb), "x staging alloc");
        CG_CUDA(cudaMalloc(&L->y_dev, yb), "y staging alloc");
        CG_CUDA(cudaHostAlloc(&L->x_pin, xb, cudaHostAllocDefault), "pinned x alloc");
        CG_CUDA(cudaHostAlloc(&L->y_pin, yb, cudaHostAllocDefault), "pinned y alloc");
        L->stage_cols = n;
    }
    std::memcpy(L->x_pin, x, xb);
    CG_CUDA(cudaMemcpyAsync(L->x_dev, L->x_pin, xb, cudaMemcpyHostToDevice, s), "x H2D");
    int rc = run_gemm(L, L->x_dev, n, L->y_dev, mode, s);
    if (rc) return rc;
    CG_CUDA(cudaMemcpyAsync(L->y_pin, L->y_dev, yb, cudaMemcpyDeviceToHost, s), "y D2H");
    CG_CUDA(cudaStreamSynchronize(s), "gemm");
    std::memcpy(y, L->y_pin, yb);
    return CG_OK;
}

int cg_layer_psumbook(cg_layer* L, const void* x, int n, float* out, void* stream) {
    if (!L || !x || !out) return fail(CG_ERR_ARG, "NULL layer/x/out");
    if (n < 1) return fail(CG_ERR_SHAPE, "x must have >= 1 column, got %d", n);
    const cg::Plan& p = L->plan;
    if (!p.fast) return fail(CG_ERR_UNSUPPORTED, "layer has no fused kernel");
    DeviceGuard guard(L->device);
    cg::DumpParams dp{};
    dp.books = L->books;
    dp.x = static_cast<const uint16_t*>(x);
    dp.cols = p.cols;
    dp.n = n;
    dp.kcount = p.kcount;
    dp.off_psum = p.smem.off_psum;
    dp.off_books = p.smem.off_books;
    dp.off_x = p.smem.off_x;
    CG_CUDA(cg::launch_psumbook_dump(p, dp, out, static_cast<cudaStream_t>(stream)),
            "psumbook dump launch");
    return CG_OK;
}

int cg_layer_unpack_codes(cg_layer* L, uint16_t* out, void* stream) {
    if (!L || !out) return fail(CG_ERR_ARG, "NULL layer/out");
    DeviceGuard guard(L->device);
    CG_CUDA(cg::launch_unpack_codes(L->plan, L->codes, L->raw16, out,
                                    static_cast<cudaStream_t>(stream)),
            "unpack launch");
    return CG_OK;
}

int cg_psumbook_build(const void* books, const void* x, int m, int b, int v, int64_t k_len, int n,
                      float* out, void* stream) {
    if (!books || !x || !out) return fail(CG_ERR_ARG, "NULL books/x/out");
    if (m < 1 || v < 1 || b < 1 || b > 16) return fail(CG_ERR_CONFIG, "bad m/v/b");
    if (k_len < 1 || k_len % v)
        return fail(CG_ERR_CONFIG, "tile width %lld not divisible by v=%d", (long long)k_len, v);
    if (n < 1) return fail(CG_ERR_SHAPE, "n must be >= 1");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(CG_ERR_CUDA, "no CUDA device available; this library has no CPU path");
    CG_CUDA(cg::launch_psumbook_build(static_cast<const uint16_t*>(books),
                                      static_cast<const uint16_t*>(x), m, b, v, k_len, n, out,
                                      static_cast<cudaStream_t>(stream)),
            "psumbook build launch");
    return CG_OK;
}

int cg_psumbook_build_f32(const float* books, const float* x, int m, int b, int v, int64_t k_len,
                          int n, float* out, void* stream) {
    if (!books || !x || !out) return fail(CG_ERR_ARG, "NULL books/x/out");
    if (m < 1 || v < 1 || b < 1 || b > 16) return fail(CG_ERR_CONFIG, "bad m/v/b");
    if (k_len < 1 || k_len % v)
        return fail(CG_ERR_CONFIG, "tile width %lld not divisible by v=%d", (long long)k_len, v);
    if (n < 1) return fail(CG_ERR_SHAPE, "n must be >= 1");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(CG_ERR_CUDA, "no CUDA device available; this library has no CPU path");
    CG_CUDA(cg::launch_psumbook_build_f32(books, x, m, b, v, k_len, n, out,
                                          static_cast<cudaStream_t>(stream)),
            "psumbook build launch");
    return CG_OK;
}

}  // extern "C"

// Diagnostics only: the batch kernel's stamps of the last launch (CG_STAMPS=1)
extern "C" int cg_debug_batch_stamps(unsigned long long* host, int64_t count) {
    if (!g_batch_stamps) return fail(CG_ERR_ARG, "no batch stamps (set CG_STAMPS=1)");
    CG_CUDA(cudaMemcpy(host, g_batch_stamps, std::min<int64_t>(count, 64 * 1024) * 8,
                       cudaMemcpyDeviceToHost),
            "stamps D2H");
    return CG_OK;
}

// Diagnostics only (not part of the ABI header): copy the per-CTA phase
// timestamps of the last fused launch (CG_STAMPS=1 at layer creation).
extern "C" int cg_debug_stamps(cg_layer* L, unsigned long long* host, int64_t count) {
    if (!L || !L->stamps) return fail(CG_ERR_ARG, "no stamps (set CG_STAMPS=1)");
    DeviceGuard guard(L->device);
    const int64_t n = std::min<int64_t>(count, (int64_t)L->sms * 128);
    CG_CUDA(cudaMemcpy(host, L->stamps, n * 8, cudaMemcpyDeviceToHost), "stamps D2H");
    return CG_OK;
}
