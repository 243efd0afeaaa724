// cg_internal.h -- layer plan + kernel launchers shared by cg_api.cu and cg_kernels.cu.
//
// HBM layout of a prepacked layer:
//
//   codes  : [slice][row_group][t][chunk][lane][16 bytes]      uint8 codes
//            slice      = 32*u consecutive segments (one lane = u segments)
//            row_group  = 16 output rows
//            lane l of a warp owns segments  slice*32u + l*u + (0..u-1)
//            the lane's 16*u bytes for (slice,row_group,t) are [row 0..15][u],
//            split in u chunks of 16 bytes laid out lane-contiguous, so one
//            warp-wide 128-bit load moves 512 contiguous bytes.
//   scales : [slice][row_group][gi][16 rows]  binary16
//            gi = the scale group a lane's segments fall in, relative to the
//            slice (lanes_per_group = 2**lg consecutive lanes share one).
//
// A CTA task = (slice, block of rg_per_task row groups).  All tiles one task
// reads are contiguous, so the task can prefetch its whole weight stream to
// L2 with bulk prefetches before the Psumbook build.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace cg {

constexpr int kThreads = 512;  // fused kernel CTA size (16 warps)
constexpr int kWarps = kThreads / 32;


// One layer of a (group) launch of the fused kernel, passed by value.
struct LayerTask {
    const uint8_t* codes;     // prepacked code tiles
    const uint16_t* scl;      // prepacked scale tiles (binary16 bits)
    const uint16_t* books;    // (m, kcount, v) binary16 bits
    const uint16_t* x;        // (cols, n) binary16 bits
    const float* x32;         // or (cols, n) binary32, rounded to binary16 when staged
    float* y;                 // (rows, n) output
    float* ws;                // split-K partials (n_slices, rows, n) when n_slices > 1
    unsigned long long* tickets;  // (n_rg, n) monotonic split-K tickets
    int64_t rows, cols, n_rg, n_slices, n_rb;
    int u, rg_per_task, lg, n_gs, kcount, n_tasks;
    int stage;                // dependency stage within the launch (non-decreasing)
    int dep;                  // layer whose y this layer's x is (row-group readiness), or -1
    unsigned long long* rg_cnt;  // [0] launches completed, [1 + rg] row-group completions
                                 // (this layer is a producer for a later layer), or null
    int xchg;                 // kXchgPush | kXchgWait (row-shard exchange launches), else 0
    // LL chain (kFlagLLChain, single GPU): a producer layer (y read by a later stage
    // of the launch) writes its split-K partial rows as (value, epoch) pairs into
    // llp[slice][row] instead of reducing them into y; a consumer (llx = producer)
    // sums the partials of its x slice in slice order, spinning on the epoch -- no
    // grid barrier, no y zeroing, deterministic; the consumer with llw set writes
    // the reduced y (its tasks of row block 0)
    float2* llp;
    int llx, llw;
    int xll;                  // x is the gathered y of a layer pushed earlier in this launch:
                              // read from the LL copy (value, epoch pairs), no stage wait
    int zero_per;             // elements of y each CTA zeroes (rows * n / grid, rounded up to 4)
    float* mirror;            // host-mapped copy of y written by the kernel once the layer's
                              // stage is complete (end-to-end path without a D2H copy), or null
};

// ---- row-shard exchange (cg_comm): every rank owns one device region; a
//      layer's y (this rank's rows of a row-sharded layer) lives inside it at
//      the same offset on every rank, so peer p's copy is y + xc_delta[p].
constexpr int kXchgPush = 1;  // after the layer's stage, copy its rows to every peer
constexpr int kXchgWait = 2;  // x is a gathered buffer of an earlier launch: wait first
constexpr int kMaxRanks = 8;
constexpr int kMaxCtas = 256;
// the region's header (bytes from its base), then the gathered buffers
constexpr int kXcArrive = 0;       // u64: exchange arrivals (one per CTA per exchange per rank)
constexpr int kXcFlags = 256;      // u64[16 + kMaxCtas]: this rank's grid-barrier flags
constexpr int kXcOwnX = 4096;      // u64[kMaxCtas]: exchanges CTA c took part in
constexpr int kXcHeader = 8192;

constexpr int kMaxGroup = 16;  // layers per launch (kernel parameters ~2.7 KB)

// A launch: up to kMaxGroup layers sharing (v, m, table size) and batch width
// n, in dependency stages (layers of one stage are independent; a stage may
// read what earlier stages wrote).  CTA c runs tasks c, c+grid, ... of every
// layer of a stage in order; grid barriers separate the stages.
struct GroupParams {
    LayerTask layer[kMaxGroup];
    int n_layers;
    int n_stages;             // stage s+1 starts after every CTA finished stage s
    int n;                    // batch columns
    int flags, pf_dist;
    unsigned bar_skip;  // LL chain: bit s set = no grid barrier after stage s
    // dynamic shared-memory layout (bytes from the dynamic smem start); the
    // Psumbook sits at a 64 KB-aligned shared-window address (see cg_api.cu)
    int off_psum, off_books, off_x, off_bar, off_list, list_cap;
    int off_scl[2], off_raw[2];  // double-buffered task inputs: scale tiles, raw books | x
    int raw_x_off;            // byte offset of the raw x slice inside a raw buffer
    int off_stage[2];         // split-K staging of a task's partial rows (reduce-add), x2
    unsigned long long* grid_flags;   // per-CTA barrier flags (zero barrier, stage barriers)
    unsigned long long* stamps;  // diagnostics: per-CTA phase timestamps (8 per CTA) or null
    // row-shard exchange (null xc_local: none)
    unsigned char* xc_local;               // this rank's region base
    unsigned char* xc_peer[kMaxRanks];     // every rank's region base (self included)
    long long xc_delta[kMaxRanks];         // peer copy address - local address (bytes)
    int xc_world, xc_rank;
    unsigned long long xc_timeout_ns;      // trap a wait that exceeds it (0: wait forever)
    // LL exchange (kFlagXcLL): stage pushes write (value, epoch) pairs into every
    // rank's LL copy of the gathered buffers -- 8 bytes per float at
    // xc_ll + 2 * (byte offset in the gathered buffers) -- and consumers spin on
    // the epoch: no fence, no counter.  The launch's last exchange pushes every
    // layer's plain rows once, fenced and counted (user-visible buffers, WAIT
    // layers of later launches, overwrite protection).
    unsigned char* xc_ll;                  // this rank's LL copy
    const unsigned char* xc_gbase;         // this rank's gathered buffers (offset origin)
};

// Psumbook dump (bit-exactness check of the fused kernel's on-chip table)
struct DumpParams {
    const uint16_t* books;
    const uint16_t* x;
    int64_t cols;
    int n, kcount;
    int off_psum, off_books, off_x;
};

// flags
constexpr int kFlagNoPrefetch = 2;
constexpr int kFlagLastArriver = 4;  // a layer has more tasks than the grid: last arriver sums
constexpr int kFlagDeterministic = 16;  // split-K by tickets + ordered sums (else L2 reduce-add)
constexpr int kFlagXRegs = 32;  // x staged through registers (unaligned x / odd cols / n > 1)
constexpr int kFlagXcLL = 128;  // exchange launch: LL stage pushes (GroupParams::xc_ll)
constexpr int kFlagLLChain = 1 << 16;  // staged launch: LL partials between stages, no barriers
// contiguous task ranges: CTA c runs a stage's tasks [c*T/G, (c+1)*T/G) (not c, c+G, ...),
// so its consecutive tasks mostly share a (layer, K-slice) and reuse that slice's
// Psumbook without a rebuild (reduce-add split-K only; the host sets it)
constexpr int kFlagContig = 1 << 17;
constexpr int kFlagDbgEarlyIssue = 1 << 19;  // next task's inputs issued before the table build (A/B)
constexpr int kFlagDbgLL8 = 1 << 20;         // LL consumers poll 8 producer partials per round (A/B)
// diagnostics only (CG_DEBUG_FLAGS): wrong results, phase isolation for timing
constexpr int kFlagRowDeps = 64;  // stages ordered by row-group readiness, not grid barriers
constexpr int kFlagDirectAdd = 1 << 14;  // split-K partials red.add'ed into y even at n == 1
constexpr int kFlagDbgXcGpuScope = 1 << 15; // exchange fences at gpu scope (ranks of one GPU only)
constexpr int kFlagDbgSkipBuild = 1 << 8;   // no Psumbook build
constexpr int kFlagDbgNoLoads = 1 << 9;     // gather reuses the preloaded code tiles
constexpr int kFlagDbgSkipGather = 1 << 10; // no gather
constexpr int kFlagDbgEmpty = 1 << 11;      // return at kernel entry
constexpr int kFlagDbgNoCoop = 1 << 12;     // launch without the cooperative attribute
constexpr int kFlagDbgNoPdl = 1 << 13;      // launch without programmatic dependent launch

// shared-memory pieces of the fused kernel for (v, m, u, kbits)
struct FusedSizes {
    int psum, books, x;  // bytes
};
bool fused_instantiated(int v, int m, int u, int kbits);
bool fused_contig_instantiated(int v, int m, int u, int kbits);  // contiguous-schedule instance
bool fused_sizes(int v, int m, int u, int kbits, FusedSizes* out);

// Dynamic smem layout.  The Psumbook must start at a 64 KB-aligned address of
// the CTA's shared window so that one PRMT builds a whole lookup address; the
// dynamic area starts `reserved` bytes into the window (1 KB on sm_100).
struct SmemLayout {
    int off_psum = 0, off_books = 0, off_x = 0, off_bar = 0, off_list = 0, total = 0;
    int off_scl[2] = {0, 0}, off_raw[2] = {0, 0}, off_stage1 = 0;
};
// Pieces go first-fit into the area below the 64 KB-aligned Psumbook (the
// dynamic area starts `reserved` bytes into the CTA window), the rest after it.
//   scl_bytes / raw_bytes: one task-input buffer (two of each are placed)
//   list_bytes: fix-up list (deterministic) or split-K staging (reduce-add);
//   a second staging buffer of stage_bytes is placed for the reduce-add flush
inline bool smem_layout(const FusedSizes& z, int scl_bytes, int raw_bytes, int list_bytes,
                        int reserved, SmemLayout* L, int stage_bytes = 0) {
    auto up = [](int v, int a) { return (v + a - 1) / a * a; };
    const int kMax = 227 * 1024;
    const int kState = 3072;  // CtaState (incl. the CTA's task list)
    struct Piece {
        int* off;
        int size;
    } pieces[] = {{&L->off_books, z.books},       {&L->off_list, list_bytes},
                  {&L->off_scl[0], scl_bytes},    {&L->off_scl[1], scl_bytes},
                  {&L->off_raw[0], raw_bytes},    {&L->off_raw[1], raw_bytes},
                  {&L->off_x, z.x},               {&L->off_bar, kState},
                  {&L->off_stage1, stage_bytes}};
    const int n = (int)(sizeof(pieces) / sizeof(pieces[0]));
    // largest first
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j)
            if (pieces[j].size > pieces[i].size) {
                Piece t = pieces[i];
                pieces[i] = pieces[j];
                pieces[j] = t;
            }
    int total_small = 0;
    for (int i = 0; i < n; ++i) total_small += up(pieces[i].size, 16);
    // the Psumbook's first 64 KB-aligned slot; grow past it if nothing fits below
    const int gap = up(reserved + 1, 65536) - reserved;
    int low = 0, high = gap + z.psum;
    L->off_psum = gap;
    for (int i = 0; i < n; ++i) {
        const int sz = up(pieces[i].size, 16);
        if (low + sz <= gap) {
            *pieces[i].off = low;
            low += sz;
        } else {
            *pieces[i].off = high;
            high += sz;
        }
    }
    (void)total_small;
    L->total = high;
    return L->total <= kMax;
}


struct Plan {
    int64_t rows = 0, cols = 0, segs = 0, g_eff = 0, groups = 0;
    int v = 0, m = 0, b = 0, kcount = 0;
    int64_t g = -1;
    bool g_row = false;
    // fused (fast) path
    bool fast = false;
    int u = 0;                // segments per lane per slice
    int kbits = 0;            // table entries per sub-table in smem = 1 << kbits (4 or 8)
    int64_t slice_segs = 0;   // 32*u
    int64_t n_slices = 0;
    int64_t rows_pad = 0, n_rg = 0;
    int lg = 0;               // log2(lanes per scale group), 0..5
    int n_gs = 0;             // scale groups per slice tile = 32 >> lg
    int rg_per_task = 0;
    int rg_cap = 0;           // largest rg_per_task whose task buffers fit shared memory
    int64_t n_rb = 0;         // row blocks (tasks per slice)
    int64_t code_bytes = 0;   // prepacked code stream
    int64_t scale_bytes = 0;  // prepacked scale tiles
    int smem_bytes = 0;       // total dynamic smem of the fused kernel
    SmemLayout smem;
};

// ---- launchers (cg_kernels.cu); all return cudaError_t of the launch ----
cudaError_t launch_prepack_codes(const Plan& p, const uint16_t* raw, uint8_t* packed,
                                 unsigned* bad, cudaStream_t s);
cudaError_t launch_prepack_scales(const Plan& p, const uint16_t* raw, uint16_t* packed,
                                  cudaStream_t s);
cudaError_t launch_check_codes(const Plan& p, const uint16_t* raw, unsigned* bad, cudaStream_t s);
cudaError_t launch_unpack_codes(const Plan& p, const uint8_t* packed, const uint16_t* raw16,
                                uint16_t* out, cudaStream_t s);
// group launch: all layers share (v, m, kbits); grid = persistent CTAs
cudaError_t launch_group_gemv(int v, int m, int u, int kbits, const GroupParams& gp, int grid,
                              int smem, bool pdl, cudaStream_t s);
cudaError_t launch_psumbook_dump(const Plan& p, const DumpParams& dp, float* out, cudaStream_t s);
cudaError_t launch_strict_gemm(const Plan& p, const uint8_t* packed, const uint16_t* raw16,
                               const uint16_t* books, const uint16_t* scales, const uint16_t* x,
                               int n, float* y, cudaStream_t s);
cudaError_t launch_unpack_packed(const uint8_t* packed, int64_t plane_bytes, int m,
                                 int64_t per_plane, int b, uint16_t* out, cudaStream_t s);
cudaError_t launch_psumbook_build(const uint16_t* books, const uint16_t* x, int m, int b, int v,
                                  int64_t k_len, int n, float* out, cudaStream_t s);
cudaError_t launch_psumbook_build_f32(const float* books, const float* x, int m, int b, int v,
                                      int64_t k_len, int n, float* out, cudaStream_t s);



}  // namespace cg
