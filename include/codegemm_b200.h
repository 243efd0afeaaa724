/*
 * codegemm_b200.h -- C ABI of the B200-native CodeGEMM decode path.
 *
 * Plain pointers and sizes only (no torch / CUDA runtime types in the
 * signatures: streams are passed as `void*` holding a cudaStream_t, NULL =
 * the legacy default stream).  The library is libcodegemm_b200.so, built for
 * sm_100a only; there is no CPU fallback -- every compute entry point fails
 * with CG_ERR_CUDA when no B200 is present.
 *
 * Each entry point replaces one piece of the reference's Python operator
 * path (/root/reference/pkg/src/codegemm/...):
 *
 *   cg_layer_create       QuantizedLayer as the engines consume it:
 *                         CodePlane (quantizer.py:135-145), Codebook
 *                         (quantizer.py:87-113), ScalePlane (quantizer.py:116-132),
 *                         segment_groups (quantizer.py:195-199).  Uploads and
 *                         prepacks the planes once (weights are static).
 *   cg_layer_gemm         codegemm_gemm(q, x, tiles, threads) (engines.py:245-316)
 *                         on device buffers; CG_MODE_STRICT reproduces its
 *                         binary32 operation order bit for bit (engines.py:15-22),
 *                         CG_MODE_FAST is the fused lookup kernel (tolerance parity).
 *   cg_layer_gemm_host    the same call with HOST buffers (the drop-in used by
 *                         the Python shim: x in, y out, copies included).
 *   cg_layer_psumbook     the fused kernel's on-chip Psumbook, dumped in the layout
 *                         of _psum_tables (engines.py:115-134) for bit-exact checks.
 *   cg_psumbook_build     standalone Psumbook build, build_psumbook / _psum_tables
 *                         (engines.py:115-156).
 *   cg_layer_unpack_codes inverse of the device prepack; returns the per-row gather
 *                         indices as uint16 planes (CodePlane.codes) for bit-exact
 *                         index parity (pack/unpack: quantizer.py:471-497).
 *
 * Errors: every int-returning function returns CG_OK (0) or a CG_ERR_* code
 * and records a message retrievable with cg_last_error() (thread-local).  The
 * codes map onto the reference exception classes (errors.py:4-37):
 * CG_ERR_CONFIG -> ConfigError, CG_ERR_SHAPE -> ShapeError,
 * CG_ERR_INTEGRITY -> IntegrityError.
 *
 * Threading: functions are reentrant across layers and streams; one layer
 * handle owns a split-K workspace, so calls on the SAME handle must be
 * ordered on one stream (or serialised by the caller).
 */
#ifndef CODEGEMM_B200_H
#define CODEGEMM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CG_ABI_VERSION 1

#define CG_OK 0
#define CG_ERR_CONFIG 1      /* bad hyper-parameters / tiling       -> ConfigError    */
#define CG_ERR_SHAPE 2       /* inconsistent operand shapes         -> ShapeError     */
#define CG_ERR_INTEGRITY 3   /* invalid layer contents (code range) -> IntegrityError */
#define CG_ERR_CUDA 4        /* CUDA runtime / launch failure, no device              */
#define CG_ERR_UNSUPPORTED 5 /* config outside the requested mode's kernels           */
#define CG_ERR_ARG 6         /* NULL / out-of-range argument                          */

#define CG_MODE_AUTO 0   /* FAST when the config has a fused kernel, else STRICT      */
#define CG_MODE_FAST 1   /* fused Psumbook + code-gather kernel (fp32 accumulate)      */
#define CG_MODE_STRICT 2 /* reference operation order: bit-identical to codegemm_gemm  */

#define CG_X_F16 0 /* x stored as binary16                                              */
#define CG_X_F32 1 /* x stored as float32, rounded to binary16 when read (staged chain) */

/* option flags for cg_layer_options.flags */
#define CG_OPT_NO_PDL 1        /* launch without programmatic dependent launch        */
#define CG_OPT_NO_L2_PREFETCH 2 /* skip the bulk L2 prefetch of the CTA's code tiles   */
#define CG_OPT_BATCH_EAGER 8  /* build the batch (n >= 2) code stream at creation, not on the
                                 first call with n >= 2                                  */
#define CG_OPT_NO_BATCH 16    /* n >= 2 runs the per-column Psumbook lookups (comparison)  */
#define CG_OPT_DETERMINISTIC 4  /* split-K partials summed in a fixed order (run-to-run
                                   bit-identical); default adds them in L2 (faster,
                                   last-bit differences between runs)                  */

typedef struct cg_layer cg_layer;
typedef struct cg_comm cg_comm;
typedef struct cg_stages cg_stages;

#define CG_IPC_HANDLE_BYTES 64 /* cudaIpcMemHandle_t */

/* cg_gemm_stages_xchg per-layer flags */
#define CG_XCHG_PUSH 1 /* y is this rank's rows of a row-sharded layer, inside the comm
                          buffer: after its stage they are copied to every peer      */
#define CG_XCHG_WAIT 2 /* x (CG_X_F32, inside the comm buffer) was gathered by earlier
                          launches: wait for every rank's rows before reading it      */

typedef struct cg_layer_options {
    int u;             /* segments per lane per K-slice (1, 2, 4); 0 = planner choice */
    int rg_per_task;   /* 16-row groups per CTA task; 0 = planner choice              */
    int flags;         /* CG_OPT_*                                                     */
    int device;        /* CUDA device ordinal; -1 = current device                    */
} cg_layer_options;

typedef struct cg_layer_info {
    int64_t rows, cols;
    int v, m, b;
    int64_t g;              /* as given (-1 = one scale per row)                       */
    int fast_supported;     /* 1 if CG_MODE_FAST has a kernel for this config           */
    int u;                  /* chosen segments-per-lane                                */
    int rg_per_task;        /* chosen 16-row groups per CTA task                       */
    int64_t n_slices;       /* K-slices of 32*u segments                               */
    int64_t n_tasks;        /* CTAs of the fused kernel                                */
    int smem_bytes;         /* dynamic shared memory of the fused kernel                */
    int launches_fast;      /* kernels one CG_MODE_FAST call launches (1 or 2)         */
    int64_t device_bytes;   /* device memory owned by the handle                       */
    int64_t algorithmic_bytes; /* codes (b bits) + scales + codebooks for one call,
                                   excluding x and y                    */
    int batch_supported;    /* 1 if n >= 2 calls run the batch kernel (K4: codebook
                               dequantised into mma.sync fragments, cg_batch.cu)       */
    int batch_ready;        /* 1 once the batch code stream exists (first n >= 2 call) */
} cg_layer_info;

int cg_abi_version(void);
const char* cg_last_error(void);

/* Number of CUDA devices visible (0 when none); never fails. */
int cg_device_count(void);

/*
 * Create a device-resident layer from HOST arrays in the reference layout.
 *   codes[t]  : (rows, cols/v) uint16, row-major, t < m    (CodePlane.codes)
 *   books[t]  : (2**b, v) binary16 bit patterns           (Codebook.entries)
 *   scales    : (rows, cols/g_eff) binary16 bit patterns  (ScalePlane.scales)
 *   g         : group size, -1 = one scale per row
 * A row shard is created by passing row-offset pointers and the shard's rows.
 * opts may be NULL (planner defaults).
 */
int cg_layer_create(const uint16_t* const* codes, const uint16_t* const* books,
                    const uint16_t* scales, int64_t rows, int64_t cols, int v, int m, int b,
                    int64_t g, const cg_layer_options* opts, cg_layer** out);
/*
 * The same from the CGMM container's code planes as stored (storage.py:95-160,
 * quantizer.py:471-497): planes[t] holds rows*(cols/v) codes of b bits each,
 * least-significant bit first, padded to a whole byte.  The planes cross PCIe
 * at b bits per code and are unpacked and prepacked on the device.
 */
int cg_layer_create_packed(const uint8_t* const* planes, const uint16_t* const* books,
                           const uint16_t* scales, int64_t rows, int64_t cols, int v, int m,
                           int b, int64_t g, const cg_layer_options* opts, cg_layer** out);
int cg_layer_destroy(cg_layer* layer);
int cg_layer_query(const cg_layer* layer, cg_layer_info* info);

/*
 * y = W x on device buffers, stream-ordered, asynchronous.
 *   x : (cols, n) binary16, row-major (Matrix layout: one column per token)
 *   y : (rows, n) float32, row-major
 * n == 1 runs the fused Psumbook kernel; n >= 2 (CG_MODE_FAST / AUTO) the batch
 * kernel when batch_supported (its code stream is built on the first such call,
 * which then allocates and synchronises), else one Psumbook per column.  Both
 * batch outputs are deterministic (split-K partials summed in slice order).
 */
int cg_layer_gemm(cg_layer* layer, const void* x, int n, float* y, int mode, void* stream);

/*
 * Grouped launch: y_i = W_i x_i for `count` (1..16) independent layers in ONE
 * launch of the fused kernel (e.g. the q/k/v or gate/up projections of a
 * decoder block, which read the same x).  Layers must share v, m, the code
 * width class (b <= 4 or b <= 8) and the device, and must all have
 * fast_supported.  Device buffers, n columns each, stream-ordered.  With
 * CG_OPT_DETERMINISTIC layers the outputs are bit-identical to separate
 * cg_layer_gemm calls (CG_MODE_FAST); without it split-K partials are added in
 * L2 in arrival order (within the fast-mode tolerance, not bit-reproducible).
 */
int cg_gemm_group(cg_layer* const* layers, const void* const* xs, float* const* ys, int count,
                  int n, void* stream);

/*
 * Dependency-staged launch: one persistent launch of the fused kernel runs
 * `count` (1..16) layers in stages; stages[i] is layer i's stage (starts at 0,
 * non-decreasing, steps of at most 1).  Layers of one stage are independent
 * (a grouped launch); a stage may read what earlier stages wrote -- e.g. a
 * decoder-block chain {q} -> {o} -> {gate,up} -> {down}.  x_dtypes[i] (NULL =
 * all CG_X_F16) says how xs[i] is stored: CG_X_F16 (cols, n) binary16, or
 * CG_X_F32 (cols, n) float32 -- typically an earlier stage's y in the same
 * launch -- rounded to binary16 (round-to-nearest-even) as it is read, the
 * reference's fp16 boundary rounding (cli.py:136).  The kernel's grid barrier
 * orders a stage's reads after the earlier stages' writes.  Same layer
 * requirements as cg_gemm_group, plus one tiling u for all layers
 * (cg_layer_options.u).  With CG_OPT_DETERMINISTIC layers the outputs are
 * bit-identical to separate cg_layer_gemm calls in stage order on the rounded
 * inputs.  An x may overlap only the y of an EARLIER stage: a y written in the
 * same or a later stage is rejected (CG_ERR_ARG) -- split-K outputs are zeroed
 * by every CTA when the launch starts, before stage 0 reads its x.
 */
int cg_gemm_stages(cg_layer* const* layers, const void* const* xs, const int* x_dtypes,
                   float* const* ys, const int* stages, int count, int n, void* stream);

/*
 * Row-shard exchange (the per-layer all-gather of the
 * row-sharded layers, fused into the staged kernel over NVLink peer memory).
 * Each rank (one process per GPU, or several ranks of one process for tests)
 * creates a comm whose device buffer holds the GATHERED outputs (all rows of
 * a sharded layer, same offsets on every rank).  A rank's layer writes its rows
 * into that buffer (ys[i] = buffer + rank's row offset) with CG_XCHG_PUSH;
 * once the layer's stage is complete on this rank, the kernel stores those rows
 * into every peer's buffer (P2P stores) and releases a system-scope arrival
 * counter on every rank.  A later stage whose x is the gathered buffer waits
 * for every rank's arrivals before reading it (no NCCL call, no extra launch);
 * a later launch reading it marks the layer CG_XCHG_WAIT.  Launch-completion
 * counters keep a rank from overwriting a peer's buffer before that peer has
 * finished its previous launch.  Every rank must issue the same sequence of
 * comm launches (the counters count arrivals of `world` ranks x `ctas` CTAs).
 *   world, rank : 1..8 ranks;  bytes: gathered-buffer bytes (same on every rank)
 *   ctas        : CTAs per launch (0 = every SM); ranks of one GPU split it
 *   timeout_ms  : a wait on peers longer than this traps the kernel (0 = none)
 */
int cg_comm_create(int world, int rank, int64_t bytes, int ctas, int timeout_ms, int device,
                   cg_comm** out);
int cg_comm_buffer(const cg_comm* comm, void** out);  /* the gathered-buffer base */
/* 64-byte IPC handle of this rank's region; exchange them (e.g. all_gather_object) */
int cg_comm_ipc_handle(const cg_comm* comm, void* out);
/* map the peers' regions: handles = world x CG_IPC_HANDLE_BYTES in rank order */
int cg_comm_open_peers(cg_comm* comm, const void* handles);
/* ranks of one process: peers[r] = rank r's comm (peers[rank] == comm) */
int cg_comm_set_peers(cg_comm* comm, cg_comm* const* peers);
int cg_comm_destroy(cg_comm* comm);
/* cg_gemm_stages plus xchg[i] = CG_XCHG_* flags of layer i; the launch runs comm's grid */
int cg_gemm_stages_xchg(cg_layer* const* layers, const void* const* xs, const int* x_dtypes,
                        float* const* ys, const int* stages, const int* xchg, int count, int n,
                        cg_comm* comm, void* stream);

/*
 * Prepared staged launch: cg_gemm_stages / cg_gemm_stages_xchg planned once
 * (task split, shared-memory layout, kernel parameters) for fixed buffers --
 * a decode loop's per-step call costs one kernel launch.  xchg and comm may
 * be NULL (no exchange).  The plan is rebuilt automatically if a layer's
 * split-K workspace was reallocated by a wider call in between.
 *   cg_stages_launch   : the launch on `stream` (device buffers, asynchronous)
 *   cg_stages_run_host : end to end with host buffers: x_bytes from x_host to
 *                        x_dev (the device buffer the plan's inputs live in),
 *                        the launch, y_bytes from y_dev to y_host, synchronise.
 *                        Use pinned host memory for asynchronous copies.
 */
int cg_stages_prepare(cg_layer* const* layers, const void* const* xs, const int* x_dtypes,
                      float* const* ys, const int* stages, const int* xchg, int count, int n,
                      cg_comm* comm, cg_stages** out);
int cg_stages_launch(cg_stages* plan, void* stream);
int cg_stages_run_host(cg_stages* plan, const void* x_host, int64_t x_bytes, void* x_dev,
                       const void* y_dev, void* y_host, int64_t y_bytes, void* stream);
int cg_stages_destroy(cg_stages* plan);
/*
 * Host mirrors of a prepared plan's outputs: host_ys[i] (pinned, device-mapped
 * host memory such as cudaHostAlloc / torch pin_memory; NULL = none) receives
 * layer i's y from the kernel itself once the layer's stage is complete, so the
 * copies overlap the later stages and cg_stages_run_host needs no D2H copy
 * (y_bytes = 0).  The last stage's copy costs one more grid barrier.  host_ys
 * = NULL removes the mirrors.  Not for exchange plans.
 */
int cg_stages_set_mirror(cg_stages* plan, void* const* host_ys);

/* Same with HOST buffers: copies x in, runs, copies y out, synchronises. */
int cg_layer_gemm_host(cg_layer* layer, const uint16_t* x, int n, float* y, int mode,
                       void* stream);

/*
 * Psumbook of the fused kernel for input x (device (cols, n) binary16), written
 * to out (device float32, (m, cols/v, 2**b, n) -- _psum_tables layout).
 * Requires fast_supported.
 */
int cg_layer_psumbook(cg_layer* layer, const void* x, int n, float* out, void* stream);

/*
 * Per-row gather indices recovered from the prepacked device layout:
 * out (device uint16, (m, rows, cols/v)).
 */
int cg_layer_unpack_codes(cg_layer* layer, uint16_t* out, void* stream);

/*
 * Standalone Psumbook build on device buffers:
 *   books : m x (2**b, v) binary16 contiguous;  x : (k_len, n) binary16
 *   out   : (m, k_len/v, 2**b, n) float32
 */
int cg_psumbook_build(const void* books, const void* x, int m, int b, int v, int64_t k_len,
                      int n, float* out, void* stream);
/*
 * The same from binary32 books and x (engines.py:137-156 widens any float
 * input to binary32): each entry is ((0 + c0*x0) + c1*x1) + ... with every
 * product and sum rounded separately, as numpy does -- bit-exact for inputs
 * that are not binary16-representable too.
 */
int cg_psumbook_build_f32(const float* books, const float* x, int m, int b, int v, int64_t k_len,
                          int n, float* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* CODEGEMM_B200_H */
