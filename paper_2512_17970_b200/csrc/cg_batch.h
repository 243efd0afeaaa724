// cg_batch.h -- K4, the batch path (n >= 2): parameters and launchers shared by
// cg_batch.cu and cg_api.cu (kept out of cg_internal.h so the batch kernel
// rebuilds without the fused kernel).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace cg {

// ---- K4 batch path (cg_batch.cu): n >= 2 columns, codebook dequantised in
//      registers into mma.sync fragments (see cg_batch.cu for the layout) ----
constexpr int kBatchRows = 32;      // rows per task (2 row tiles of 16)
constexpr int kMaxBatchGroup = 8;   // layers per batch launch
struct BatchLayer {
    const uint8_t* codes;     // batch code stream [row tile][chunk][t][lane'][16 B]
    const uint16_t* scl;      // batch scales [32-row set][group][32] binary16
    const uint16_t* books;    // (m, kcount, v) binary16
    const uint16_t* x;        // (cols, n) binary16, row stride ld: this launch's first column
    const uint16_t* x0;       // column 0 of x (16-byte aligned)
    float* y;                 // (rows, n), row stride ld
    float* ws;                // (n_slices, rows, n) partials when n_slices > 1
    int64_t rows, cols, groups, g_eff;
    int g_row, kcount;
    int n_rt, n_chunks;       // row tiles, K chunks of 128
    int ks_chunks, n_slices, n_rsets, n_tasks;
    int spg, gis;             // k16 steps per scale group (whole slice: 8*ks); groups per slice
};
struct BatchParams {
    BatchLayer layer[kMaxBatchGroup];
    int n_layers, n;          // columns of this launch (<= 32)
    int ld;                   // row stride of x and y (all columns of the call)
    int total_tasks;
    int off_tbl, off_x, off_codes[2], off_scl[2], off_red, off_bar;
    int code_tile_bytes;      // one row tile's code bytes of a task (buffer stride)
    unsigned long long* stamps;  // diagnostics: per-CTA globaltimer stamps (64 per CTA) or null
};
bool batch_supported_vm(int v, int m);
int batch_nt_for(int n);
int batch_layout(int v, int m, int kcount, int nt, int ks_chunks, int gis, BatchParams* bp);
int64_t batch_code_bytes(int64_t rows, int64_t cols, int v, int m);
int64_t batch_scale_bytes(int64_t rows, int64_t groups);
cudaError_t launch_prepack_batch(const uint16_t* raw, uint8_t* out, int64_t rows, int64_t segs,
                                 int m, int v, const uint16_t* scales, int64_t groups,
                                 uint16_t* scl_out, cudaStream_t s);
cudaError_t launch_batch_gemm(int v, int m, int nt, const BatchParams& bp, int grid, int smem,
                              cudaStream_t s, bool pdl);

}  // namespace cg
