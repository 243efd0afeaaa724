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
    int64_t n_rb = 0;         // row blocks (tasks per slice)
    int64_t code_bytes = 0;   // prepacked code stream
    int64_t scale_bytes = 0;  // prepacked scale tiles
    int smem_bytes = 0;
};

struct GatherParams {
    const uint8_t* codes;     // prepacked code tiles
    const uint16_t* scl;      // prepacked scale tiles (binary16 bits)
    const uint16_t* books;    // (m, kcount_real, v) binary16 bits
    const uint16_t* x;        // (cols, n) binary16 bits
    float* out;               // y (rows, n) or split-K workspace (n_slices, rows, n)
    int64_t rows, cols, n_rg, n_slices, n_rb;
    int64_t out_slice_stride; // rows*n when writing the workspace, else 0
    int n, kcount, rg_per_task, lg, n_gs, flags;
};

// flags inside GatherParams
constexpr int kFlagNoPrefetch = 2;

// ---- launchers (cg_kernels.cu); all return cudaError_t of the launch ----
cudaError_t launch_prepack_codes(const Plan& p, const uint16_t* raw, uint8_t* packed,
                                 unsigned* bad, cudaStream_t s);
cudaError_t launch_prepack_scales(const Plan& p, const uint16_t* raw, uint16_t* packed,
                                  cudaStream_t s);
cudaError_t launch_check_codes(const Plan& p, const uint16_t* raw, unsigned* bad, cudaStream_t s);
cudaError_t launch_unpack_codes(const Plan& p, const uint8_t* packed, const uint16_t* raw16,
                                uint16_t* out, cudaStream_t s);
cudaError_t launch_fused_gemv(const Plan& p, const GatherParams& gp, bool pdl, cudaStream_t s);
cudaError_t launch_reduce_slices(const float* ws, float* y, int64_t count, int64_t n_slices,
                                 bool pdl, cudaStream_t s);
cudaError_t launch_psumbook_dump(const Plan& p, const GatherParams& gp, float* out,
                                 cudaStream_t s);
cudaError_t launch_strict_gemm(const Plan& p, const uint8_t* packed, const uint16_t* raw16,
                               const uint16_t* books, const uint16_t* scales, const uint16_t* x,
                               int n, float* y, cudaStream_t s);
cudaError_t launch_psumbook_build(const uint16_t* books, const uint16_t* x, int m, int b, int v,
                                  int64_t k_len, int n, float* out, cudaStream_t s);

// smem bytes / feasibility of the fused kernel for (v, m, u, kbits)
bool fused_instantiated(int v, int m, int u, int kbits);
int fused_smem_bytes(int v, int m, int u, int kbits);
int fused_max_ctas_per_sm(const Plan& p);

}  // namespace cg
