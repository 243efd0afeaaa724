// cg_kernels.cu -- sm_100a kernels of the B200 CodeGEMM decode path.
//
//   prepack / unpack   K3: uint16 CodePlanes <-> lane-tiled uint8 code stream
//   fused_gemv         K2: per CTA task, build the slice Psumbook in shared memory
//                      (bit-exact binary32 dot products, engines.py:115-134), then
//                      stream the task's code tiles from HBM with 128-bit loads and
//                      gather-accumulate (engines.py:286-294) with per-group scales
//                      and a warp transpose-reduction.  Weights are never dequantised.
//   reduce_slices      deterministic split-K sum of per-slice partial outputs
//   strict_gemm        reference operation order, bit-identical to codegemm_gemm
//   psumbook_build     K1 standalone (m, K/v, 2**b, n) table, bit-exact
//   psumbook_dump      the fused kernel's smem table, dumped for bit-exact checks
//
// See DESIGN.md for the layout and the roofline of each kernel.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "cg_internal.h"

namespace cg {
namespace {

__device__ __forceinline__ float h2f(uint16_t h) { return __half2float(__ushort_as_half(h)); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ float lds_f32(uint32_t addr) {
    float v;
    asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}

// streaming 128-bit load: read once, do not keep in L1
__device__ __forceinline__ uint4 ldg_stream_v4(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Programmatic dependent launch: everything before pdl_wait() may overlap the
// previous kernel in the stream, so only weights (never written by anyone) are
// touched before it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" :::);
}

__device__ __forceinline__ uint32_t word_of(const uint4& q, int i) {
    return i == 0 ? q.x : (i == 1 ? q.y : (i == 2 ? q.z : q.w));
}

// ---------------------------------------------------------------------------
// code addressing in the prepacked stream (cg_internal.h)
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t packed_index(int64_t t, int64_t r, int64_t seg, int m, int u,
                                                int64_t n_rg) {
    const int64_t slice_segs = 32 * u;
    const int64_t slice = seg / slice_segs;
    const int64_t within = seg - slice * slice_segs;
    const int64_t lane = within / u;
    const int64_t uu = within - lane * u;
    const int64_t rg = r >> 4;
    const int64_t rr = r & 15;
    const int64_t idx = rr * u + uu;  // position in the lane's [row][u] bytes
    const int64_t tile = ((slice * n_rg + rg) * m + t) * (int64_t)(u * 512);
    return tile + (idx >> 4) * 512 + lane * 16 + (idx & 15);
}

// ---------------------------------------------------------------------------
// K3: prepack / unpack / validation
// ---------------------------------------------------------------------------
__global__ void prepack_codes_kernel(const uint16_t* __restrict__ raw, uint8_t* __restrict__ out,
                                     int64_t total, int64_t rows, int64_t segs, int m, int u,
                                     int64_t n_rg, uint32_t code_limit,
                                     unsigned* __restrict__ bad) {
    // one thread per output byte, decoding (slice, rg, t, chunk, lane, byte)
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
         o += (int64_t)gridDim.x * blockDim.x) {
        const int64_t tile_bytes = (int64_t)u * 512;
        int64_t rest = o;
        const int64_t in_tile = rest % tile_bytes;
        rest /= tile_bytes;
        const int64_t t = rest % m;
        rest /= m;
        const int64_t rg = rest % n_rg;
        const int64_t slice = rest / n_rg;
        const int64_t chunk = in_tile / 512;
        const int64_t lane = (in_tile % 512) / 16;
        const int64_t idx = chunk * 16 + (in_tile % 16);
        const int64_t rr = idx / u, uu = idx % u;
        const int64_t r = rg * 16 + rr;
        const int64_t seg = slice * 32 * u + lane * u + uu;
        uint8_t val = 0;
        if (r < rows && seg < segs) {
            const uint16_t c = raw[(t * rows + r) * segs + seg];
            if (c >= code_limit) atomicOr(bad, 1u);
            val = static_cast<uint8_t>(c);
        }
        out[o] = val;
    }
}

__global__ void prepack_scales_kernel(const uint16_t* __restrict__ raw, uint16_t* __restrict__ out,
                                      int64_t total, int64_t rows, int64_t groups, int64_t n_rg,
                                      int n_gs, int64_t slice_elems, int64_t g_eff, int lg) {
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
         o += (int64_t)gridDim.x * blockDim.x) {
        int64_t rest = o;
        const int64_t rr = rest % 16;
        rest /= 16;
        const int64_t gi = rest % n_gs;
        rest /= n_gs;
        const int64_t rg = rest % n_rg;
        const int64_t slice = rest / n_rg;
        const int64_t r = rg * 16 + rr;
        // first element of the lanes that own group gi within this slice
        const int64_t lanes_per_group = 1LL << lg;
        const int64_t elem = slice * slice_elems + gi * lanes_per_group * (slice_elems / 32);
        const int64_t grp = elem / g_eff;
        uint16_t val = 0;
        if (r < rows && grp < groups) val = raw[r * groups + grp];
        out[o] = val;
    }
}

__global__ void check_codes_kernel(const uint16_t* __restrict__ raw, int64_t total,
                                   uint32_t code_limit, unsigned* __restrict__ bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x)
        if (raw[i] >= code_limit) atomicOr(bad, 1u);
}

__global__ void unpack_codes_kernel(const uint8_t* __restrict__ packed,
                                    const uint16_t* __restrict__ raw16, uint16_t* __restrict__ out,
                                    int64_t rows, int64_t segs, int m, int u, int64_t n_rg) {
    const int64_t total = (int64_t)m * rows * segs;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (raw16) {
            out[i] = raw16[i];
        } else {
            const int64_t seg = i % segs;
            const int64_t r = (i / segs) % rows;
            const int64_t t = i / (segs * rows);
            out[i] = packed[packed_index(t, r, seg, m, u, n_rg)];
        }
    }
}

// ---------------------------------------------------------------------------
// Psumbook build into shared memory (shared by the fused kernel and the dump)
//
// smem table of sub-table j = t*U + u  (t = codebook, u = segment-in-lane):
//   region j>>1, 256-byte row per code, half j&1 of the row, lane-major floats
//   psum[(j>>1)][code][j&1][lane]  -> byte offset (code<<8) | ((j&1)<<7) | (lane<<2)
// so the gather addresses an entry with one PRMT and every lane hits its own
// bank whatever the code (conflict-free lookups).
//
// Each entry = ((+0 + c0*x0) + c1*x1) + ...: fmaf with an exact product is the
// reference's separate multiply-then-add (engines.py:126-133), bit for bit.
// ---------------------------------------------------------------------------
template <int V, int M, int U, int KB>
struct FusedShape {
    static constexpr int kSub = M * U;
    static constexpr int kRegions = (kSub + 1) / 2;
    static constexpr int kCodes = 1 << KB;
    static constexpr int kRegionFloats = kCodes * 64;
    static constexpr int kPsumFloats = kRegions * kRegionFloats;
    static constexpr int kBookFloats = M * kCodes * V;
    static constexpr int kXFloats = 32 * U * V;
    static constexpr int kSmemBytes = 4 * (kPsumFloats + kBookFloats + kXFloats);
    static constexpr int kTileBytes = M * U * 512;  // codes per (slice, row group)
};

template <int V, int M, int U, int KB>
__device__ __forceinline__ void build_psumbook_smem(float* psum, const float* books32,
                                                    const float* x32, int kcount, int tid) {
    using S = FusedShape<V, M, U, KB>;
    const int lane = tid & 31, warp = tid >> 5;
    const int q = lane & 7;     // this thread writes lanes 4q..4q+3 of a code row
    const int csub = lane >> 3; // 4 codes per warp per pass
#pragma unroll 1
    for (int j = 0; j < S::kSub; ++j) {
        const int t = j / U, uu = j % U;
        float xv[4][V];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int k = 0; k < V; ++k) xv[i][k] = x32[((4 * q + i) * U + uu) * V + k];
        float* dst = psum + (j >> 1) * S::kRegionFloats + (j & 1) * 32 + q * 4;
        const float* bk = books32 + t * S::kCodes * V;
#pragma unroll 2
        for (int c = csub + 4 * warp; c < kcount; c += 4 * kWarps) {
            float cv[V];
#pragma unroll
            for (int k = 0; k < V; ++k) cv[k] = bk[c * V + k];
            float e[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                float acc = fmaf(cv[0], xv[i][0], 0.0f);
#pragma unroll
                for (int k = 1; k < V; ++k) acc = fmaf(cv[k], xv[i][k], acc);
                e[i] = acc;
            }
            *reinterpret_cast<float4*>(dst + c * 64) = make_float4(e[0], e[1], e[2], e[3]);
        }
    }
}

// stage codebooks and the slice of x (column `col`) into smem as binary32
template <int V, int M, int U, int KB>
__device__ __forceinline__ void stage_books(float* books32, const uint16_t* books, int kcount,
                                            int tid) {
    using S = FusedShape<V, M, U, KB>;
    for (int i = tid; i < M * kcount * V; i += kThreads) {
        const int t = i / (kcount * V);
        const int rest = i - t * kcount * V;
        books32[t * S::kCodes * V + rest] = h2f(books[i]);
    }
}

template <int V, int M, int U, int KB>
__device__ __forceinline__ void stage_x(float* x32, const uint16_t* x, int64_t slice, int64_t cols,
                                        int n, int col, int tid) {
    using S = FusedShape<V, M, U, KB>;
    const int64_t e0 = slice * S::kXFloats;
    for (int i = tid; i < S::kXFloats; i += kThreads) {
        const int64_t e = e0 + i;
        x32[i] = e < cols ? h2f(x[e * n + col]) : 0.0f;
    }
}

// ---------------------------------------------------------------------------
// warp transpose-reduction helpers
//
// a[0..CNT) holds one partial per row for this lane; a halving step with xor
// mask `mk` leaves CNT/2 values: the lane keeps the upper half of the rows if
// (lane & mk) else the lower half, and adds its partner's copy of those rows.
// After the steps for masks 1,2,4,8 a lane holds the row
// bit0*8 + bit1*4 + bit2*2 + bit3 summed over the 16 lanes sharing bit4.
// ---------------------------------------------------------------------------
template <int CNT>
__device__ __forceinline__ void halve(float (&a)[16], int lane, int mk) {
    const bool up = (lane & mk) != 0;
#pragma unroll
    for (int i = 0; i < CNT / 2; ++i) {
        const float lo = a[i], hi = a[i + CNT / 2];
        const float send = up ? lo : hi;
        const float keep = up ? hi : lo;
        a[i] = keep + __shfl_xor_sync(0xffffffffu, send, mk);
    }
}

template <int CNT>
__device__ __forceinline__ void apply_scales(float (&a)[16], const float (&sc)[16]) {
#pragma unroll
    for (int i = 0; i < CNT; ++i) a[i] *= sc[i];
}

// load this lane's CNT scale values (binary16) for rows base..base+CNT-1
template <int CNT>
__device__ __forceinline__ void load_scales(float (&sc)[16], const uint16_t* p) {
    if constexpr (CNT == 16) {
        const uint4 a = *reinterpret_cast<const uint4*>(p);
        const uint4 b = *reinterpret_cast<const uint4*>(p + 8);
        const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
            sc[2 * i] = f.x;
            sc[2 * i + 1] = f.y;
        }
    } else if constexpr (CNT == 8) {
        const uint4 a = *reinterpret_cast<const uint4*>(p);
        const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
            sc[2 * i] = f.x;
            sc[2 * i + 1] = f.y;
        }
    } else if constexpr (CNT == 4) {
        const uint2 a = *reinterpret_cast<const uint2*>(p);
        float2 f = __half22float2(*reinterpret_cast<const __half2*>(&a.x));
        sc[0] = f.x;
        sc[1] = f.y;
        f = __half22float2(*reinterpret_cast<const __half2*>(&a.y));
        sc[2] = f.x;
        sc[3] = f.y;
    } else if constexpr (CNT == 2) {
        const uint32_t a = *reinterpret_cast<const uint32_t*>(p);
        const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&a));
        sc[0] = f.x;
        sc[1] = f.y;
    } else {
        sc[0] = h2f(*p);
    }
}

// ---------------------------------------------------------------------------
// K2: fused Psumbook build + code-gather accumulate
// ---------------------------------------------------------------------------
template <int V, int M, int U, int KB>
__global__ void __launch_bounds__(kThreads, 1) fused_gemv_kernel(const GatherParams p) {
    using S = FusedShape<V, M, U, KB>;
    extern __shared__ __align__(16) float smem[];
    float* psum = smem;
    float* books32 = smem + S::kPsumFloats;
    float* x32 = books32 + S::kBookFloats;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t task = blockIdx.x;
    const int64_t slice = task / p.n_rb;
    const int64_t rb = task - slice * p.n_rb;
    const int col = blockIdx.y;
    const int64_t rg0 = rb * p.rg_per_task;
    const int64_t rg1 = min(rg0 + (int64_t)p.rg_per_task, p.n_rg);
    const uint8_t* tiles = p.codes + slice * p.n_rg * (int64_t)S::kTileBytes;

    // 1. put this task's whole code stream in flight towards L2 (weights only)
    if (!(p.flags & kFlagNoPrefetch) && warp == kWarps - 1) {
        const uint8_t* beg = tiles + rg0 * S::kTileBytes;
        const int64_t bytes = (rg1 - rg0) * S::kTileBytes;
        constexpr int64_t kChunk = 32768;
        for (int64_t off = lane * kChunk; off < bytes; off += 32 * kChunk)
            prefetch_l2_bulk(beg + off, (uint32_t)min(kChunk, bytes - off));
    }
    stage_books<V, M, U, KB>(books32, p.books, p.kcount, tid);
    // 2. x may be produced by the previous kernel in the stream
    pdl_wait();
    stage_x<V, M, U, KB>(x32, p.x, slice, p.cols, p.n, col, tid);
    __syncthreads();
    build_psumbook_smem<V, M, U, KB>(psum, books32, x32, p.kcount, tid);
    __syncthreads();
    pdl_launch_dependents();

    // 3. gather: warp w takes row groups rg0+w, rg0+w+16, ...
    const uint32_t lb[2] = {(uint32_t)lane << 2, ((uint32_t)lane << 2) | 0x80u};
    const uint32_t psum_base = smem_u32(psum);
    const int lg = p.lg;
    const int ls = lg < 4 ? lg : 4;
    int sbase = 0;  // first row of this lane's scale run after `ls` halving steps
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (j < ls && (lane >> j & 1)) sbase += 8 >> j;
    const int gi = lg >= 5 ? 0 : (lane >> lg);
    const int out_row = (lane & 1) * 8 + (lane >> 1 & 1) * 4 + (lane >> 2 & 1) * 2 + (lane >> 3 & 1);
    float* out = p.out + slice * p.out_slice_stride;

    int64_t rg = rg0 + warp;
    uint4 cw[M][U];
    if (rg < rg1) {
        const uint8_t* tp = tiles + rg * S::kTileBytes + lane * 16;
#pragma unroll
        for (int t = 0; t < M; ++t)
#pragma unroll
            for (int c = 0; c < U; ++c) cw[t][c] = ldg_stream_v4(tp + (t * U + c) * 512);
    }
    for (; rg < rg1; rg += kWarps) {
        // scales for this row group (small, L2/L1 resident)
        float sc[16];
        const uint16_t* sp = p.scl + ((slice * p.n_rg + rg) * p.n_gs + gi) * 16 + sbase;
        switch (ls) {
            case 0: load_scales<16>(sc, sp); break;
            case 1: load_scales<8>(sc, sp); break;
            case 2: load_scales<4>(sc, sp); break;
            case 3: load_scales<2>(sc, sp); break;
            default: load_scales<1>(sc, sp); break;
        }
        // software pipeline: next row group's codes
        uint4 nw[M][U];
        const int64_t rgn = rg + kWarps;
        if (rgn < rg1) {
            const uint8_t* tp = tiles + rgn * S::kTileBytes + lane * 16;
#pragma unroll
            for (int t = 0; t < M; ++t)
#pragma unroll
                for (int c = 0; c < U; ++c) nw[t][c] = ldg_stream_v4(tp + (t * U + c) * 512);
        }
        // lookups: a[r] = sum over (t, u) of psum_t[seg(lane,u)][code]
        float a[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            float s = 0.0f;
#pragma unroll
            for (int t = 0; t < M; ++t)
#pragma unroll
                for (int uu = 0; uu < U; ++uu) {
                    constexpr int dummy = 0;
                    (void)dummy;
                    const int idx = r * U + uu;
                    const uint32_t w = word_of(cw[t][idx >> 4], (idx >> 2) & 3);
                    const int j = t * U + uu;
                    const uint32_t off =
                        __byte_perm(w, lb[j & 1], 0x5504u | ((uint32_t)(idx & 3) << 4));
                    const float val =
                        lds_f32(psum_base + off + (uint32_t)((j >> 1) * S::kRegionFloats * 4));
                    s = (t == 0 && uu == 0) ? val : s + val;
                }
            a[r] = s;
        }
        // reduce across the lanes of a scale group, scale, finish the reduction
        if (lg == 0) apply_scales<16>(a, sc);
        halve<16>(a, lane, 1);
        if (lg == 1) apply_scales<8>(a, sc);
        halve<8>(a, lane, 2);
        if (lg == 2) apply_scales<4>(a, sc);
        halve<4>(a, lane, 4);
        if (lg == 3) apply_scales<2>(a, sc);
        halve<2>(a, lane, 8);
        if (lg == 4) apply_scales<1>(a, sc);
        a[0] += __shfl_xor_sync(0xffffffffu, a[0], 16);
        if (lg >= 5) a[0] *= sc[0];
        if (lane < 16) {
            const int64_t r = rg * 16 + out_row;
            if (r < p.rows) out[r * p.n + col] = a[0];
        }
#pragma unroll
        for (int t = 0; t < M; ++t)
#pragma unroll
            for (int c = 0; c < U; ++c) cw[t][c] = nw[t][c];
    }
}

// dump the fused kernel's smem Psumbook in _psum_tables layout (m, segs, 2**b, n)
template <int V, int M, int U, int KB>
__global__ void __launch_bounds__(kThreads, 1)
    psumbook_dump_kernel(const GatherParams p, float* __restrict__ out, int64_t segs) {
    using S = FusedShape<V, M, U, KB>;
    extern __shared__ __align__(16) float smem[];
    float* psum = smem;
    float* books32 = smem + S::kPsumFloats;
    float* x32 = books32 + S::kBookFloats;
    const int tid = threadIdx.x;
    const int64_t slice = blockIdx.x;
    const int col = blockIdx.y;
    stage_books<V, M, U, KB>(books32, p.books, p.kcount, tid);
    stage_x<V, M, U, KB>(x32, p.x, slice, p.cols, p.n, col, tid);
    __syncthreads();
    build_psumbook_smem<V, M, U, KB>(psum, books32, x32, p.kcount, tid);
    __syncthreads();
    const int total = S::kSub * p.kcount * 32;
    for (int i = tid; i < total; i += kThreads) {
        const int lane = i & 31;
        const int c = (i >> 5) % p.kcount;
        const int j = (i >> 5) / p.kcount;
        const int t = j / U, uu = j % U;
        const int64_t seg = slice * 32 * U + lane * U + uu;
        if (seg >= segs) continue;
        const float v = psum[(j >> 1) * S::kRegionFloats + c * 64 + (j & 1) * 32 + lane];
        out[(((int64_t)t * segs + seg) * p.kcount + c) * p.n + col] = v;
    }
}

// deterministic split-K reduction: y[i] = sum_s ws[s][i], s ascending
__global__ void reduce_slices_kernel(const float* __restrict__ ws, float* __restrict__ y,
                                     int64_t count, int64_t n_slices) {
    pdl_wait();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if ((count & 3) == 0) {
        const int64_t c4 = count >> 2;
        const float4* w4 = reinterpret_cast<const float4*>(ws);
        float4* y4 = reinterpret_cast<float4*>(y);
        for (int64_t i = i0; i < c4; i += stride) {
            float4 s = w4[i];
            for (int64_t k = 1; k < n_slices; ++k) {
                const float4 v = w4[k * c4 + i];
                s.x += v.x;
                s.y += v.y;
                s.z += v.z;
                s.w += v.w;
            }
            y4[i] = s;
        }
    } else {
        for (int64_t i = i0; i < count; i += stride) {
            float s = ws[i];
            for (int64_t k = 1; k < n_slices; ++k) s += ws[k * count + i];
            y[i] = s;
        }
    }
    pdl_launch_dependents();
}

// ---------------------------------------------------------------------------
// strict mode: one thread per output element, the reference's exact order
// (engines.py:211-231 mirrored == engines.py:245-316 codegemm, bit for bit)
// ---------------------------------------------------------------------------
__global__ void strict_gemm_kernel(const uint8_t* __restrict__ packed,
                                   const uint16_t* __restrict__ raw16,
                                   const uint16_t* __restrict__ books,
                                   const uint16_t* __restrict__ scales,
                                   const uint16_t* __restrict__ x, float* __restrict__ y,
                                   int64_t rows, int64_t segs, int v, int m, int kcount,
                                   int64_t groups, int64_t g_eff, int n, int u, int64_t n_rg) {
    pdl_wait();
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= rows * n) return;
    const int64_t r = idx % rows;  // consecutive lanes = consecutive rows: x reads broadcast
    const int col = (int)(idx / rows);
    float acc = 0.0f;
    for (int64_t seg = 0; seg < segs; ++seg) {
        float seg_sum = 0.0f;
        for (int t = 0; t < m; ++t) {
            const uint32_t code = raw16 ? raw16[((int64_t)t * rows + r) * segs + seg]
                                        : packed[packed_index(t, r, seg, m, u, n_rg)];
            const uint16_t* c = books + ((int64_t)t * kcount + code) * v;
            const uint16_t* xs = x + seg * v * (int64_t)n + col;
            float psum = 0.0f;
            for (int k = 0; k < v; ++k) psum = fmaf(h2f(c[k]), h2f(xs[(int64_t)k * n]), psum);
            seg_sum = __fadd_rn(seg_sum, psum);
        }
        const float s = h2f(scales[r * groups + (seg * v) / g_eff]);
        acc = __fadd_rn(acc, __fmul_rn(s, seg_sum));
    }
    y[r * n + col] = acc;
}

// K1 standalone: out[t][seg][i][col], bit-exact _psum_tables
__global__ void psumbook_build_kernel(const uint16_t* __restrict__ books,
                                      const uint16_t* __restrict__ x, float* __restrict__ out,
                                      int m, int kcount, int v, int64_t segs, int n) {
    const int64_t total = (int64_t)m * segs * kcount * n;
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
         o += (int64_t)gridDim.x * blockDim.x) {
        const int col = (int)(o % n);
        const int64_t i = (o / n) % kcount;
        const int64_t seg = (o / ((int64_t)n * kcount)) % segs;
        const int64_t t = o / ((int64_t)n * kcount * segs);
        const uint16_t* c = books + (t * kcount + i) * v;
        float acc = 0.0f;
        for (int k = 0; k < v; ++k)
            acc = fmaf(h2f(c[k]), h2f(x[(seg * v + k) * (int64_t)n + col]), acc);
        out[o] = acc;
    }
}

int grid_for(int64_t total, int threads) {
    int64_t blocks = (total + threads - 1) / threads;
    if (blocks > 148 * 32) blocks = 148 * 32;
    return blocks < 1 ? 1 : (int)blocks;
}

// ---------------------------------------------------------------------------
// template dispatch
// ---------------------------------------------------------------------------
template <int V, int M, int U, int KB>
cudaError_t launch_fused_t(const GatherParams& gp, int64_t grid_x, bool pdl, cudaStream_t s) {
    using S = FusedShape<V, M, U, KB>;
    auto kern = fused_gemv_kernel<V, M, U, KB>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         S::kSmemBytes);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid_x, (unsigned)gp.n, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = S::kSmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, gp);
}

template <int V, int M, int U, int KB>
cudaError_t launch_dump_t(const GatherParams& gp, int64_t n_slices, float* out, int64_t segs,
                          cudaStream_t s) {
    using S = FusedShape<V, M, U, KB>;
    auto kern = psumbook_dump_kernel<V, M, U, KB>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         S::kSmemBytes);
    if (e != cudaSuccess) return e;
    kern<<<dim3((unsigned)n_slices, (unsigned)gp.n), kThreads, S::kSmemBytes, s>>>(gp, out, segs);
    return cudaGetLastError();
}

template <int V, int M, int U, int KB>
int occupancy_t() {
    using S = FusedShape<V, M, U, KB>;
    auto kern = fused_gemv_kernel<V, M, U, KB>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kSmemBytes) !=
        cudaSuccess)
        return 1;
    int n = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kThreads, S::kSmemBytes) !=
        cudaSuccess)
        return 1;
    return n < 1 ? 1 : n;
}

// Visit the instantiation for runtime (v, m, u, kb).  Instantiated set:
// v in {2,4,8,16}, (m,u) in {(1,1),(1,2),(1,4),(2,1),(2,2),(3,1),(4,1)}, kb in {4,8}.
template <typename F>
bool visit(int v, int m, int u, int kb, F&& f) {
#define CG_KB(V_, M_, U_)                         \
    if (kb == 4) return f.template run<V_, M_, U_, 4>(), true; \
    if (kb == 8) return f.template run<V_, M_, U_, 8>(), true; \
    return false;
#define CG_MU(V_)                                  \
    if (m == 1 && u == 1) { CG_KB(V_, 1, 1) }      \
    if (m == 1 && u == 2) { CG_KB(V_, 1, 2) }      \
    if (m == 1 && u == 4) { CG_KB(V_, 1, 4) }      \
    if (m == 2 && u == 1) { CG_KB(V_, 2, 1) }      \
    if (m == 2 && u == 2) { CG_KB(V_, 2, 2) }      \
    if (m == 3 && u == 1) { CG_KB(V_, 3, 1) }      \
    if (m == 4 && u == 1) { CG_KB(V_, 4, 1) }      \
    return false;
    switch (v) {
        case 2: { CG_MU(2) }
        case 4: { CG_MU(4) }
        case 8: { CG_MU(8) }
        case 16: { CG_MU(16) }
        default: return false;
    }
#undef CG_MU
#undef CG_KB
}

struct SmemQuery {
    int bytes = 0;
    template <int V, int M, int U, int KB>
    void run() { bytes = FusedShape<V, M, U, KB>::kSmemBytes; }
};
struct OccQuery {
    int n = 1;
    template <int V, int M, int U, int KB>
    void run() { n = occupancy_t<V, M, U, KB>(); }
};
struct FusedLaunch {
    const GatherParams* gp;
    int64_t grid_x;
    bool pdl;
    cudaStream_t s;
    cudaError_t err = cudaErrorInvalidConfiguration;
    template <int V, int M, int U, int KB>
    void run() { err = launch_fused_t<V, M, U, KB>(*gp, grid_x, pdl, s); }
};
struct DumpLaunch {
    const GatherParams* gp;
    int64_t n_slices;
    float* out;
    int64_t segs;
    cudaStream_t s;
    cudaError_t err = cudaErrorInvalidConfiguration;
    template <int V, int M, int U, int KB>
    void run() { err = launch_dump_t<V, M, U, KB>(*gp, n_slices, out, segs, s); }
};

}  // namespace

bool fused_instantiated(int v, int m, int u, int kbits) {
    SmemQuery q;
    return visit(v, m, u, kbits, q);
}

int fused_smem_bytes(int v, int m, int u, int kbits) {
    SmemQuery q;
    if (!visit(v, m, u, kbits, q)) return -1;
    return q.bytes;
}

int fused_max_ctas_per_sm(const Plan& p) {
    OccQuery q;
    if (!visit(p.v, p.m, p.u, p.kbits, q)) return 1;
    return q.n;
}

cudaError_t launch_prepack_codes(const Plan& p, const uint16_t* raw, uint8_t* packed,
                                 unsigned* bad, cudaStream_t s) {
    const int64_t total = p.code_bytes;
    prepack_codes_kernel<<<grid_for(total, 256), 256, 0, s>>>(
        raw, packed, total, p.rows, p.segs, p.m, p.u, p.n_rg, 1u << p.b, bad);
    return cudaGetLastError();
}

cudaError_t launch_prepack_scales(const Plan& p, const uint16_t* raw, uint16_t* packed,
                                  cudaStream_t s) {
    const int64_t total = p.scale_bytes / 2;
    prepack_scales_kernel<<<grid_for(total, 256), 256, 0, s>>>(
        raw, packed, total, p.rows, p.groups, p.n_rg, p.n_gs, p.slice_segs * p.v,
        p.g_row ? (int64_t)1 << 62 : p.g_eff, p.lg);
    return cudaGetLastError();
}

cudaError_t launch_check_codes(const Plan& p, const uint16_t* raw, unsigned* bad, cudaStream_t s) {
    const int64_t total = (int64_t)p.m * p.rows * p.segs;
    check_codes_kernel<<<grid_for(total, 256), 256, 0, s>>>(raw, total, 1u << p.b, bad);
    return cudaGetLastError();
}

cudaError_t launch_unpack_codes(const Plan& p, const uint8_t* packed, const uint16_t* raw16,
                                uint16_t* out, cudaStream_t s) {
    const int64_t total = (int64_t)p.m * p.rows * p.segs;
    unpack_codes_kernel<<<grid_for(total, 256), 256, 0, s>>>(packed, raw16, out, p.rows, p.segs,
                                                            p.m, p.u, p.n_rg);
    return cudaGetLastError();
}

cudaError_t launch_fused_gemv(const Plan& p, const GatherParams& gp, bool pdl, cudaStream_t s) {
    FusedLaunch f{&gp, p.n_slices * p.n_rb, pdl, s};
    if (!visit(p.v, p.m, p.u, p.kbits, f)) return cudaErrorInvalidConfiguration;
    return f.err;
}

cudaError_t launch_reduce_slices(const float* ws, float* y, int64_t count, int64_t n_slices,
                                 bool pdl, cudaStream_t s) {
    const int64_t work = (count & 3) == 0 ? count / 4 : count;
    int blocks = (int)((work + 255) / 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks, 1, 1);
    cfg.blockDim = dim3(256, 1, 1);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, reduce_slices_kernel, ws, y, count, n_slices);
}

cudaError_t launch_psumbook_dump(const Plan& p, const GatherParams& gp, float* out,
                                 cudaStream_t s) {
    DumpLaunch f{&gp, p.n_slices, out, p.segs, s};
    if (!visit(p.v, p.m, p.u, p.kbits, f)) return cudaErrorInvalidConfiguration;
    return f.err;
}

cudaError_t launch_strict_gemm(const Plan& p, const uint8_t* packed, const uint16_t* raw16,
                               const uint16_t* books, const uint16_t* scales, const uint16_t* x,
                               int n, float* y, cudaStream_t s) {
    const int64_t total = p.rows * n;
    const int threads = 128;
    const int64_t blocks = (total + threads - 1) / threads;
    strict_gemm_kernel<<<(unsigned)blocks, threads, 0, s>>>(
        packed, raw16, books, scales, x, y, p.rows, p.segs, p.v, p.m, p.kcount, p.groups,
        p.g_eff, n, p.u, p.n_rg);
    return cudaGetLastError();
}

cudaError_t launch_psumbook_build(const uint16_t* books, const uint16_t* x, int m, int b, int v,
                                  int64_t k_len, int n, float* out, cudaStream_t s) {
    const int kcount = 1 << b;
    const int64_t segs = k_len / v;
    const int64_t total = (int64_t)m * segs * kcount * n;
    psumbook_build_kernel<<<grid_for(total, 256), 256, 0, s>>>(books, x, out, m, kcount, v, segs,
                                                               n);
    return cudaGetLastError();
}

}  // namespace cg
