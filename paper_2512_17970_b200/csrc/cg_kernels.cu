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
#include <type_traits>

#include "cg_internal.h"

namespace cg {
namespace {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel, device and
// size (it costs microseconds of host time; a decode loop launches every step).
// `done` is the calling launcher's own static (one per kernel instantiation).
template <typename K>
cudaError_t set_smem_once(K kern, int smem, int (&done)[64]) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && done[dev] >= smem) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess && dev >= 0 && dev < 64 && smem > done[dev]) done[dev] = smem;
    return e;
}


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

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ uint32_t word_of(const uint4& q, int i) {
    return i == 0 ? q.x : (i == 1 ? q.y : (i == 2 ? q.z : q.w));
}

// ---------------------------------------------------------------------------
// code addressing in the prepacked stream (cg_internal.h)
//
// Lane l stores its 16 rows in XOR-permuted order: slot i holds row
// i ^ row_mask(l), row_mask(l) = bit-reverse of the low 4 lane bits.  With this
// order every halving step of the warp transpose-reduction keeps slots
// [0, CNT/2) and sends slots [CNT/2, CNT) -- the partner's sent slot i holds
// the same row as my kept slot i -- so the reduction needs no selects.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ int row_mask(int lane) {
    return ((lane & 1) << 3) | ((lane >> 1 & 1) << 2) | ((lane >> 2 & 1) << 1) | (lane >> 3 & 1);
}

// Byte mode (b > 4): one byte per code; the lane's 16*u bytes of a (slice, row
// group, codebook) tile are [slot][u] code indices idx = slot*u + uu, in u
// chunks of 16 bytes laid out lane-contiguous: byte idx&15 of chunk idx>>4.
// Nibble mode (b <= 4, 16-entry tables): two codes per byte, 8*u bytes per
// lane and tile.  Code idx sits in 32-bit word idx>>3 of the lane, byte idx&3,
// low nibble if (idx&4) == 0 else high nibble -- so masking a word with
// 0x0f0f0f0f (or shifting it right by 4 first) yields four codes as bytes and
// the gather's byte extraction is unchanged.  Words are laid out in 16-byte
// chunks lane-contiguous (u >= 2) or as 8 bytes per lane (u = 1).
// cbits: bits per code in the stream -- 4 (16-entry tables), 6 (64-entry
// tables, u = 4 only: four codes in three bytes, 48 bytes per lane), 8 (else)
__host__ __device__ __forceinline__ int64_t tile_bytes_of(int u, int cbits) {
    return cbits == 4 ? (int64_t)u * 256 : (cbits == 6 ? (int64_t)u * 384 : (int64_t)u * 512);
}
// byte offset of the lane's 32-bit word wi (nibble mode) inside a tile
__host__ __device__ __forceinline__ int64_t nib_word_off(int u, int lane, int wi) {
    return u >= 2 ? ((int64_t)(wi >> 2) * 32 + lane) * 16 + (wi & 3) * 4 : (int64_t)lane * 8 + wi * 4;
}

__device__ __forceinline__ uint32_t packed_code(const uint8_t* packed, int64_t t, int64_t r,
                                                int64_t seg, int m, int u, int64_t n_rg, int cbits) {
    const int64_t slice_segs = 32 * u;
    const int64_t slice = seg / slice_segs;
    const int64_t within = seg - slice * slice_segs;
    const int64_t lane = within / u;
    const int64_t uu = within - lane * u;
    const int64_t rg = r >> 4;
    const int64_t rr = r & 15;
    const int64_t slot = rr ^ row_mask((int)lane);
    const int64_t idx = slot * u + uu;  // position in the lane's [slot][u] codes
    const int64_t tile = ((slice * n_rg + rg) * m + t) * tile_bytes_of(u, cbits);
    if (cbits == 8) return packed[tile + (idx >> 4) * 512 + lane * 16 + (idx & 15)];
    if (cbits == 6) {  // bits [6 idx, 6 idx + 6) of the lane's byte stream (16-byte chunks)
        const int64_t bit = 6 * idx, p0 = bit >> 3, p1 = p0 + 1;
        const uint32_t b0 = packed[tile + (p0 >> 4) * 512 + lane * 16 + (p0 & 15)];
        const uint32_t b1 = p1 < 12 * u ? packed[tile + (p1 >> 4) * 512 + lane * 16 + (p1 & 15)] : 0u;
        return ((b0 | (b1 << 8)) >> (bit & 7)) & 63u;
    }
    const uint8_t byte = packed[tile + nib_word_off(u, (int)lane, (int)(idx >> 3)) + (idx & 3)];
    return (idx & 4) ? (byte >> 4) : (byte & 15u);
}

// ---------------------------------------------------------------------------
// K3: prepack / unpack / validation
// ---------------------------------------------------------------------------
__global__ void prepack_codes_kernel(const uint16_t* __restrict__ raw, uint8_t* __restrict__ out,
                                     int64_t total, int64_t rows, int64_t segs, int m, int u,
                                     int64_t n_rg, uint32_t code_limit,
                                     unsigned* __restrict__ bad, int cbits) {
    // one thread per output byte, decoding (slice, rg, t, lane, position)
    const int64_t tile_bytes = tile_bytes_of(u, cbits);
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
         o += (int64_t)gridDim.x * blockDim.x) {
        int64_t rest = o;
        const int64_t in_tile = rest % tile_bytes;
        rest /= tile_bytes;
        const int64_t t = rest % m;
        rest /= m;
        const int64_t rg = rest % n_rg;
        const int64_t slice = rest / n_rg;
        int64_t lane, idx[2];
        int ncodes;
        int sh[2] = {0, 4};
        if (cbits == 8) {
            const int64_t chunk = in_tile / 512;
            lane = (in_tile % 512) / 16;
            idx[0] = chunk * 16 + (in_tile % 16);
            ncodes = 1;
        } else if (cbits == 6) {
            // lane byte p holds bits [8p, 8p + 8) of the lane's 6-bit code stream
            const int64_t chunk = in_tile / 512;
            lane = (in_tile % 512) / 16;
            const int64_t pb = chunk * 16 + (in_tile % 16);
            idx[0] = (8 * pb) / 6;
            idx[1] = (8 * pb + 7) / 6;
            ncodes = idx[1] != idx[0] ? 2 : 1;
            sh[0] = (int)(6 * idx[0] - 8 * pb);  // may be negative: the code's low bits precede
            sh[1] = (int)(6 * idx[1] - 8 * pb);
        } else {
            int64_t wi, bw;
            if (u >= 2) {
                const int64_t chunk = in_tile / 512;
                lane = (in_tile % 512) / 16;
                wi = chunk * 4 + (in_tile % 16) / 4;
                bw = in_tile % 4;
            } else {
                lane = in_tile / 8;
                wi = (in_tile % 8) / 4;
                bw = in_tile % 4;
            }
            idx[0] = wi * 8 + bw;  // low nibble
            idx[1] = idx[0] + 4;   // high nibble
            ncodes = 2;
        }
        uint32_t val = 0;
        for (int k = 0; k < ncodes; ++k) {
            if (idx[k] >= 16 * u) continue;
            const int64_t slot = idx[k] / u, uu = idx[k] % u;
            const int64_t r = rg * 16 + (slot ^ row_mask((int)lane));
            const int64_t seg = slice * 32 * u + lane * u + uu;
            if (r < rows && seg < segs) {
                const uint16_t c = raw[(t * rows + r) * segs + seg];
                if (c >= code_limit) atomicOr(bad, 1u);
                val |= sh[k] >= 0 ? ((uint32_t)c << sh[k]) : ((uint32_t)c >> -sh[k]);
            }
        }
        out[o] = static_cast<uint8_t>(val);
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
                                    int64_t rows, int64_t segs, int m, int u, int64_t n_rg,
                                    int cbits) {
    const int64_t total = (int64_t)m * rows * segs;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (raw16) {
            out[i] = raw16[i];
        } else {
            const int64_t seg = i % segs;
            const int64_t r = (i / segs) % rows;
            const int64_t t = i / (segs * rows);
            out[i] = (uint16_t)packed_code(packed, t, r, seg, m, u, n_rg, cbits);
        }
    }
}

// CGMM code planes as stored (quantizer.py:471-497 pack_codes: code i in bits
// [i*b, (i+1)*b) of the plane, least-significant bit first, each plane padded
// to a whole byte) -> uint16 planes on the device (the loader never
// materialises uint16 planes on the host)
__global__ void unpack_packed_kernel(const uint8_t* __restrict__ packed, int64_t plane_bytes,
                                     int m, int64_t per_plane, int b,
                                     uint16_t* __restrict__ out) {
    const int64_t total = (int64_t)m * per_plane;
    const uint32_t mask = (1u << b) - 1u;
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
         o += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = o / per_plane, i = o - t * per_plane;
        const uint8_t* pl = packed + t * plane_bytes;
        const int64_t bit = i * b;
        const int64_t byte = bit >> 3;
        const int sh = (int)(bit & 7);
        uint32_t w = pl[byte];
        if (sh + b > 8) w |= (uint32_t)pl[byte + 1] << 8;
        if (sh + b > 16) w |= (uint32_t)pl[byte + 2] << 16;
        out[o] = (uint16_t)((w >> sh) & mask);
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
// Build: thread (q = lane&7, csub = lane>>3) of warp w writes the entries of
// lanes 4q..4q+3 (4 segments) for codes c0 + 64i, c0 = csub + 4w, with one
// STS.128 per code (the 8 threads of a phase cover one 128-byte code row:
// conflict-free).  The 4 dot products run as 2 FFMA2 chains over k:
//   centroid c_k       binary32 scalar, broadcast to both FFMA2 lanes
//   x pairs            (x_{seg0,k}, x_{seg1,k}), (x_{seg2,k}, x_{seg3,k})
// Each entry = ((+0 + c0*x0) + c1*x1) + ...: every lane of an FFMA2 is an
// IEEE fma with an exact product (binary16 x binary16 fits binary32), i.e.
// the reference's separate multiply and add (engines.py:126-133), bit for bit.
//
// The centroids of a thread's codes are read once per codebook straight from
// the raw binary16 codebook buffer (TMA-staged) and kept in registers across
// the U sub-tables; x is staged once per task as binary32 pairs in the layout
// the FFMA2 operands want (x_index), 16-byte skewed per lane quad so the 8
// threads of a phase read 8 distinct bank quads.  Shared-memory traffic of a
// build is then dominated by the table stores themselves.
// ---------------------------------------------------------------------------
template <int V, int M, int U, int KB>
struct FusedShape {
    static constexpr int kSub = M * U;
    static constexpr int kRegions = (kSub + 1) / 2;
    static constexpr int kCodes = 1 << KB;
    static constexpr int kRegionFloats = kCodes * 64;
    static constexpr int kPsumFloats = kRegions * kRegionFloats;
    static constexpr int kSliceSegs = 32 * U;
    // staged x: per (u, lane quad q) a block of 2V binary32 pairs + 16-B skew
    static constexpr int kXQF = 4 * V + 4;  // floats per block
    static constexpr int kXFloats = U * 8 * kXQF;
    static constexpr int kPsumBytes = 4 * kPsumFloats;
    static constexpr int kXBytes = 4 * kXFloats;
    // code stream: KB bits per code (16-entry tables: two codes per byte; 64-entry:
    // four codes in three bytes, u = 4 only; else one byte)
    static constexpr bool kNib = KB == 4;
    static_assert(KB != 6 || U == 4, "6-bit code streams are laid out for u = 4");
    static constexpr int kTileBytes = M * U * (KB == 4 ? 256 : (KB == 6 ? 384 : 512));
    static constexpr int kLaneBytes = (kNib && U == 1) ? 8 : 16;   // lane offset in a chunk
    static constexpr int kXPerThread = (V * kSliceSegs + kThreads - 1) / kThreads;
    static constexpr int kCPT = kCodes / (4 * kWarps) > 0 ? kCodes / (4 * kWarps) : 1;
    static constexpr bool kFullCodes = kCPT * 4 * kWarps == kCodes;
    // centroids of all of a thread's codes held in registers across u
    #ifdef CG_NOHOIST
    static constexpr bool kHoist = false;
#else
    static constexpr bool kHoist = kCPT * V <= 16;
#endif
    // register pipeline depth of the code-tile stream (tiles of 16*M*U bytes per lane)
    #ifdef CG_DEPTH
    static constexpr int kDepth = CG_DEPTH;
#else
    static constexpr int kDepth = M * U < 4 ? 3 : 2;
#endif
};

// float index (in the staged x buffer) of element k of slice segment s: the
// pair (x_{s0,k}, x_{s1,k}) of lanes 4q+2h, 4q+2h+1 at the same u is one
// 8-byte FFMA2 operand, element lo; binary32 so the build converts nothing.
template <int V, int M, int U, int KB>
__device__ __forceinline__ int x_index(int s, int k) {
    using S = FusedShape<V, M, U, KB>;
    const int l = s / U, u = s - (s / U) * U;
    const int q = l >> 2, i = l & 3, h = i >> 1, lo = i & 1;
    return (u * 8 + q) * S::kXQF + ((h * V + k) << 1) + lo;
}

// Load this thread's share of the slice of x (column `col`), binary16.
template <int V, int M, int U, int KB>
__device__ __forceinline__ void load_x(uint16_t (&r)[FusedShape<V, M, U, KB>::kXPerThread],
                                       const uint16_t* x, int64_t slice, int64_t cols, int n,
                                       int col, int tid) {
    using S = FusedShape<V, M, U, KB>;
    const int64_t e0 = slice * (int64_t)(S::kSliceSegs * V);
#pragma unroll
    for (int i = 0; i < S::kXPerThread; ++i) {
        const int l = tid + i * kThreads;
        const int64_t e = e0 + l;
        r[i] = (l < S::kSliceSegs * V && e < cols) ? x[e * n + col] : (uint16_t)0;
    }
}

// A layer's x given as binary32 (an earlier stage's y, written in this
// launch: read through L2) is rounded to binary16 (RNE) as it is staged.
template <int V, int M, int U, int KB>
__device__ __forceinline__ void load_x(uint16_t (&r)[FusedShape<V, M, U, KB>::kXPerThread],
                                       const LayerTask& L, int64_t slice, int n, int col, int tid) {
    using S = FusedShape<V, M, U, KB>;
    if (L.x32 == nullptr) return load_x<V, M, U, KB>(r, L.x, slice, L.cols, n, col, tid);
    const int64_t e0 = slice * (int64_t)(S::kSliceSegs * V);
#pragma unroll
    for (int i = 0; i < S::kXPerThread; ++i) {
        const int l = tid + i * kThreads;
        const int64_t e = e0 + l;
        r[i] = (l < S::kSliceSegs * V && e < L.cols)
                   ? __half_as_ushort(__float2half_rn(__ldcg(L.x32 + e * n + col)))
                   : (uint16_t)0;
    }
}

// x of an LL consumer: element e lives at xc_ll + 2 * (byte offset of x32 + e in
// the gathered buffers) as (value, epoch); spin until this launch's epoch shows
// (an 8-byte store is single-copy atomic: value and epoch arrive together)
__device__ __forceinline__ float ll_load(const float* x32, const GroupParams& p, unsigned epoch) {
    const int64_t off = reinterpret_cast<const unsigned char*>(x32) - p.xc_gbase;
    const float2* a = reinterpret_cast<const float2*>(p.xc_ll + 2 * off);
    unsigned long long t0 = 0;
    while (true) {
        uint32_t v, ep;
        asm volatile("ld.volatile.global.v2.u32 {%0,%1}, [%2];" : "=r"(v), "=r"(ep) : "l"(a) : "memory");
        if (ep == epoch) return __uint_as_float(v);
        if (p.xc_timeout_ns) {
            const unsigned long long t = gtimer();
            if (t0 == 0) t0 = t;
            else if (t - t0 > p.xc_timeout_ns) __trap();  // a peer never pushed
        }
    }
}

template <int V, int M, int U, int KB>
__device__ __forceinline__ void load_x_ll(uint16_t (&r)[FusedShape<V, M, U, KB>::kXPerThread],
                                          const LayerTask& L, const GroupParams& p, unsigned epoch,
                                          int64_t slice, int n, int col, int tid) {
    using S = FusedShape<V, M, U, KB>;
    const int64_t e0 = slice * (int64_t)(S::kSliceSegs * V);
#pragma unroll
    for (int i = 0; i < S::kXPerThread; ++i) {
        const int l = tid + i * kThreads;
        const int64_t e = e0 + l;
        r[i] = (l < S::kSliceSegs * V && e < L.cols)
                   ? __half_as_ushort(__float2half_rn(ll_load(L.x32 + e * n + col, p, epoch)))
                   : (uint16_t)0;
    }
}

// x of an LL-chain consumer: element e = sum over the producer's slices (in slice
// order: deterministic) of its partial row e, each an (value, epoch) pair spun on
// until this launch's epoch shows; the writer consumer also stores the reduced y
// (kLLGroup partials in flight per round: a 28-slice producer takes 2 rounds, not 4 --
// 8B block 38.32 -> 37.79 us, 70B 93.5 -> 91.3 us on one box; `grp` = 8 restores the
// old rounds for A/B)
constexpr int kLLGroup = 16;  // (32: 456 bytes of spills, 8B block 50 us)
__device__ __forceinline__ float llc_sum(const float2* llp, int64_t rows, int ns, int64_t e,
                                         unsigned epoch, int grp) {
    float acc = 0.0f;
    for (int s0 = 0; s0 < ns; s0 += grp) {
        uint32_t v[kLLGroup], ep[kLLGroup];
        const int k = min(grp, ns - s0);
        const float2* a = llp + (int64_t)s0 * rows + e;
#pragma unroll
        for (int j = 0; j < kLLGroup; ++j) {  // up to kLLGroup partials in flight
            ep[j] = epoch;
            if (j < k)
                asm volatile("ld.volatile.global.v2.u32 {%0,%1}, [%2];"
                             : "=r"(v[j]), "=r"(ep[j]) : "l"(a + j * rows));
        }
        // poll in rounds: every partial still stale is re-read in the same round
        // (one round trip per round, not one per partial)
        unsigned long long t0 = 0;
        while (true) {
            bool ready = true;
#pragma unroll
            for (int j = 0; j < kLLGroup; ++j) ready &= ep[j] == epoch;
            if (ready) break;
#pragma unroll
            for (int j = 0; j < kLLGroup; ++j)
                if (ep[j] != epoch)
                    asm volatile("ld.volatile.global.v2.u32 {%0,%1}, [%2];"
                                 : "=r"(v[j]), "=r"(ep[j]) : "l"(a + j * rows));
            const unsigned long long t = gtimer();
            if (t0 == 0) t0 = t;
            else if (t - t0 > 2000000000ull) __trap();  // a producer never wrote (2 s)
            __nanosleep(64);  // (fewer polls in flight: less L2 queueing; 8B block -0.2 us)
        }
#pragma unroll
        for (int j = 0; j < kLLGroup; ++j)
            if (j < k) acc += __uint_as_float(v[j]);
    }
    return acc;
}

template <int V, int M, int U, int KB>
__device__ __forceinline__ void load_x_llc(uint16_t (&r)[FusedShape<V, M, U, KB>::kXPerThread],
                                           const LayerTask& L, const LayerTask& P, unsigned epoch,
                                           bool write_y, int64_t slice, int tid, int grp) {
    using S = FusedShape<V, M, U, KB>;
    const int64_t e0 = slice * (int64_t)(S::kSliceSegs * V);
#pragma unroll
    for (int i = 0; i < S::kXPerThread; ++i) {
        const int l = tid + i * kThreads;
        const int64_t e = e0 + l;
        uint16_t h = 0;
        if (l < S::kSliceSegs * V && e < L.cols) {
            const float y = llc_sum(P.llp, P.rows, (int)P.n_slices, e, epoch, grp);
            if (write_y) P.y[e] = y;
            h = __half_as_ushort(__float2half_rn(y));
        }
        r[i] = h;
    }
}

template <int V, int M, int U, int KB>
__device__ __forceinline__ void store_x(float* xs,
                                        const uint16_t (&r)[FusedShape<V, M, U, KB>::kXPerThread],
                                        int tid) {
    using S = FusedShape<V, M, U, KB>;
#pragma unroll
    for (int i = 0; i < S::kXPerThread; ++i) {
        const int l = tid + i * kThreads;
        if (l < S::kSliceSegs * V) xs[x_index<V, M, U, KB>(l / V, l % V)] = h2f(r[i]);
    }
}

// raw binary16 x slice (TMA-staged, `valid` elements) -> staged pairs, zero past the end
template <int V, int M, int U, int KB>
__device__ __forceinline__ void stage_x_raw(float* xs, const uint16_t* xr, int valid, int tid) {
    using S = FusedShape<V, M, U, KB>;
    for (int e = tid; e < S::kSliceSegs * V; e += kThreads)
        xs[x_index<V, M, U, KB>(e / V, e % V)] = e < valid ? h2f(xr[e]) : 0.0f;
}
// the same from a binary32 slice (an earlier stage's y), rounded to binary16 as read
template <int V, int M, int U, int KB>
__device__ __forceinline__ void stage_x_raw32(float* xs, const float* xr, int valid, int tid) {
    using S = FusedShape<V, M, U, KB>;
    for (int e = tid; e < S::kSliceSegs * V; e += kThreads)
        xs[x_index<V, M, U, KB>(e / V, e % V)] =
            e < valid ? __half2float(__float2half_rn(xr[e])) : 0.0f;
}

// V binary16 centroid components -> binary32
template <int V>
__device__ __forceinline__ void load_centroid(float (&c)[V], const uint16_t* p) {
    uint32_t w[V / 2 > 0 ? V / 2 : 1];
    if constexpr (V == 2) {
        w[0] = *reinterpret_cast<const uint32_t*>(p);
    } else if constexpr (V == 4) {
        const uint2 a = *reinterpret_cast<const uint2*>(p);
        w[0] = a.x;
        w[1] = a.y;
    } else {
#pragma unroll
        for (int i = 0; i < V / 8; ++i) {
            const uint4 a = reinterpret_cast<const uint4*>(p)[i];
            w[4 * i] = a.x;
            w[4 * i + 1] = a.y;
            w[4 * i + 2] = a.z;
            w[4 * i + 3] = a.w;
        }
    }
#pragma unroll
    for (int i = 0; i < V / 2; ++i) {
        const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
        c[2 * i] = f.x;
        c[2 * i + 1] = f.y;
    }
}

// One sub-table (codebook t, segment-in-lane uu) of the build below.
template <int V, int M, int U, int KB, bool FULL>
__device__ __forceinline__ void build_subtable(float* psum, const uint16_t* bk, const float* xs,
                                               int kcount, int t, int uu, int q, int c0,
                                               const float (&cc)[FusedShape<V, M, U, KB>::kHoist
                                                                      ? FusedShape<V, M, U, KB>::kCPT
                                                                      : 1][V]) {
    using S = FusedShape<V, M, U, KB>;
    constexpr int kCPT = S::kCPT;
    const int j = t * U + uu;
    // x of this thread's 4 segments, paired for FFMA2:
    // x01[k] = (x_s0k, x_s1k), x23[k] = (x_s2k, x_s3k)
    float2 x01[V], x23[V];
    {
        const float4* src = reinterpret_cast<const float4*>(xs + (uu * 8 + q) * S::kXQF);
#pragma unroll
        for (int c = 0; c < V; ++c) {  // 2V pairs = V float4
            const float4 w = src[c];
            float2* d = (2 * c < V) ? &x01[2 * c] : &x23[2 * c - V];
            d[0] = make_float2(w.x, w.y);
            d[1] = make_float2(w.z, w.w);
        }
    }
    float* dst = psum + (j >> 1) * S::kRegionFloats + (j & 1) * 32 + q * 4;
    if constexpr (S::kHoist) {
        float2 a01[kCPT], a23[kCPT];
#pragma unroll
        for (int k = 0; k < V; ++k)
#pragma unroll
            for (int i = 0; i < kCPT; ++i) {
                const float2 cb = make_float2(cc[i][k], cc[i][k]);
                a01[i] = k == 0 ? __ffma2_rn(cb, x01[0], make_float2(0.0f, 0.0f))
                                : __ffma2_rn(cb, x01[k], a01[i]);
                a23[i] = k == 0 ? __ffma2_rn(cb, x23[0], make_float2(0.0f, 0.0f))
                                : __ffma2_rn(cb, x23[k], a23[i]);
            }
#pragma unroll
        for (int i = 0; i < kCPT; ++i) {
            const int c = c0 + 4 * kWarps * i;
            if (FULL || c < kcount)
                *reinterpret_cast<float4*>(dst + c * 64) =
                    make_float4(a01[i].x, a01[i].y, a23[i].x, a23[i].y);
        }
    } else {
#pragma unroll 1
        for (int c = c0; c < kcount; c += 4 * kWarps) {
            float ci[V];
            load_centroid<V>(ci, bk + c * V);
            float2 a01 = make_float2(0.0f, 0.0f), a23 = make_float2(0.0f, 0.0f);
#pragma unroll
            for (int k = 0; k < V; ++k) {
                a01 = __ffma2_rn(make_float2(ci[k], ci[k]), x01[k], a01);
                a23 = __ffma2_rn(make_float2(ci[k], ci[k]), x23[k], a23);
            }
            *reinterpret_cast<float4*>(dst + c * 64) = make_float4(a01.x, a01.y, a23.x, a23.y);
        }
    }
}

// books16: raw binary16 codebooks [t][kcount][V];  xs: staged x pairs.
// FULL (kcount == 2**KB, every b = 8 / b = 4 table): no per-code bounds test,
// so the kCPT codes' 2*kCPT FFMA2 chains of a sub-table are interleaved
// k-outer (independent chains back to back; a per-code branch would serialise
// them and expose the FFMA2 latency).  Each entry is still the chain
// ((+0 + c0*x0) + c1*x1) + ... of exact products: bit-exact.
template <int V, int M, int U, int KB, bool FULL>
__device__ __forceinline__ void build_psumbook_impl(float* psum, const uint16_t* books16,
                                                    const float* xs, int kcount, int tid) {
    using S = FusedShape<V, M, U, KB>;
    const int lane = tid & 31, warp = tid >> 5;
    const int q = lane & 7;      // this thread writes lanes 4q..4q+3 of a code row
    const int csub = lane >> 3;  // 4 codes per warp per pass
    const int c0 = csub + 4 * warp;
    constexpr int kCPT = S::kCPT;
#pragma unroll 1
    for (int t = 0; t < M; ++t) {
        const uint16_t* bk = books16 + t * kcount * V;
        float cc[S::kHoist ? kCPT : 1][V];
        if constexpr (S::kHoist) {
#pragma unroll
            for (int i = 0; i < kCPT; ++i) {
                const int c = c0 + 4 * kWarps * i;
                if (FULL || c < kcount) load_centroid<V>(cc[i], bk + c * V);
                else {
#pragma unroll
                    for (int k = 0; k < V; ++k) cc[i][k] = 0.0f;
                }
            }
        }
        // (FULL: the sub-table loop unrolled, so the table stores of one sub-table
        // overlap the FFMA2 chains of the next instead of alternating with them)
#pragma unroll
        for (int uu = 0; uu < (FULL ? U : 1); ++uu) {
            build_subtable<V, M, U, KB, FULL>(psum, bk, xs, kcount, t, uu, q, c0, cc);
        }
#pragma unroll 1
        for (int uu = FULL ? U : 0; uu < U; ++uu) {
            build_subtable<V, M, U, KB, FULL>(psum, bk, xs, kcount, t, uu, q, c0, cc);
        }
    }
}
#if 0
        {
            {
                const int j = t * U;
                const int uu = 0;
            float2 x01[V], x23[V];
            {
                const float4* src = reinterpret_cast<const float4*>(xs + (uu * 8 + q) * S::kXQF);
#pragma unroll
                for (int c = 0; c < V; ++c) {  // 2V pairs = V float4
                    const float4 w = src[c];
                    float2* d = (2 * c < V) ? &x01[2 * c] : &x23[2 * c - V];
                    d[0] = make_float2(w.x, w.y);
                    d[1] = make_float2(w.z, w.w);
                }
            }
            float* dst = psum + (j >> 1) * S::kRegionFloats + (j & 1) * 32 + q * 4;
            if constexpr (S::kHoist) {
                float2 a01[kCPT], a23[kCPT];
#pragma unroll
                for (int k = 0; k < V; ++k)
#pragma unroll
                    for (int i = 0; i < kCPT; ++i) {
                        const float2 cb = make_float2(cc[i][k], cc[i][k]);
                        a01[i] = k == 0 ? __ffma2_rn(cb, x01[0], make_float2(0.0f, 0.0f))
                                        : __ffma2_rn(cb, x01[k], a01[i]);
                        a23[i] = k == 0 ? __ffma2_rn(cb, x23[0], make_float2(0.0f, 0.0f))
                                        : __ffma2_rn(cb, x23[k], a23[i]);
                    }
#pragma unroll
                for (int i = 0; i < kCPT; ++i) {
                    const int c = c0 + 4 * kWarps * i;
                    if (FULL || c < kcount)
                        *reinterpret_cast<float4*>(dst + c * 64) =
                            make_float4(a01[i].x, a01[i].y, a23[i].x, a23[i].y);
                }
            } else {
#pragma unroll 1
                for (int c = c0; c < kcount; c += 4 * kWarps) {
                    float ci[V];
                    load_centroid<V>(ci, bk + c * V);
                    float2 a01 = make_float2(0.0f, 0.0f), a23 = make_float2(0.0f, 0.0f);
#pragma unroll
                    for (int k = 0; k < V; ++k) {
                        a01 = __ffma2_rn(make_float2(ci[k], ci[k]), x01[k], a01);
                        a23 = __ffma2_rn(make_float2(ci[k], ci[k]), x23[k], a23);
                    }
                    *reinterpret_cast<float4*>(dst + c * 64) = make_float4(a01.x, a01.y, a23.x, a23.y);
                }
            }
        }
    }
}
#endif

#ifdef CG_BUILD_R01
template <int V>
__device__ __forceinline__ void psum_entries(float* dst, const float (&cc)[V],
                                             const float2 (&x01)[V], const float2 (&x23)[V]) {
    float2 a01 = make_float2(0.0f, 0.0f), a23 = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int k = 0; k < V; ++k) {
        a01 = __ffma2_rn(make_float2(cc[k], cc[k]), x01[k], a01);
        a23 = __ffma2_rn(make_float2(cc[k], cc[k]), x23[k], a23);
    }
    *reinterpret_cast<float4*>(dst) = make_float4(a01.x, a01.y, a23.x, a23.y);
}

// (CG_BUILD_R01: the round-1 build, per-code bounds tests, for A/B timing)
template <int V, int M, int U, int KB>
__device__ __forceinline__ void build_psumbook_r01(float* psum, const uint16_t* books16,
                                                    const float* xs, int kcount, int tid) {
    using S = FusedShape<V, M, U, KB>;
    const int lane = tid & 31, warp = tid >> 5;
    const int q = lane & 7;      // this thread writes lanes 4q..4q+3 of a code row
    const int csub = lane >> 3;  // 4 codes per warp per pass
    const int c0 = csub + 4 * warp;
    constexpr int kCPT = S::kCPT;
    const bool full = S::kFullCodes && kcount == S::kCodes;
#pragma unroll 1
    for (int t = 0; t < M; ++t) {
        const uint16_t* bk = books16 + t * kcount * V;
        float cc[S::kHoist ? kCPT : 1][V];
        if constexpr (S::kHoist) {
#pragma unroll
            for (int i = 0; i < kCPT; ++i) {
                const int c = c0 + 4 * kWarps * i;
                if (full || c < kcount) load_centroid<V>(cc[i], bk + c * V);
            }
        }
#pragma unroll 1
        for (int uu = 0; uu < U; ++uu) {
            const int j = t * U + uu;
            // x of this thread's 4 segments, paired for FFMA2:
            // x01[k] = (x_s0k, x_s1k), x23[k] = (x_s2k, x_s3k)
            float2 x01[V], x23[V];
            {
                const float4* src = reinterpret_cast<const float4*>(xs + (uu * 8 + q) * S::kXQF);
#pragma unroll
                for (int c = 0; c < V; ++c) {  // 2V pairs = V float4
                    const float4 w = src[c];
                    float2* d = (2 * c < V) ? &x01[2 * c] : &x23[2 * c - V];
                    d[0] = make_float2(w.x, w.y);
                    d[1] = make_float2(w.z, w.w);
                }
            }
            float* dst = psum + (j >> 1) * S::kRegionFloats + (j & 1) * 32 + q * 4;
            if constexpr (S::kHoist) {
#pragma unroll
                for (int i = 0; i < kCPT; ++i) {
                    const int c = c0 + 4 * kWarps * i;
                    if (full || c < kcount) psum_entries<V>(dst + c * 64, cc[i], x01, x23);
                }
            } else {
#pragma unroll 1
                for (int c = c0; c < kcount; c += 4 * kWarps) {
                    float ci[V];
                    load_centroid<V>(ci, bk + c * V);
                    psum_entries<V>(dst + c * 64, ci, x01, x23);
                }
            }
        }
    }
}

#endif

template <int V, int M, int U, int KB>
__device__ __forceinline__ void build_psumbook_smem(float* psum, const uint16_t* books16,
                                                    const float* xs, int kcount, int tid) {
    using S = FusedShape<V, M, U, KB>;
#ifdef CG_BUILD_R01
    return build_psumbook_r01<V, M, U, KB>(psum, books16, xs, kcount, tid);
#endif
    if (S::kFullCodes && kcount == S::kCodes)
        build_psumbook_impl<V, M, U, KB, true>(psum, books16, xs, kcount, tid);
    else
        build_psumbook_impl<V, M, U, KB, false>(psum, books16, xs, kcount, tid);
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
// butterfly shuffle as inline PTX (every lane of the warp participates: the
// gather loop is warp-uniform), so ptxas sees a plain SHFL rather than the
// intrinsic's divergence-checked form
__device__ __forceinline__ float shfl_bfly(float v, int mk) {
#ifdef CG_SHFL_INTRINSIC
    return __shfl_xor_sync(0xffffffffu, v, mk);
#else
    float r;
    asm("shfl.sync.bfly.b32 %0, %1, %2, 0x1f, 0xffffffff;" : "=f"(r) : "f"(v), "r"(mk));
    return r;
#endif
}

// halving step on slot-permuted partials: keep slots [0, CNT/2), add the
// partner's slots [CNT/2, CNT) (same rows, see row_mask)
template <int CNT>
__device__ __forceinline__ void halve(float (&a)[16], int mk) {
#pragma unroll
    for (int i = 0; i < CNT / 2; i += 2) {
        if constexpr (CNT >= 4) {
            const float2 mine = make_float2(a[i], a[i + 1]);
            const float2 other = make_float2(shfl_bfly(a[i + CNT / 2], mk),
                                             shfl_bfly(a[i + 1 + CNT / 2], mk));
            const float2 sum = __fadd2_rn(mine, other);
            a[i] = sum.x;
            a[i + 1] = sum.y;
        } else {
            a[i] += shfl_bfly(a[i + CNT / 2], mk);
        }
    }
}

// Multiply slots [0, CNT) by their rows' scales.  Slot i holds row
// base + (i ^ m) with m = row_mask & (CNT-1); the smem tile p[0..CNT) is in row
// order, so the binary16 words are permuted by m before use.
template <int CNT>
__device__ __forceinline__ void apply_scales(float (&a)[16], const uint16_t* p, int m) {
    if constexpr (CNT == 1) {
        a[0] *= h2f(*p);
    } else {
        uint32_t w[CNT / 2];
#pragma unroll
        for (int i = 0; i < CNT / 2; ++i) w[i] = reinterpret_cast<const uint32_t*>(p)[i];
        // word-level swaps for mask bits >= 1 (blocks of 2^(b-1) words)
#pragma unroll
        for (int b = CNT / 4; b >= 1; b >>= 1) {
            if (m & (2 * b)) {
#pragma unroll
                for (int i = 0; i < CNT / 2; ++i)
                    if ((i & b) == 0) {
                        const uint32_t tmp = w[i];
                        w[i] = w[i + b];
                        w[i + b] = tmp;
                    }
            }
        }
        const uint32_t sel = (m & 1) ? 0x1032u : 0x3210u;  // swap the halves within a word
#pragma unroll
        for (int i = 0; i < CNT / 2; ++i) {
            const uint32_t ww = __byte_perm(w[i], 0u, sel);
            const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&ww));
            const float2 r = __fmul2_rn(make_float2(a[2 * i], a[2 * i + 1]), f);
            a[2 * i] = r.x;
            a[2 * i + 1] = r.y;
        }
    }
}

// ---- mbarrier + bulk async copy (TMA 1-D) for the task's scale tiles ----
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// split-K partials of a task: smem -> global y, added in L2 by the bulk engine
__device__ __forceinline__ void bulk_reduce_add_f32(float* dst, const float* src, uint32_t bytes) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile(
        "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst),
        "r"(smem_u32(src)), "r"(bytes)
        : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// all but the most recent bulk group have finished reading shared memory
__device__ __forceinline__ void bulk_wait_read_prev() {
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// fine-grained diagnostics of one task switch (CG_FINE_STAMPS builds only)
#ifdef CG_FINE_STAMPS
#define CG_FST(k) \
    if (p.stamps && tid == 0 && task_idx == 1) p.stamps[blockIdx.x * 128 + 112 + (k)] = gtimer();
#else
#define CG_FST(k)
#endif

// ---------------------------------------------------------------------------
// K2: fused Psumbook build + code-gather accumulate (persistent, task-driven)
//
// A launch runs a group of independent layers; CTA c executes tasks c,
// c+grid, ... of each layer in order (a task = one K-slice x one block of row
// groups).  Per task: the codebooks, the x slice and the first code tiles are
// put in flight, the task's scale tiles arrive by bulk async copy (TMA 1-D,
// mbarrier), the slice Psumbook is built in shared memory, and each warp walks
// its row groups with a two-deep register pipeline.
//
// Split-K without barriers: a row group's partial goes to the workspace and
// the writing warp takes a ticket on a monotonic per-row-group counter; the
// slice that arrives last for a row group sums that row group over all
// slices (fixed order -- deterministic).  The ticket is read one row group
// later (its round trip overlaps the next lookups) and the sums run at the
// start of the CTA's next task, overlapping that task's input loads.
// ---------------------------------------------------------------------------
template <int V, int M, int U, int KB>
__device__ __forceinline__ void load_tile(uint4 (&cw)[M][U], const uint8_t* tp) {
    using S = FusedShape<V, M, U, KB>;
    if constexpr (KB == 6) {  // 3 chunks of 16 bytes per lane and codebook: 64 codes x 6 bits
#pragma unroll
        for (int t = 0; t < M; ++t)
#pragma unroll
            for (int c = 0; c < 3; ++c) cw[t][c] = ldg_stream_v4(tp + (t * 3 + c) * 512);
    } else if constexpr (!S::kNib) {
#pragma unroll
        for (int t = 0; t < M; ++t)
#pragma unroll
            for (int c = 0; c < U; ++c) cw[t][c] = ldg_stream_v4(tp + (t * U + c) * 512);
    } else if constexpr (U == 1) {  // 8 bytes per lane and codebook
#pragma unroll
        for (int t = 0; t < M; ++t) {
            uint2 v;
            asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                         : "=r"(v.x), "=r"(v.y)
                         : "l"(tp + t * 256));
            cw[t][0] = make_uint4(v.x, v.y, 0u, 0u);
        }
    } else {  // U/2 chunks of 16 bytes per lane and codebook
#pragma unroll
        for (int t = 0; t < M; ++t)
#pragma unroll
            for (int c = 0; c < U / 2; ++c) cw[t][c] = ldg_stream_v4(tp + (t * (U / 2) + c) * 512);
    }
}

// the 32-bit word whose byte (idx & 3) is code idx: byte mode, nibble mode, or
// the 6-bit stream (u = 4: codes 4q..4q+3 = bits [24q, 24q + 24) of the lane's
// words, spread into bytes with three shifts)
template <int KB, int U>
__device__ __forceinline__ uint32_t code_word(const uint4 (&cw)[U], int idx) {
    if constexpr (KB == 8) {
        return word_of(cw[idx >> 4], (idx >> 2) & 3);
    } else if constexpr (KB == 4) {
        const uint32_t w = word_of(cw[(idx >> 3) >> 2], (idx >> 3) & 3);
        return (idx & 4) ? ((w >> 4) & 0x0f0f0f0fu) : (w & 0x0f0f0f0fu);
    } else {
        const int bit = 24 * (idx >> 2);
        const int k = bit >> 5, sh = bit & 31;
        const uint32_t lo = word_of(cw[k >> 2], k & 3);
        const uint32_t hi = (k + 1 < 12) ? word_of(cw[(k + 1) >> 2], (k + 1) & 3) : 0u;
        const uint32_t x = __funnelshift_r(lo, hi, sh);
        return (x & 0x3fu) | ((x << 2) & 0x3f00u) | ((x << 4) & 0x3f0000u) | ((x << 6) & 0x3f000000u);
    }
}

// lb0/lb1 = per-lane PRMT constants: byte0 = lane<<2 | half<<7, bytes 1-2 =
// bits 16-31 of the Psumbook's 64 KB-aligned shared address.  One PRMT then
// yields  base | code<<8 | half<<7 | lane<<2  and the region offset rides in
// the LDS immediate: one PRMT + one LDS per lookup, no address arithmetic.
template <int V, int M, int U, int KB>
__device__ __forceinline__ float gather_row_group(const uint4 (&cw)[M][U], const uint16_t* sp,
                                                  uint32_t lb0, uint32_t lb1, int mask,
                                                  bool early) {
    using S = FusedShape<V, M, U, KB>;
    // lookups: a[i] = sum over (t, u) of psum_t[seg(lane,u)][code of slot i],
    // two slots at a time with packed FADD2
    float a[16];
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
        float2 s2 = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int t = 0; t < M; ++t)
#pragma unroll
            for (int uu = 0; uu < U; ++uu) {
                const int j = t * U + uu;
                const uint32_t lb = (j & 1) ? lb1 : lb0;
                const uint32_t region = (uint32_t)((j >> 1) * S::kRegionFloats * 4);
                float2 v;
                {
                    const int idx = i * U + uu;
                    const uint32_t w = code_word<KB, U>(cw[t], idx);
                    v.x = lds_f32(__byte_perm(w, lb, 0x6504u | ((uint32_t)(idx & 3) << 4)) + region);
                }
                {
                    const int idx = (i + 1) * U + uu;
                    const uint32_t w = code_word<KB, U>(cw[t], idx);
                    v.y = lds_f32(__byte_perm(w, lb, 0x6504u | ((uint32_t)(idx & 3) << 4)) + region);
                }
                s2 = (t == 0 && uu == 0) ? v : __fadd2_rn(s2, v);
            }
        a[i] = s2.x;
        a[i + 1] = s2.y;
    }
    // Transpose-reduce the 16 slot partials across lanes; lanes 0-15 keep their
    // rows' sums.  When a scale group spans >= 8 lanes (lg >= 3; every g = 128
    // configuration), after the first three halvings (lanes
    // differing in bits 0-2 summed) all lanes still to be combined share each
    // row's scale: the scales are applied there, to the two remaining slots.
    // Smaller groups (g = v, 2v, 32 ... : 1, 2 or 4 lanes per group, `early`)
    // scale all 16 slots of the lane before the first halving -- the
    // reference's per-segment scale (engines.py:294) applied per lane.
    // `sp` is the lane's group tile (16 rows, row order).
    if (early) apply_scales<16>(a, sp, mask);
    halve<16>(a, 1);
    halve<8>(a, 2);
    halve<4>(a, 4);
    if (!early) apply_scales<2>(a, sp + (mask & ~1), mask & 1);
    halve<2>(a, 8);
    a[0] += shfl_bfly(a[0], 16);
    return a[0];
}

// y[row][col] = sum over slices of the partials, slices ascending: the fixed
// order that makes the split-K result independent of scheduling and tiling.
__device__ __forceinline__ float sum_slices(const LayerTask& L, int n, int64_t row, int col) {
    const int ns = (int)L.n_slices;
    const int64_t plane = L.rows * n;
    const float* src = L.ws + row * n + col;
    float acc = __ldcg(src);
#pragma unroll 4
    for (int s = 1; s < ns; ++s) acc += __ldcg(src + (int64_t)s * plane);
    return acc;
}

// whole row group (16 rows) by lanes 0-15 of a warp
__device__ __forceinline__ void fixup_row_group(const LayerTask& L, int n, int64_t rg, int col,
                                             int lane) {
    const int64_t row = rg * 16 + lane;
    if (lane < 16 && row < L.rows) L.y[row * n + col] = sum_slices(L, n, row, col);
}

struct FixupEntry {
    int layer, col;
    long long rg;
};

// CTA-uniform state kept in shared memory (off_bar), not registers: the
// mbarrier, the fix-up count, the previous task (closed at the start of the
// next task, after that task's input loads are in flight, or at kernel end)
// and the zero-barrier generation.
constexpr int kTaskList = 32;
struct CtaState {
    uint64_t in_bar[2];           // mbarriers of the two task-input buffers
    int list_count;
    unsigned in_phase;            // parity bit per input buffer
    unsigned long long bar_base;  // this CTA's grid flag at launch start
    int n_arrive;                 // grid-barrier arrivals so far in this launch
    int zero_ready;
    int prev_layer;
    long long prev_slice, prev_rg0, prev_rg1;
    int n_bar;                    // stage barriers passed (diagnostics)
    int zero_pending;             // this CTA's zeroing arrival (grid barrier 1) not made yet
    int sig_layer;                // row deps: producer task whose completion is still to signal
    long long sig_rg0, sig_rg1;
    // this CTA's task list, enumerated once at kernel start (task switches
    // must not walk the layer table: indexed parameter loads are slow)
    int l_stage[kMaxGroup], l_tasks[kMaxGroup];  // per layer, copied from the parameters
    int l_xcopy[kMaxGroup];       // per layer: x travels by bulk copy (x_by_copy)
    unsigned long long l_gen[kMaxGroup];  // producer layers: completed launches (row deps)
    // per layer, copied at kernel start by one thread each (loops over the layer
    // table would be chains of dependent indexed parameter loads, ~0.2 us per layer)
    float* xc_y[kMaxGroup];       // y
    int xc_elems[kMaxGroup];      // elements of y (rows * n)
    int z_per[kMaxGroup];         // elements of y each CTA zeroes (0: not split)
    float* mir[kMaxGroup];        // host mirror of y (null: none)
    long long xc_dl[kMaxRanks];   // peer address deltas (exchange launches)
    unsigned mir_stages;          // stages with a mirrored layer
    // row-shard exchange: counts at launch start, exchanges made, stages that push
    unsigned long long xc_base;
    int xc_n, xc_pushed;
    unsigned xc_push_mask, xc_layer_mask;  // stages that push, pushed layers (<= 32 each)
    int n_tl;                     // entries (kTaskList = more tasks follow)
    int tl_l[kTaskList], tl_g[kTaskList];
    long long tl_t[kTaskList];
};
static_assert(sizeof(CtaState) <= 3072, "CtaState exceeds its shared-memory slot (kState)");
struct PrevTask {
    int layer;
    long long slice, rg0, rg1;
};

// ---- grid barriers: one monotonic arrival counter ----
// grid_flags[0] counts arrival units of all CTAs over all launches that used
// this array; grid_flags[16 + c] (another cache line) is CTA c's own count,
// written at kernel end and read at the next launch's start.  Every such
// launch runs the full grid and every CTA arrives kBarUnits units per barrier,
// so at launch start counter = grid * own.  An arrival is a release reduction
// (fire-and-forget: no contended round trip); barrier k is passed once the
// counter reaches grid * (own + kBarUnits * k).
constexpr int kBarUnits = kWarps;  // the zero barrier: one unit per warp
__device__ __forceinline__ void grid_red(const GroupParams& p, unsigned units) {
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p.grid_flags),
                 "l"((unsigned long long)units)
                 : "memory");
}
// one thread; returns once every CTA made arrival k
__device__ __forceinline__ void grid_wait(const GroupParams& p, const CtaState& cs, int k) {
    const unsigned long long want =
        (cs.bar_base + (unsigned long long)kBarUnits * (unsigned long long)k) * gridDim.x;
    unsigned long long f;
    while (true) {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(f) : "l"(p.grid_flags) : "memory");
        if (f >= want) break;
        __nanosleep(32);
    }
}

// The zeroing arrival (grid barrier 1): every thread's zero stores are
// fenced (cheap by now), then one reduction per warp.
__device__ __forceinline__ void zero_arrive(const GroupParams& p, int tid) {
    __threadfence();
    __syncwarp();
    if ((tid & 31) == 0) grid_red(p, 1);
}

// ---- row-group readiness (kFlagRowDeps) ----
// A producer layer's counter rg_cnt[1 + rg] gains one per slice task covering
// row group rg once that task's contribution to y is complete (bulk
// reduce-adds drained, or plain stores) and released; rg_cnt[0] counts the
// launches that completed, so in this launch the row group is final at
// (gen + 1) * n_slices.  A consumer task waits (one warp) for the row groups
// of the producer's y that its x slice reads.
__device__ __forceinline__ void wait_rows(const unsigned long long* cnt, unsigned long long want,
                                          int64_t rg0, int64_t rg1, int lane) {
    for (int64_t rg = rg0 + lane; rg < rg1; rg += 32) {
        unsigned long long f;
        while (true) {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(f) : "l"(cnt + 1 + rg)
                         : "memory");
            if (f >= want) break;
            __nanosleep(32);
        }
    }
    __syncwarp();
}

// Signal the previous producer task's row groups (thread 0): its bulk
// reduce-adds are drained first and the async-proxy writes fenced; one
// release fence then orders everything before the relaxed increments.
__device__ __forceinline__ void signal_rows(const GroupParams& p, CtaState& cs) {
    if (cs.sig_layer < 0) return;
    const LayerTask& L = p.layer[cs.sig_layer];
    bulk_wait_all();
    asm volatile("fence.proxy.async.global;" ::: "memory");
    asm volatile("fence.acq_rel.gpu;" ::: "memory");  // one release for all the row groups
    for (long long rg = cs.sig_rg0; rg < cs.sig_rg1; ++rg)
        asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(L.rg_cnt + 1 + rg) : "memory");
    cs.sig_layer = -1;
}

// Split-K close of a task.  Every (row group, column) of the task takes a
// ticket (acq_rel atomic: releases our partials, acquires the others').
// Owner mode (persistent grid, one task per layer per CTA): slice s owns the
// s-th 1/n_slices of the row block's row groups; it waits until all slices
// have arrived on its row groups and sums them.  The wait is only on tasks of
// earlier layers (or at kernel end), which never wait on us: no deadlock.
// Last-arriver mode (grids beyond one wave): whoever arrives last sums.
__device__ __noinline__ void close_task_slow(const GroupParams& p, unsigned char* smem_raw, int tid);

// (the common case -- nothing to close -- stays inline; the deterministic
// split-K sums are out of line, keeping the hot kernel body small)
__device__ __forceinline__ void close_task(const GroupParams& p, unsigned char* smem_raw, int tid) {
    const CtaState& cs = *reinterpret_cast<const CtaState*>(smem_raw + p.off_bar);
    if (cs.prev_layer < 0) return;
    close_task_slow(p, smem_raw, tid);
}

__device__ __noinline__ void close_task_slow(const GroupParams& p, unsigned char* smem_raw, int tid) {
    CtaState& cs = *reinterpret_cast<CtaState*>(smem_raw + p.off_bar);
    const PrevTask prev{cs.prev_layer, cs.prev_slice, cs.prev_rg0, cs.prev_rg1};
    if (prev.layer < 0) return;
    const LayerTask& L = p.layer[prev.layer];
    if (L.n_slices <= 1) return;
    const int n = p.n, lane = tid & 31, warp = tid >> 5;
    const unsigned long long ns = (unsigned long long)L.n_slices;
    int* list_count = &cs.list_count;
    const int64_t nrg = prev.rg1 - prev.rg0;
    const bool owner_mode = !(p.flags & kFlagLastArriver);
    const int64_t share = (nrg + (int64_t)ns - 1) / (int64_t)ns;
    const int64_t own0 = prev.rg0 + prev.slice * share;
    const int64_t own1 = min(own0 + share, (int64_t)prev.rg1);
    unsigned long long* targets = reinterpret_cast<unsigned long long*>(smem_raw + p.off_list);
    FixupEntry* list = reinterpret_cast<FixupEntry*>(smem_raw + p.off_list);
    for (int64_t e = tid; e < nrg * n; e += kThreads) {
        const int64_t rg = prev.rg0 + e / n;
        const int col = (int)(e % n);
        unsigned long long old;
        asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;"
                     : "=l"(old)
                     : "l"(L.tickets + rg * n + col)
                     : "memory");
        if (owner_mode) {
            if (rg >= own0 && rg < own1) targets[(rg - own0) * n + col] = (old / ns + 1) * ns;
        } else if (old % ns == ns - 1) {
            const int slot = atomicAdd(list_count, 1);
            list[slot] = FixupEntry{prev.layer, col, (long long)rg};
        }
    }
    __syncthreads();
    if (owner_mode) {
        const int64_t nown = own1 > own0 ? own1 - own0 : 0;
        // wait for the other slices on the owned row groups
        for (int64_t e = tid; e < nown * n; e += kThreads) {
            const unsigned long long* t = L.tickets + (own0 + e / n) * n + (e % n);
            const unsigned long long want = targets[e];
            unsigned long long cur;
            do {
                asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(cur) : "l"(t) : "memory");
            } while (cur < want);
        }
        __syncthreads();
        // one thread per (row, column) of the owned row groups
        const int64_t r_lo = own0 * 16, r_hi = min(own1 * 16, L.rows);
        const int64_t nrows = r_hi > r_lo ? r_hi - r_lo : 0;
        for (int64_t e = tid; e < nrows * n; e += kThreads) {
            const int64_t row = r_lo + e / n;
            const int col = (int)(e % n);
            L.y[row * n + col] = sum_slices(L, n, row, col);
        }
    } else {
        const int cnt = *list_count;
        for (int e = warp; e < cnt; e += kWarps) {
            const FixupEntry f = list[e];
            fixup_row_group(p.layer[f.layer], n, f.rg, f.col, lane);
        }
    }
    __syncthreads();
    if (tid == 0) *list_count = 0;
}

// ---- task inputs: raw codebooks + x slice + scale tiles by TMA bulk copies
// into one of two smem buffers (double-buffered across tasks), so the next
// task's inputs travel while the current task gathers.
// A task is (layer l, task t of that layer).  Within a stage the tasks of
// all its layers are numbered consecutively (layer order) and CTA c runs
// numbers c, c + grid, ...; g is that stage-wide number.
struct TaskCoord {
    int l;
    int64_t t;
    int64_t g;
};

// stage-wide task number g of stage s -> (l, t), false past the stage; walks
// the shared-memory copy of the layers' {stage, n_tasks} (no dependent
// parameter-space loads: they cost ~0.8 us per walk)
__device__ __forceinline__ bool locate_s(const CtaState& cs, int nl, int s, int64_t g,
                                         TaskCoord& c) {
    int l = 0;
    while (l < nl && cs.l_stage[l] < s) ++l;
    int64_t r = g;
    while (l < nl && cs.l_stage[l] == s && r >= cs.l_tasks[l]) {
        r -= cs.l_tasks[l];
        ++l;
    }
    if (l >= nl || cs.l_stage[l] != s) return false;
    c.l = l;
    c.t = r;
    c.g = g;
    return true;
}
// the stage-wide task numbers of stage s this CTA runs: g0, g0 + step, ... below
// g_end.  Strided (c, c + G, ...) or, with kFlagContig and more tasks than CTAs,
// one contiguous range [c*T/G, (c+1)*T/G): tasks are numbered (layer, slice,
// row block) with the row block fastest, so a range crosses few K-slices.
__device__ __forceinline__ void stage_share(const CtaState& cs, int nl, int s, bool contig,
                                            int64_t& g0, int64_t& step, int64_t& g_end) {
    int64_t total = 0;
    for (int l = 0; l < nl; ++l)
        if (cs.l_stage[l] == s) total += cs.l_tasks[l];
    const int64_t G = gridDim.x, c = blockIdx.x;
    if (contig && total > G) {
        g0 = c * total / G;
        g_end = (c + 1) * total / G;
        step = 1;
    } else {
        g0 = c;
        g_end = total;
        step = G;
    }
}
__device__ __forceinline__ bool first_task_s(const CtaState& cs, int nl, int s, bool contig,
                                             TaskCoord& c) {
    int64_t g0, step, g_end;
    stage_share(cs, nl, s, contig, g0, step, g_end);
    return g0 < g_end && locate_s(cs, nl, s, g0, c);
}
__device__ __forceinline__ bool next_task_strided(const CtaState& cs, int nl, int ns, TaskCoord& c) {
    const int s = cs.l_stage[c.l];
    if (locate_s(cs, nl, s, c.g + gridDim.x, c)) return true;
    for (int s2 = s + 1; s2 < ns; ++s2)
        if (locate_s(cs, nl, s2, (int64_t)blockIdx.x, c)) return true;
    return false;
}
__device__ __forceinline__ bool next_task_s(const CtaState& cs, int nl, int ns, bool contig,
                                            TaskCoord& c) {
    const int s = cs.l_stage[c.l];
    int64_t g0, step, g_end;
    stage_share(cs, nl, s, contig, g0, step, g_end);
    if (c.g + step < g_end && locate_s(cs, nl, s, c.g + step, c)) return true;
    for (int s2 = s + 1; s2 < ns; ++s2)
        if (first_task_s(cs, nl, s2, contig, c)) return true;
    return false;
}

// x travels by bulk copy (binary16 or binary32) unless several columns or
// unaligned slices; not for a row-readiness consumer (its x is waited for
// per row group inside the task, after the copy would have been issued)
__device__ __forceinline__ bool x_by_copy(const GroupParams& p, const LayerTask& L) {
    return p.n == 1 && !(p.flags & kFlagXRegs) && (L.x32 == nullptr || L.dep < 0) && !L.xll &&
           L.llx < 0;
}

// Task geometry (all task counts fit in 32 bits).
struct TaskGeom {
    int slice, rb;
    int64_t rg0, rg1;
};
__device__ __forceinline__ TaskGeom task_geom(const LayerTask& L, int64_t t) {
    TaskGeom g;
    g.slice = (int)t / (int)L.n_rb;
    g.rb = (int)t - g.slice * (int)L.n_rb;
    g.rg0 = (int64_t)g.rb * L.rg_per_task;
    g.rg1 = min(g.rg0 + (int64_t)L.rg_per_task, L.n_rg);
    return g;
}

// One thread.  weights: scale tiles + codebooks (TMA bulk -> smem, mbarrier)
// and, unless disabled, a bulk L2 prefetch of the task's whole code range
// (contiguous in the prepacked layout) so HBM streams the codes while the
// CTA waits for x and builds the table; x: the slice of x (n == 1).
template <int V, int M, int U, int KB>
__device__ __forceinline__ void issue_inputs(const GroupParams& p, TaskCoord c, int buf,
                                             unsigned char* smem_raw, bool weights, bool x) {
    using S = FusedShape<V, M, U, KB>;
    const LayerTask& L = p.layer[c.l];
    CtaState& cs = *reinterpret_cast<CtaState*>(smem_raw + p.off_bar);
    const TaskGeom g = task_geom(L, c.t);
    const uint32_t scl_bytes = (uint32_t)((g.rg1 - g.rg0) * L.n_gs * 32);
    const uint32_t book_bytes = (uint32_t)((M * L.kcount * V * 2 + 15) & ~15);  // alloc is padded
    const int64_t e0 = (int64_t)g.slice * (S::kSliceSegs * V);
    const int64_t xn = min((int64_t)(S::kSliceSegs * V), L.cols - e0);
    const uint32_t x_bytes =
        x_by_copy(p, L) ? (uint32_t)(xn * (L.x32 ? 4 : 2)) : 0u;  // host: 16-B multiple
    uint64_t* bar = &cs.in_bar[buf];
    unsigned char* raw = smem_raw + p.off_raw[buf];
    if (weights) {
        mbar_expect_tx(bar, scl_bytes + book_bytes + x_bytes);
        bulk_g2s(smem_raw + p.off_scl[buf], L.scl + ((int64_t)g.slice * L.n_rg + g.rg0) * L.n_gs * 16,
                 scl_bytes, bar);
        bulk_g2s(raw, L.books, book_bytes, bar);
        if (!(p.flags & kFlagNoPrefetch)) {
            const uint8_t* base =
                L.codes + ((int64_t)g.slice * L.n_rg + g.rg0) * (int64_t)S::kTileBytes;
            // the whole range, or (pf_dist > 0) the first pf_dist rounds of row
            // groups; the gather then keeps pf_dist rounds ahead (rolling window)
            int64_t bytes = (g.rg1 - g.rg0) * (int64_t)S::kTileBytes;
            if (p.pf_dist > 0)
                bytes = min(bytes, (int64_t)p.pf_dist * kWarps * (int64_t)S::kTileBytes);
            constexpr int64_t kChunk = 32 * 1024;
            for (int64_t o = 0; o < bytes; o += kChunk)
                prefetch_l2_bulk(base + o, (uint32_t)min(kChunk, bytes - o));
        }
    }
    if (x && x_bytes)
        bulk_g2s(raw + p.raw_x_off,
                 L.x32 ? static_cast<const void*>(L.x32 + e0) : static_cast<const void*>(L.x + e0),
                 x_bytes, bar);
}

template <int V, int M, int U, int KB, bool CONTIG>
__device__ __forceinline__ void run_task(const GroupParams& p, TaskCoord c, int buf, bool first_task,
                                         bool has_next, bool x_next, TaskCoord nc,
                                         unsigned char* smem_raw, int tid, int task_idx,
                                         bool zero_todo, int& prev_l, int& prev_slice) {
    using S = FusedShape<V, M, U, KB>;
    constexpr int D = S::kDepth;
    const int l = c.l;
    const LayerTask& L = p.layer[l];
    float* psum = reinterpret_cast<float*>(smem_raw + p.off_psum);
    float* xs = reinterpret_cast<float*>(smem_raw + p.off_x);
    const uint16_t* scl_s = reinterpret_cast<const uint16_t*>(smem_raw + p.off_scl[buf]);
    const uint16_t* raw = reinterpret_cast<const uint16_t*>(smem_raw + p.off_raw[buf]);
    CtaState& cs = *reinterpret_cast<CtaState*>(smem_raw + p.off_bar);
    unsigned long long* stamps =
        (p.stamps && task_idx < 11) ? p.stamps + blockIdx.x * 128 + task_idx * 8 : nullptr;
#define CG_STAMP(k) \
    if (stamps && tid == 0) stamps[k] = gtimer();

    const int lane = tid & 31, warp = tid >> 5;
    const int n = p.n;
    const TaskGeom g = task_geom(L, c.t);
    const int slice = g.slice;
    const int64_t rg0 = g.rg0, rg1 = g.rg1;
    const int n_gs = L.n_gs;
    const uint8_t* tiles = L.codes + (int64_t)slice * L.n_rg * (int64_t)S::kTileBytes;
    const bool split = L.n_slices > 1;
    // the previous task of this CTA built this (layer, K-slice)'s Psumbook: the
    // table in shared memory is still valid (one column; nothing else writes it)
    bool reuse = false;
    if constexpr (CONTIG) {
        reuse = (p.flags & kFlagContig) && n == 1 && l == prev_l && slice == prev_slice;
        prev_l = l;
        prev_slice = slice;
    }
    CG_STAMP(0)

    // 1. this warp's first D code tiles into registers: they travel (from L2,
    //    where the task's range was bulk-prefetched) during the input wait
    //    and the table build
    const int my_rgs = rg0 + warp < rg1 ? (int)((rg1 - rg0 - warp + kWarps - 1) / kWarps) : 0;
    const uint8_t* cptr = tiles + (rg0 + warp) * S::kTileBytes + lane * S::kLaneBytes;
    constexpr int64_t kStep = (int64_t)kWarps * S::kTileBytes;
    uint4 tb[D][M][U];
#pragma unroll
    for (int d = 0; d < D; ++d)
        if (d < my_rgs) load_tile<V, M, U, KB>(tb[d], cptr + d * kStep);
    CG_FST(3)
    if (tid == 0) signal_rows(p, cs);  // the previous task, if a producer
    if (L.dep >= 0 && !reuse) {
        // x is an earlier stage's y: wait for the row groups this slice reads
        if (warp == 0) {
            const LayerTask& P = p.layer[L.dep];
            const int64_t e0 = (int64_t)slice * (S::kSliceSegs * V);
            const int64_t e1 = min(e0 + (int64_t)(S::kSliceSegs * V), L.cols);
            wait_rows(P.rg_cnt, (cs.l_gen[L.dep] + 1) * (unsigned long long)P.n_slices, e0 >> 4,
                      (e1 + 15) >> 4, lane);
        }
        __syncthreads();
    }
    uint16_t xreg[S::kXPerThread];
    if (reuse) {
    } else if (L.llx >= 0)
        load_x_llc<V, M, U, KB>(xreg, L, p.layer[L.llx], (unsigned)(cs.l_gen[L.llx] + 1),
                                L.llw && g.rb == 0, slice, tid,
                                (p.flags & kFlagDbgLL8) ? 8 : kLLGroup);
    else if (L.xll) load_x_ll<V, M, U, KB>(xreg, L, p, (unsigned)(cs.xc_base + 1), slice, n, 0, tid);
    else if (!x_by_copy(p, L)) load_x<V, M, U, KB>(xreg, L, slice, n, 0, tid);
    CG_FST(4)

    // 2. the previous task is done with the table; the staging buffer of two
    //    tasks ago has been read by its flush (the next task's inputs may be
    //    requested from here on: after the build, below); close the previous
    //    task's row groups (deterministic mode)
    if (tid == 0) bulk_wait_read_prev();
    __syncthreads();
    CG_STAMP(7)
    // (the next task's inputs are requested after this task's table build: issued
    // here, their TMA writes and the bulk L2 prefetch slowed the build by ~0.6 us
    // per stage -- 8B block 39.55 -> 38.0 us on one box, 70B unchanged)
    const bool early_issue = (p.flags & kFlagDbgEarlyIssue) != 0;
    if (tid == kThreads - 32 && has_next && early_issue)
        issue_inputs<V, M, U, KB>(p, nc, buf ^ 1, smem_raw, true, x_next);
    close_task(p, smem_raw, tid);
    mbar_wait(&cs.in_bar[buf], (cs.in_phase >> buf) & 1u);
    CG_STAMP(4)

    // per-lane constants of the gather (Psumbook base must be 64 KB aligned)
    const uint32_t psum_addr = smem_u32(psum);
    if (psum_addr & 0xffffu) __trap();
    const uint32_t lb0 = ((uint32_t)lane << 2) | ((psum_addr >> 16) << 8);
    const uint32_t lb1 = lb0 | 0x80u;
    const int lg = L.lg;  // lanes per scale group = 2**lg (host planner)
    const bool early = lg < 3;  // scales applied per lane (small groups)
    const int mask = row_mask(lane);
    const int gi = lg >= 5 ? 0 : (lane >> lg);
    const uint16_t* sp0 = scl_s + (warp * n_gs + gi) * 16;
    const int sstep = kWarps * n_gs * 16;
    // split-K partials: staged in smem and flushed by one bulk reduce-add per
    // task (one column), or -- several columns -- added straight into y with
    // red.global.add (staging would shrink tasks by the column count)
    const bool direct = split && !(p.flags & kFlagDeterministic) &&
                        (n > 1 || (p.flags & kFlagDirectAdd));
    const bool stage_out = (split && !(p.flags & kFlagDeterministic) && !direct) || L.llp != nullptr;
    const int64_t row_step = (int64_t)kWarps * 16;

    for (int col = 0; col < n; ++col) {
        if (col > 0) {
            __syncthreads();  // previous column's table is no longer read
            if (L.xll) load_x_ll<V, M, U, KB>(xreg, L, p, (unsigned)(cs.xc_base + 1), slice, n, col, tid);
            else load_x<V, M, U, KB>(xreg, L, slice, n, col, tid);
        }
        if (reuse) {
            // (no x, no build: the table of the previous task is this task's)
        } else if (x_by_copy(p, L)) {
            const int64_t e0 = (int64_t)slice * (S::kSliceSegs * V);
            const int valid = (int)min((int64_t)(S::kSliceSegs * V), L.cols - e0);
            if (L.x32)
                stage_x_raw32<V, M, U, KB>(
                    xs, reinterpret_cast<const float*>(raw + p.raw_x_off / 2), valid, tid);
            else
                stage_x_raw<V, M, U, KB>(xs, raw + p.raw_x_off / 2, valid, tid);
        } else {
            store_x<V, M, U, KB>(xs, xreg, tid);
        }
        if (!reuse) {
            __syncthreads();
            if (col == 0) CG_STAMP(5)
            if (!(p.flags & kFlagDbgSkipBuild))
                build_psumbook_smem<V, M, U, KB>(psum, raw, xs,
                                                 L.kcount, tid);
#ifdef CG_FINE_STAMPS
            if (p.stamps && lane == 0 && task_idx == 1) p.stamps[blockIdx.x * 128 + 96 + warp] = gtimer();
#endif
            __syncthreads();
        }
        if (col == 0) CG_STAMP(6)
        if (col == 0 && !early_issue && tid == kThreads - 32 && has_next)
            issue_inputs<V, M, U, KB>(p, nc, buf ^ 1, smem_raw, true, x_next);
        if (col == 0 && first_task) pdl_launch_dependents();
        if (col == 0 && zero_todo) zero_arrive(p, tid);
        if (col > 0) {
#pragma unroll
            for (int d = 0; d < D; ++d)
                if (d < my_rgs) load_tile<V, M, U, KB>(tb[d], cptr + d * kStep);
        }
        float* out = stage_out ? reinterpret_cast<float*>(smem_raw + p.off_stage[buf]) - rg0 * 16 * n
                               : (direct ? L.y : (split ? L.ws + (int64_t)slice * L.rows * n : L.y));
        if (direct && !cs.zero_ready) {  // y zeroed grid-wide before the first add
            __syncthreads();
            if (tid == 0) grid_wait(p, cs, 1);
            __syncthreads();
            if (tid == 0) cs.zero_ready = 1;
        }
        int64_t row = (rg0 + warp) * 16 + mask;
        // the output store of a row group, one predicated instruction per mode (no
        // generic-address branches in the loop: they split it into basic blocks the
        // scheduler cannot interleave): smem staging, red.add into y, or plain store
        const int64_t rows_l = L.rows;
        const uint32_t out_s = stage_out ? smem_u32(out) : 0u;
        const int out_mode = stage_out ? 1 : (direct ? 2 : 0);
        // D-deep register pipeline: tile i+D is requested as soon as tile i is consumed
        const int n_rgs = (p.flags & kFlagDbgSkipGather) ? 0 : my_rgs;
        const int pf = (p.flags & kFlagNoPrefetch) ? 0 : p.pf_dist;
        const int load_rgs = (p.flags & kFlagDbgNoLoads) ? 0 : my_rgs;
        for (int i0 = 0; i0 < n_rgs; i0 += D) {
#pragma unroll
            for (int d = 0; d < D; ++d) {
                const int i = i0 + d;
                if (i < n_rgs) {
                    if (pf > 0 && lane == 0 && i + pf < load_rgs)
                        prefetch_l2_bulk(cptr - lane * S::kLaneBytes + (i + pf) * kStep, S::kTileBytes);
                    const float v = gather_row_group<V, M, U, KB>(tb[d], sp0 + i * sstep, lb0, lb1,
                                                                  mask, early);
                    if (i + D < load_rgs) load_tile<V, M, U, KB>(tb[d], cptr + (i + D) * kStep);
                    {
                        const bool w = lane < 16 && row < rows_l;
                        const int64_t o = row * n + col;
                        asm volatile(
                            "{\n\t.reg .pred pw, pg, ps, pr;\n\t"
                            "setp.ne.s32 pw, %3, 0;\n\t"
                            "setp.eq.and.s32 pg, %2, 0, pw;\n\t"
                            "setp.eq.and.s32 ps, %2, 1, pw;\n\t"
                            "setp.eq.and.s32 pr, %2, 2, pw;\n\t"
                            "@pg st.global.f32 [%0], %4;\n\t"
                            "@ps st.shared.f32 [%1], %4;\n\t"
                            "@pr red.global.add.f32 [%0], %4;\n\t}"
                            ::"l"(out + o), "r"(out_s + (uint32_t)(o * 4)), "r"(out_mode),
                            "r"((int)w), "f"(v)
                            : "memory");
                    }
                    row += row_step;
                }
            }
        }
    }
    CG_STAMP(1)
    if (L.llp) {
        // LL-chain producer: the task's partial rows (slice `slice`) as (value,
        // epoch) pairs -- no reduction, no zeroed y, no barrier for the consumers
        __syncthreads();
        const float* stg = reinterpret_cast<const float*>(smem_raw + p.off_stage[buf]);
        const uint32_t epoch = (uint32_t)(cs.l_gen[l] + 1);
        const int64_t r1 = min(rg1 * 16, L.rows);
        float2* dst = L.llp + (int64_t)slice * L.rows + rg0 * 16;
        for (int64_t e = tid; e < r1 - rg0 * 16; e += kThreads)
            asm volatile("st.volatile.global.v2.u32 [%0], {%1,%2};" ::"l"(dst + e),
                         "r"(__float_as_uint(stg[e])), "r"(epoch));
    } else if (stage_out) {
        // flush the task's partial rows into y (L2 reduce-add); y was zeroed
        // by the grid at kernel start -- wait for that (arrival 1) once
        __syncthreads();
        if (warp == 0) {
            if (lane == 0) {
                if (!cs.zero_ready) {
                    grid_wait(p, cs, 1);
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                }
                cs.zero_ready = 1;
                CG_STAMP(2)
                const float* stage = reinterpret_cast<const float*>(smem_raw + p.off_stage[buf]);
                const int64_t r1 = min(rg1 * 16, L.rows);
                const int64_t elems = (r1 - rg0 * 16) * n;
                const int64_t body = elems & ~int64_t(3);  // 16-byte multiple
                if (body > 0) bulk_reduce_add_f32(L.y + rg0 * 16 * n, stage, (uint32_t)(body * 4));
                for (int64_t e = body; e < elems; ++e) atomicAdd(L.y + rg0 * 16 * n + e, stage[e]);
            }
        }
    }
    __syncthreads();
    if (tid == 0) {
        if (L.rg_cnt && !L.llp) {  // a later stage reads this y: signal at the next task start
            cs.sig_layer = l;
            cs.sig_rg0 = rg0;
            cs.sig_rg1 = rg1;
        }
        cs.in_phase ^= (1u << buf);
        cs.prev_layer = (split && (p.flags & kFlagDeterministic)) ? l : -1;
        cs.prev_slice = slice;
        cs.prev_rg0 = rg0;
        cs.prev_rg1 = rg1;
    }
    CG_STAMP(3)
#undef CG_STAMP
}

// ---- row-shard exchange over peer memory (NVLink P2P stores) ----
// One counter in each rank's region header (kXcArrive), written by every
// rank's CTAs with a system-scope fence + reductions and polled with
// system-scope acquires: it gains one per CTA per rank per exchange, so
// exchange k (counted over all launches on the comm) is complete at
// k * world * grid.  Every launch ends with an exchange (its last stage's rows,
// or none), made after all of the rank's reads: a rank writes into a peer's
// buffers only after every rank's previous exchanges -- hence previous
// launches -- are complete.  Per-CTA exchange counts at launch start come from
// the CTA's own slot (kXcOwnX), written at kernel end.
__device__ __forceinline__ void xc_fence(bool gpu_scope) {
    if (gpu_scope) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    else asm volatile("fence.acq_rel.sys;" ::: "memory");
}
// (arguments by value: called from out-of-line code, where every parameter
// access would be a generic load)
__device__ __forceinline__ void xc_wait(const unsigned long long* a, unsigned long long want,
                                        bool gpu_scope, unsigned long long timeout_ns) {
    unsigned long long f, t0 = 0;
    while (true) {
        if (gpu_scope) asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(f) : "l"(a) : "memory");
        else asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(f) : "l"(a) : "memory");
        if (f >= want) break;
        if (timeout_ns) {
            const unsigned long long t = gtimer();
            if (t0 == 0) t0 = t;
            else if (t - t0 > timeout_ns) __trap();  // a peer never arrived
        }
        __nanosleep(64);
    }
}
// one thread, after a CTA barrier that ordered the CTA's accesses before it:
// one fence releases them all, then plain reductions on every rank's counter
__device__ __forceinline__ void xc_signal(const GroupParams& p, int off) {
    const bool gs = (p.flags & kFlagDbgXcGpuScope) != 0;
    xc_fence(gs);
    for (int r = 0; r < p.xc_world; ++r)
        asm volatile("red.relaxed.sys.global.add.u64 [%0], 1;" ::"l"(p.xc_peer[r] + off) : "memory");
}
// thread 0, after griddepcontrol.wait: this CTA's counts, the pushing stages,
// and -- if a layer reads a buffer gathered by earlier launches -- the wait
// for every rank's pushes so far
__device__ __noinline__ void xc_prologue(const GroupParams& p, CtaState& cs) {
    const unsigned long long* own_x =
        reinterpret_cast<const unsigned long long*>(p.xc_local + kXcOwnX);
    cs.xc_base = own_x[blockIdx.x];
    cs.xc_n = 0;
    cs.xc_pushed = 0;
    unsigned mask = 0, lmask = 0;
    bool wait = false;
    for (int l = 0; l < p.n_layers; ++l) {
        const LayerTask& L = p.layer[l];
        if (L.xchg & kXchgPush) {
            mask |= 1u << L.stage;
            lmask |= 1u << l;
        }
        wait |= (L.xchg & kXchgWait) != 0;
    }
    cs.xc_push_mask = mask;
    cs.xc_layer_mask = lmask;
    if (wait) {
        xc_wait(reinterpret_cast<const unsigned long long*>(p.xc_local + kXcArrive),
                cs.xc_base * p.xc_world * gridDim.x, (p.flags & kFlagDbgXcGpuScope) != 0,
                p.xc_timeout_ns);
        asm volatile("fence.proxy.async.global;" ::: "memory");  // the x copies are TMA reads
    }
}
// all threads, after the grid barrier that closed `stage`: copy this CTA's
// share of the stage's pushed layers to every peer, release, signal (at the
// end of the launch also with nothing to push)
// (peer address deltas are read from the CTA state in shared memory: a pointer
// into the kernel parameters read from out-of-line code is a generic load per use)
__device__ __noinline__ void xc_push(unsigned char* smem_raw, int off_bar, int stage, int tid,
                                     int n_layers, int world, int rank,
                                     const unsigned long long* arrive, bool gpu_scope,
                                     unsigned long long timeout_ns, bool all_stages) {
    CtaState& cs = *reinterpret_cast<CtaState*>(smem_raw + off_bar);
    // (a launch's closing arrival with nothing to push; LL launches push every
    // stage's plain rows here, once)
    if (!all_stages && !((cs.xc_push_mask >> stage) & 1)) return;
    if (all_stages && !cs.xc_push_mask) return;
    if (!cs.xc_pushed) {
        // the first stores into peers' buffers in this launch: every rank has
        // finished its previous launches (and their reads)
        if (tid == 0) xc_wait(arrive, cs.xc_base * (unsigned long long)world * gridDim.x, gpu_scope,
                              timeout_ns);
        __syncthreads();
    }
    for (int r = 0; r < world; ++r) {
        if (r == rank) continue;
        const long long d = cs.xc_dl[r];
        for (int l = 0; l < n_layers; ++l) {
            if ((!all_stages && cs.l_stage[l] != stage) || !((cs.xc_layer_mask >> l) & 1)) continue;
            float* y = cs.xc_y[l];
            const int elems = cs.xc_elems[l];
            const int per = (((elems + (int)gridDim.x - 1) / (int)gridDim.x) + 3) & ~3;
            const int e0 = min((int)blockIdx.x * per, elems), e1 = min(e0 + per, elems);
            const bool vec = (reinterpret_cast<uintptr_t>(y) & 15) == 0;
            const int body = vec ? e0 + ((e1 - e0) & ~3) : e0;
            float* dst = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(y) + d);
            for (int e = e0 + 4 * tid; e < body; e += 4 * kThreads)
                *reinterpret_cast<float4*>(dst + e) = __ldcg(reinterpret_cast<const float4*>(y + e));
            for (int e = body + tid; e < e1; e += kThreads) dst[e] = __ldcg(y + e);
        }
    }
    __syncthreads();
}

// LL push (all threads, after the grid barrier that closed `stage`): this CTA's
// share of the stage's pushed layers into every rank's LL copy as (value,
// epoch) pairs -- 8-byte stores, no fence, no counter; consumers spin on the
// epoch.  The first stores of a launch wait until every rank finished its
// previous launches (their last exchange), so no LL slot is overwritten while
// a peer may still read it.
__device__ __noinline__ void xc_push_ll(unsigned char* smem_raw, int off_bar, int stage, int tid,
                                        int n_layers, int world,
                                        const unsigned long long* arrive, unsigned char* ll,
                                        const unsigned char* gbase, unsigned long long timeout_ns) {
    CtaState& cs = *reinterpret_cast<CtaState*>(smem_raw + off_bar);
    if (!((cs.xc_push_mask >> stage) & 1)) return;
    if (!cs.xc_pushed) {
        if (tid == 0) xc_wait(arrive, cs.xc_base * (unsigned long long)world * gridDim.x, false,
                              timeout_ns);
        __syncthreads();
        if (tid == 0) cs.xc_pushed = 1;
    }
    const uint32_t epoch = (uint32_t)(cs.xc_base + 1);
    for (int l = 0; l < n_layers; ++l) {
        if (cs.l_stage[l] != stage || !((cs.xc_layer_mask >> l) & 1)) continue;
        const float* y = cs.xc_y[l];
        const int elems = cs.xc_elems[l];
        const int per = (elems + (int)gridDim.x - 1) / (int)gridDim.x;
        const int e0 = min((int)blockIdx.x * per, elems), e1 = min(e0 + per, elems);
        unsigned char* dst0 = ll + 2 * (reinterpret_cast<const unsigned char*>(y) - gbase);
        for (int e = e0 + tid; e < e1; e += kThreads) {
            const uint32_t v = __float_as_uint(__ldcg(y + e));
            for (int r = 0; r < world; ++r) {
                float2* d = reinterpret_cast<float2*>(dst0 + cs.xc_dl[r]) + e;
                // (no "memory" clobber: the next layer's loads may be issued ahead of
                // these stores instead of one L2 round trip per layer)
                asm volatile("st.volatile.global.v2.u32 [%0], {%1,%2};" ::"l"(d), "r"(v), "r"(epoch));
            }
        }
    }
}

// Host mirror (all threads, after the grid barrier that closed `stage`): this
// CTA's share of the stage's mirrored layers copied to their host-mapped
// buffers -- plain stores over PCIe/C2C that overlap the later stages; stream
// completion makes them visible to the host.
__device__ __noinline__ void mirror_copy(unsigned char* smem_raw, int off_bar, int stage, int tid,
                                         int n_layers) {
    const CtaState& cs = *reinterpret_cast<const CtaState*>(smem_raw + off_bar);
    for (int l = 0; l < n_layers; ++l) {
        if (cs.l_stage[l] != stage || !cs.mir[l]) continue;
        const float* y = cs.xc_y[l];
        float* h = cs.mir[l];
        const int elems = cs.xc_elems[l];
        const int per = (((elems + (int)gridDim.x - 1) / (int)gridDim.x) + 3) & ~3;
        const int e0 = min((int)blockIdx.x * per, elems), e1 = min(e0 + per, elems);
        const bool vec = ((reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(h)) & 15) == 0;
        const int body = vec ? e0 + ((e1 - e0) & ~3) : e0;
        for (int e = e0 + 4 * tid; e < body; e += 4 * kThreads)
            *reinterpret_cast<float4*>(h + e) = __ldcg(reinterpret_cast<const float4*>(y + e));
        for (int e = body + tid; e < e1; e += kThreads) h[e] = __ldcg(y + e);
    }
}

// Grid barrier between dependent stages of a launch (the monotonic counter
// above).  Everything this CTA wrote in the stage -- plain stores and the bulk
// (async-proxy) reduce-adds -- is complete and released before the arrival;
// the next stage's x, read by TMA, is acquired after.  In an exchange launch
// the stage's rows then go to the peers (and, unless `final`, every rank's
// rows are awaited).
__device__ __forceinline__ void stage_barrier(const GroupParams& p, unsigned char* smem_raw,
                                              int tid, int stage, bool final = false) {
    __syncthreads();
    close_task(p, smem_raw, tid);  // deterministic split-K: pending ordered sums
    CtaState& cs = *reinterpret_cast<CtaState*>(smem_raw + p.off_bar);
    unsigned long long* st =
#ifdef CG_FINE_STAMPS
        nullptr;  // (slots 96.. hold per-warp stamps)
#else
        (p.stamps && cs.n_bar < 7) ? p.stamps + blockIdx.x * 128 + 96 + 4 * cs.n_bar : nullptr;
#endif
    if (tid == 0) {
        if (st) st[0] = gtimer();
        cs.prev_layer = -1;
        bulk_wait_all();
        asm volatile("fence.proxy.async.global;" ::: "memory");
        if (st) st[1] = gtimer();
        ++cs.n_arrive;
        grid_red(p, kBarUnits);
        if (st) st[2] = gtimer();
        grid_wait(p, cs, cs.n_arrive);
        asm volatile("fence.proxy.async.global;" ::: "memory");
        if (st) st[3] = gtimer();
        ++cs.n_bar;
    }
    __syncthreads();
    if ((cs.mir_stages >> stage) & 1) mirror_copy(smem_raw, p.off_bar, stage, tid, p.n_layers);
    if (p.xc_local && (p.flags & kFlagXcLL) && !final) {
        // LL: the stage's rows to every rank as (value, epoch) pairs; the next
        // stage's consumers spin on them -- no fence, no wait here
        if ((cs.xc_push_mask >> stage) & 1) {
            unsigned long long* xst = (p.stamps && stage < 4) ? p.stamps + blockIdx.x * 128 + 112 + 2 * stage
                                                              : nullptr;
            if (xst && tid == 0) xst[0] = gtimer();
            xc_push_ll(smem_raw, p.off_bar, stage, tid, p.n_layers, p.xc_world,
                       reinterpret_cast<const unsigned long long*>(p.xc_local + kXcArrive), p.xc_ll,
                       p.xc_gbase, p.xc_timeout_ns);
            if (xst && tid == 0) xst[1] = gtimer();
        }
        return;
    }
    if (p.xc_local && (((cs.xc_push_mask >> stage) & 1) || final)) {
        // row-shard exchange: the stage's rows to every peer, then (unless the
        // launch ends here) every rank's rows before the next stage reads them
        const bool gs = (p.flags & kFlagDbgXcGpuScope) != 0;
        const unsigned long long* arrive =
            reinterpret_cast<const unsigned long long*>(p.xc_local + kXcArrive);
        xc_push(smem_raw, p.off_bar, stage, tid, p.n_layers, p.xc_world, p.xc_rank,
                arrive, gs, p.xc_timeout_ns, (p.flags & kFlagXcLL) != 0);
        if (tid == 0) {
            // (the system-scope fence in here is the exchange's main cost: ~1.1 us
            // idle, ~4.5 us inside the kernel -- tools/micro/membar.cu, stamps)
            xc_signal(p, kXcArrive);
            cs.xc_pushed |= (cs.xc_push_mask >> stage) & 1;
            ++cs.xc_n;
        }
        unsigned long long* xst = (p.stamps && stage < 4) ? p.stamps + blockIdx.x * 128 + 112 + 2 * stage
                                                          : nullptr;
        if (xst && tid == 0) xst[0] = gtimer();
        if (!final && tid == 0) {
            xc_wait(arrive, (cs.xc_base + cs.xc_n) * (unsigned long long)p.xc_world * gridDim.x, gs,
                    p.xc_timeout_ns);
            asm volatile("fence.proxy.async.global;" ::: "memory");
            if (xst) xst[1] = gtimer();
        }
        __syncthreads();
    }
}

// this CTA's task list (warp 1, once per launch, beside thread 0's input
// issue): lane s counts the CTA's tasks in stage s (c, c + grid, ... below the
// stage's task total), a prefix scan places the stages in the list, and each
// lane locates list entries k = lane, lane + 32, ...  `scratch` is 128 ints of
// shared memory that no task uses yet.
template <bool CONTIG>
__device__ __forceinline__ void enumerate_tasks(int n_layers, int n_stages, CtaState& cs,
                                                int* scratch, int lane, bool contig) {
    int cnt = 0;
    int64_t g0 = 0, step = 1, g_end = 0;
    if constexpr (CONTIG) {
        if (lane < n_stages) {
            stage_share(cs, n_layers, lane, contig, g0, step, g_end);
            cnt = g0 < g_end ? (int)((g_end - g0 + step - 1) / step) : 0;
        }
    } else {
        const int G = gridDim.x, c = blockIdx.x;
        int total_s = 0;
        if (lane < n_stages)
            for (int l = 0; l < n_layers; ++l)
                if (cs.l_stage[l] == lane) total_s += cs.l_tasks[l];
        cnt = (lane < n_stages && c < total_s) ? (total_s - c + G - 1) / G : 0;
        g0 = c;
        step = G;
    }
    int pre = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, pre, off);
        if (lane >= off) pre += v;
    }
    const int total = __shfl_sync(0xffffffffu, pre, 31);
    scratch[lane] = pre - cnt;  // first list slot of stage `lane` (stages <= layers <= 32)
    scratch[32 + lane] = cnt;
    scratch[64 + lane] = (int)g0;
    scratch[96 + lane] = (int)step;
    __syncwarp();
    const int n = min(total, kTaskList);
    for (int k = lane; k < n; k += 32) {
        int s = 0;
        while (!(k >= scratch[s] && k < scratch[s] + scratch[32 + s])) ++s;
        TaskCoord e;
        locate_s(cs, n_layers, s, (int64_t)scratch[64 + s] + (int64_t)(k - scratch[s]) * scratch[96 + s],
                 e);
        cs.tl_l[k] = e.l;
        cs.tl_t[k] = e.t;
        cs.tl_g[k] = (int)e.g;
    }
    if (lane == 0) cs.n_tl = total > kTaskList ? kTaskList + 1 : total;
}

// A launch runs a chain of stages (all layers share the tiling u: one
// instantiation per (v, m, u, code width)); the layers of one stage are independent
// (a grouped launch: {q,k,v}, {gate,up}), stage s+1 may read what stage s
// wrote (its x is stage s's y).  CTA c runs tasks c, c+grid, ... of every
// layer of a stage, in layer order; stages are separated by grid barriers.
// The next task's weights (codebooks, scale tiles, code range into L2) are
// requested one task ahead -- across a stage boundary too -- and its x as
// soon as it is safe (same stage: at once; next stage: after the barrier).
template <int V, int M, int U, int KB, bool CONTIG>
__global__ void __launch_bounds__(kThreads, 1)
    group_gemv_kernel(const __grid_constant__ GroupParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (p.flags & kFlagDbgEmpty) return;
    const int tid = threadIdx.x;
    if (p.stamps && tid == 0) p.stamps[blockIdx.x * 128 + 124] = gtimer();
    CtaState& cs = *reinterpret_cast<CtaState*>(smem_raw + p.off_bar);
    // the layer table's per-layer fields into shared memory, one layer per warp
    // (lane 0): later loops over the layers read shared memory only
    for (int l = tid >> 5; l < p.n_layers; l += kWarps) {
        if ((tid & 31) == 0) {
            const LayerTask& L = p.layer[l];
            cs.l_stage[l] = L.stage;
            cs.l_tasks[l] = L.n_tasks;
            cs.xc_y[l] = L.y;
            cs.xc_elems[l] = (int)(L.rows * p.n);
            cs.z_per[l] = L.n_slices > 1 ? L.zero_per : 0;
            cs.mir[l] = L.mirror;
            cs.l_xcopy[l] = x_by_copy(p, L) ? 1 : 0;
        }
    }
    if (tid < kMaxRanks) cs.xc_dl[tid] = p.xc_delta[tid];
    if (tid == 0) {
        unsigned ms = 0;
        for (int l = 0; l < p.n_layers; ++l)
            if (p.layer[l].mirror) ms |= 1u << p.layer[l].stage;
        cs.mir_stages = ms;
    }
    __syncthreads();
    if (p.stamps && tid == 0) p.stamps[blockIdx.x * 128 + 88] = gtimer();
    TaskCoord c{0, 0, 0};
    bool have = false;
    const bool contig = CONTIG && (p.flags & kFlagContig) != 0;
    if constexpr (CONTIG) {
        for (int s = 0; s < p.n_stages && !have; ++s) have = first_task_s(cs, p.n_layers, s, contig, c);
    } else {
        for (int s = 0; s < p.n_stages && !have; ++s) have = locate_s(cs, p.n_layers, s, blockIdx.x, c);
    }
    if (p.stamps && tid == 0) p.stamps[blockIdx.x * 128 + 89] = gtimer();
    if (tid == 0) {
        mbar_init(&cs.in_bar[0], 1);
        mbar_init(&cs.in_bar[1], 1);
        cs.list_count = 0;
        cs.in_phase = 0;
        cs.zero_ready = 0;
        cs.prev_layer = -1;
        cs.n_bar = 0;
        cs.zero_pending = 0;
        cs.n_arrive = 0;
        cs.sig_layer = -1;
        // weights of the first task (and its code range into L2) travel
        // before the wait on the previous kernel
        if (have) issue_inputs<V, M, U, KB>(p, c, 0, smem_raw, true, false);
        if (p.stamps) p.stamps[blockIdx.x * 128 + 90] = gtimer();
    }
    if (tid >= 32 && tid < 64) {
        enumerate_tasks<CONTIG>(p.n_layers, p.n_stages, cs, reinterpret_cast<int*>(smem_raw + p.off_list),
                                tid & 31, contig);
        if (p.stamps && tid == 32) p.stamps[blockIdx.x * 128 + 91] = gtimer();
    }
    // every layer's x (and y, for write-after-read) belongs to earlier work
    pdl_wait();
    if (p.stamps && tid == 0) p.stamps[blockIdx.x * 128 + 126] = gtimer();
    int stage = 0;
    if (tid == 0 && p.xc_local) xc_prologue(p, cs);  // (gathered x: wait before it is copied)
    if (tid == 0 && have && cs.l_stage[c.l] == 0)
        issue_inputs<V, M, U, KB>(p, c, 0, smem_raw, false, true);
    if (p.stamps && tid == 0) p.stamps[blockIdx.x * 128 + 92] = gtimer();
    if (p.flags & (kFlagRowDeps | kFlagLLChain)) {  // producer generations, one layer per warp
        for (int l = tid >> 5; l < p.n_layers; l += kWarps) {
            if ((tid & 31) == 0 && p.layer[l].rg_cnt) {
                unsigned long long gv;
                asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(gv) : "l"(p.layer[l].rg_cnt)
                             : "memory");
                cs.l_gen[l] = gv;
            }
        }
    }
    if (tid == 32) {  // barrier state (used by thread 0 after the prologue barrier)
        unsigned long long b;
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(b)
                     : "l"(p.grid_flags + 16 + blockIdx.x)
                     : "memory");
        cs.bar_base = b;
    }
    if (!(p.flags & kFlagDeterministic)) {
        // zero this CTA's share of every split layer's output; each warp
        // releases its own stores (arrival 1: one unit per warp), so no CTA
        // barrier sits on this path -- the first flush waits for the grid
        bool any = false;
        const int nl = p.n_layers;
#pragma unroll 1
        for (int l = 0; l < nl; ++l) {
            const int per = cs.z_per[l];
            if (per == 0) continue;
            any = true;
            const int elems = cs.xc_elems[l];
            const int e0 = min((int)blockIdx.x * per, elems), e1 = min(e0 + per, elems);
            float* y = cs.xc_y[l];
            // (warps 0 and 1 issue the task inputs and list the tasks meanwhile)
            for (int e = e0 + tid - 64; e < e1 && tid >= 64; e += kThreads - 64) y[e] = 0.0f;
        }
        // the arrival (fenced) is made after the CTA's first Psumbook build,
        // when these stores have long completed -- off the prologue's path
        if ((any || (p.flags & (kFlagRowDeps | kFlagLLChain))) && tid == 0) {
            cs.n_arrive = 1;
            cs.zero_pending = 1;
        }
    }
    if (p.stamps && tid == 0) p.stamps[blockIdx.x * 128 + 93] = gtimer();
    __syncthreads();  // CTA state (task list, mbarriers) visible to every thread
    bool zero_todo = cs.zero_pending != 0;  // (same in every thread)
    if (p.stamps && tid == 0) p.stamps[blockIdx.x * 128 + 125] = gtimer();
    int buf = 0, task_idx = 0;
    int prev_l = -1, prev_slice = -1;  // (layer, K-slice) of the table in shared memory
    bool first = true;
    while (true) {
        CG_FST(0)
        const int target = have ? cs.l_stage[c.l] : p.n_stages - 1;
        while (stage < target) {  // (CTAs without tasks in a stage still take part)
            if (zero_todo) {  // the zeroing arrival precedes every stage arrival
                zero_arrive(p, tid);
                zero_todo = false;
            }
            if (!(p.flags & kFlagRowDeps) && !((p.bar_skip >> stage) & 1u))
                stage_barrier(p, smem_raw, tid, stage);
            ++stage;
            if (tid == 0 && have && stage == target && cs.l_xcopy[c.l])
                issue_inputs<V, M, U, KB>(p, c, buf, smem_raw, false, true);
        }
        CG_FST(1)
        if (!have) break;
        TaskCoord nc = c;
        bool has_next;
        if (task_idx + 1 < min(cs.n_tl, kTaskList)) {
            nc.l = cs.tl_l[task_idx + 1];
            nc.t = cs.tl_t[task_idx + 1];
            nc.g = cs.tl_g[task_idx + 1];
            has_next = true;
        } else if (cs.n_tl <= kTaskList && task_idx + 1 >= cs.n_tl) {
            has_next = false;
        } else {
            if constexpr (CONTIG)  // beyond the list (rare)
                has_next = next_task_s(cs, p.n_layers, p.n_stages, contig, nc);
            else
                has_next = next_task_strided(cs, p.n_layers, p.n_stages, nc);
        }
        const bool x_next = has_next && cs.l_stage[nc.l] == stage;
        CG_FST(2)
        run_task<V, M, U, KB, CONTIG>(p, c, buf, first, has_next, x_next, nc, smem_raw, tid, task_idx++,
                              zero_todo, prev_l, prev_slice);
        zero_todo = false;
        first = false;
        buf ^= 1;
        c = nc;
        have = has_next;
    }
    if (zero_todo) zero_arrive(p, tid);  // (a CTA without any task)
    // the last stage's mirrored outputs are final once every CTA closed its tasks:
    // one more grid barrier, then the copy (stage_barrier mirrors that stage)
    if ((cs.mir_stages >> (p.n_stages - 1)) & 1) stage_barrier(p, smem_raw, tid, p.n_stages - 1);
    // the last stage's rows to the peers (its consumers wait in a later
    // launch); the arrival also tells the peers this rank is done reading
    if (p.xc_local) stage_barrier(p, smem_raw, tid, p.n_stages - 1, true);
    // close the last task's row groups; drain the bulk reduce-adds
    __syncthreads();
    close_task(p, smem_raw, tid);
    if (tid == 0) {
        bulk_wait_all();
        signal_rows(p, cs);
        if ((p.flags & (kFlagRowDeps | kFlagLLChain)) && blockIdx.x == 0) {
            // every CTA read the generations before its arrival 1
            grid_wait(p, cs, 1);
            for (int l = 0; l < p.n_layers; ++l)
                if (p.layer[l].rg_cnt)
                    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p.layer[l].rg_cnt),
                                 "l"(cs.l_gen[l] + 1ull)
                                 : "memory");
        }
        // this CTA's arrival count for the next launch on these flags
        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p.grid_flags + 16 + blockIdx.x),
                     "l"(cs.bar_base + (unsigned long long)kBarUnits * cs.n_arrive)
                     : "memory");
        if (p.xc_local)  // exchange count for the next launch
            reinterpret_cast<unsigned long long*>(p.xc_local + kXcOwnX)[blockIdx.x] =
                cs.xc_base + (unsigned long long)cs.xc_n;
    }
    __syncthreads();
    if (p.stamps && tid == 0) p.stamps[blockIdx.x * 128 + 127] = gtimer();
}

// dump the fused kernel's smem Psumbook in _psum_tables layout (m, segs, 2**b, n):
// the same staging and build as the fused kernel, inputs read directly
template <int V, int M, int U, int KB>
__global__ void __launch_bounds__(kThreads, 1)
    psumbook_dump_kernel(const DumpParams p, float* __restrict__ out, int64_t segs) {
    using S = FusedShape<V, M, U, KB>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* psum = reinterpret_cast<float*>(smem_raw + p.off_psum);
    uint16_t* books16 = reinterpret_cast<uint16_t*>(smem_raw + p.off_books);
    float* xs = reinterpret_cast<float*>(smem_raw + p.off_x);
    const int tid = threadIdx.x;
    const int64_t slice = blockIdx.x;
    const int col = blockIdx.y;
    for (int e = tid; e < M * p.kcount * V; e += kThreads) books16[e] = p.books[e];
    uint16_t xreg[S::kXPerThread];
    load_x<V, M, U, KB>(xreg, p.x, slice, p.cols, p.n, col, tid);
    store_x<V, M, U, KB>(xs, xreg, tid);
    __syncthreads();
    build_psumbook_smem<V, M, U, KB>(psum, books16, xs,
                                     p.kcount, tid);
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
                                   int64_t groups, int64_t g_eff, int n, int u, int64_t n_rg,
                                   int cbits) {
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
                                        : packed_code(packed, t, r, seg, m, u, n_rg, cbits);
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

// K1 from binary32 inputs (engines.py:137-156 widens any float tile/book to
// binary32): products and sums rounded separately, as numpy's multiply + add
// (engines.py:126-133) -- with binary32 operands a product is not exact, so
// no fma here
__global__ void psumbook_build_f32_kernel(const float* __restrict__ books,
                                          const float* __restrict__ x, float* __restrict__ out,
                                          int m, int kcount, int v, int64_t segs, int n) {
    const int64_t total = (int64_t)m * segs * kcount * n;
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
         o += (int64_t)gridDim.x * blockDim.x) {
        const int col = (int)(o % n);
        const int64_t i = (o / n) % kcount;
        const int64_t seg = (o / ((int64_t)n * kcount)) % segs;
        const int64_t t = o / ((int64_t)n * kcount * segs);
        const float* c = books + (t * kcount + i) * v;
        float acc = 0.0f;
        for (int k = 0; k < v; ++k)
            acc = __fadd_rn(acc, __fmul_rn(c[k], x[(seg * v + k) * (int64_t)n + col]));
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
// the contiguous-schedule instance (Psumbook reuse) exists for the headline
// tilings only; elsewhere the host leaves kFlagContig clear
template <int V, int M, int U, int KB>
constexpr bool kContigInst = KB == 8 && ((V == 4 && M == 1 && U == 4) || (V == 8 && M == 2 && U == 2));

template <int V, int M, int U, int KB>
cudaError_t launch_group_t(const GroupParams& gp, int grid, int smem, bool pdl, cudaStream_t s) {
    void (*kern)(GroupParams) = group_gemv_kernel<V, M, U, KB, false>;
    static int smem_set[64] = {0};
    static int smem_set_c[64] = {0};
    cudaError_t e;
    if constexpr (kContigInst<V, M, U, KB>) {
        if (gp.flags & kFlagContig) {
            kern = group_gemv_kernel<V, M, U, KB, true>;
            e = set_smem_once(kern, smem, smem_set_c);
        } else {
            e = set_smem_once(kern, smem, smem_set);
        }
    } else {
        e = set_smem_once(kern, smem, smem_set);
    }
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    // grid barriers and owner-mode split-K wait on other CTAs: co-residency
    // guaranteed by a cooperative launch of the persistent (one-wave) grid
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (!(gp.flags & kFlagDbgNoCoop)) {
        attr[na].id = cudaLaunchAttributeCooperative;
        attr[na].val.cooperative = 1;
        ++na;
    }
    if (pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, gp);
}

template <int V, int M, int U, int KB>
cudaError_t launch_dump_t(const DumpParams& dp, int64_t n_slices, float* out, int64_t segs,
                          int smem, cudaStream_t s) {
    auto kern = psumbook_dump_kernel<V, M, U, KB>;
    static int smem_set[64] = {0};
    cudaError_t e = set_smem_once(kern, smem, smem_set);
    if (e != cudaSuccess) return e;
    kern<<<dim3((unsigned)n_slices, (unsigned)dp.n), kThreads, smem, s>>>(dp, out, segs);
    return cudaGetLastError();
}

// Instantiated set: v in {2,4,8,16}, m in {1,2,3,4}, kb in {4,8}; the group
// kernel switches on u at run time among u in {1,2,4} with m*u <= 4.
template <typename F>
bool visit_vmk(int v, int m, int kb, F&& f) {
#define CG_KB(V_, M_)                                  \
    if (kb == 4) return f.template run<V_, M_, 4>(), true; \
    if (kb == 8) return f.template run<V_, M_, 8>(), true; \
    if (kb == 6 && V_ == 4 && M_ == 1) return f.template run<V_, M_, 6>(), true; \
    return false;
#define CG_M(V_)                      \
    if (m == 1) { CG_KB(V_, 1) }      \
    if (m == 2) { CG_KB(V_, 2) }      \
    if (m == 3) { CG_KB(V_, 3) }      \
    if (m == 4) { CG_KB(V_, 4) }      \
    return false;
#ifdef CG_DEV_SUBSET  // fast edit-compile cycles: the two 2-bit headline configs only
    if (kb != 8) return false;
    if (v == 4 && m == 1) return f.template run<4, 1, 8>(), true;
    if (v == 8 && m == 2) return f.template run<8, 2, 8>(), true;
    return false;
#else
    switch (v) {
        case 2: { CG_M(2) }
        case 4: { CG_M(4) }
        case 8: { CG_M(8) }
        case 16: { CG_M(16) }
        default: return false;
    }
#endif
#undef CG_M
#undef CG_KB
}

template <typename F>
struct WithU {
    F& f;
    int u;
    template <int V, int M, int KB>
    void run() {
        if constexpr (KB == 6) {  // (6-bit streams: u = 4 only -- visit() checks)
            if constexpr (V == 4 && M == 1) f.template run<V, M, 4, KB>();
            return;
        } else {
        if constexpr (M * 4 <= 4) {
            if (u == 4) { f.template run<V, M, 4, KB>(); return; }
        }
        if constexpr (M * 2 <= 4) {
            if (u == 2) { f.template run<V, M, 2, KB>(); return; }
        }
        f.template run<V, M, 1, KB>();
        }
    }
};

template <typename F>
bool visit(int v, int m, int u, int kb, F&& f) {
    if (!(u == 1 || u == 2 || u == 4) || m * u > 4) return false;
    if (kb == 6 && u != 4) return false;
    WithU<std::remove_reference_t<F>> inner{f, u};
    return visit_vmk(v, m, kb, inner);
}

struct SizeQuery {
    FusedSizes z{};
    template <int V, int M, int U, int KB>
    void run() {
        using S = FusedShape<V, M, U, KB>;
        z = FusedSizes{S::kPsumBytes, M * S::kCodes * V * 2, S::kXBytes};
    }
};
struct GroupLaunch {
    const GroupParams* gp;
    int grid, smem;
    bool pdl;
    cudaStream_t s;
    cudaError_t err = cudaErrorInvalidConfiguration;
    template <int V, int M, int U, int KB>
    void run() { err = launch_group_t<V, M, U, KB>(*gp, grid, smem, pdl, s); }
};
struct DumpLaunch {
    const DumpParams* dp;
    int64_t n_slices;
    float* out;
    int64_t segs;
    int smem;
    cudaStream_t s;
    cudaError_t err = cudaErrorInvalidConfiguration;
    template <int V, int M, int U, int KB>
    void run() { err = launch_dump_t<V, M, U, KB>(*dp, n_slices, out, segs, smem, s); }
};

}  // namespace

bool fused_contig_instantiated(int v, int m, int u, int kbits) {
    return kbits == 8 && ((v == 4 && m == 1 && u == 4) || (v == 8 && m == 2 && u == 2));
}

bool fused_instantiated(int v, int m, int u, int kbits) {
    SizeQuery q;
    return visit(v, m, u, kbits, q);
}

bool fused_sizes(int v, int m, int u, int kbits, FusedSizes* out) {
    SizeQuery q;
    if (!visit(v, m, u, kbits, q)) return false;
    *out = q.z;
    return true;
}

cudaError_t launch_prepack_codes(const Plan& p, const uint16_t* raw, uint8_t* packed,
                                 unsigned* bad, cudaStream_t s) {
    const int64_t total = p.code_bytes;
    prepack_codes_kernel<<<grid_for(total, 256), 256, 0, s>>>(
        raw, packed, total, p.rows, p.segs, p.m, p.u, p.n_rg, 1u << p.b, bad, p.kbits);
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
                                                            p.m, p.u, p.n_rg, p.kbits);
    return cudaGetLastError();
}

cudaError_t launch_group_gemv(int v, int m, int u, int kbits, const GroupParams& gp, int grid,
                              int smem, bool pdl, cudaStream_t s) {
    GroupLaunch f{&gp, grid, smem, pdl, s};
    if (!visit(v, m, u, kbits, f)) return cudaErrorInvalidConfiguration;
    return f.err;
}

cudaError_t launch_psumbook_dump(const Plan& p, const DumpParams& dp, float* out, cudaStream_t s) {
    DumpLaunch f{&dp, p.n_slices, out, p.segs, p.smem.total, s};
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
        p.g_eff, n, p.u, p.n_rg, p.kbits);
    return cudaGetLastError();
}

cudaError_t launch_unpack_packed(const uint8_t* packed, int64_t plane_bytes, int m,
                                 int64_t per_plane, int b, uint16_t* out, cudaStream_t s) {
    unpack_packed_kernel<<<grid_for((int64_t)m * per_plane, 256), 256, 0, s>>>(
        packed, plane_bytes, m, per_plane, b, out);
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

cudaError_t launch_psumbook_build_f32(const float* books, const float* x, int m, int b, int v,
                                      int64_t k_len, int n, float* out, cudaStream_t s) {
    const int kcount = 1 << b;
    const int64_t segs = k_len / v;
    const int64_t total = (int64_t)m * segs * kcount * n;
    psumbook_build_f32_kernel<<<grid_for(total, 256), 256, 0, s>>>(books, x, out, m, kcount, v,
                                                                   segs, n);
    return cudaGetLastError();
}

}  // namespace cg
