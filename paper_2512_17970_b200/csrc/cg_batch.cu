// cg_batch.cu -- K4: the batch path (n >= 2 columns) of the code-gather GEMM.
//
// At batch 1 the Psumbook lookup (cg_kernels.cu) reads one binary32 table entry
// per code: shared-memory traffic m*rows*(K/v)*n entries, linear in the batch
// (engines.py:126-133, 293: one table per column).  At n >= 2 the same
// codebook reconstruction is cheaper as a register-level dequantisation feeding
// the tensor cores: each thread looks up the binary16 centroid pieces of its
// mma.sync A fragment in a lane-replicated codebook (one conflict-free LDS.64
// per 4 weights, independent of n) and the n columns ride in the MMA's N
// dimension.  The scales are applied per scale group to the binary32
// accumulators, i.e. y[r] = sum_groups s[r,g] * (sum over the group's
// segments of sum_t c_t[code] . x) -- the reference's per-segment structure
// (engines.py:286-294) with the products summed by the tensor core in binary32.
//
// Why mma.sync and not tcgen05 here: the A operand (the dequantised weights)
// is produced in registers by the lookups; tcgen05.mma reads A from shared
// memory or TMEM, which would add a store and a read of 2 bytes per weight on
// the same shared-memory pipe that bounds the lookups.  At n <= 32 the MMA work
// is a few percent of the tensor pipe; the kernel is bound by HBM (codes) and
// the LSU pipe (lookups), see DESIGN.md §4.
//
// Work split: a CTA task is (layer, 32 rows = 2 row tiles, K-slice); the 8 warps
// of the CTA take the slice's 128-element chunks round-robin, each warp
// accumulating both row tiles over its chunks, and the CTA sums the 8 warp
// partials in a fixed order through shared memory (deterministic).  CTAs are
// persistent: the lane-replicated codebook is built once, the x^T slice is
// staged once per (layer, slice) and kept while consecutive tasks share it,
// and each task's code tiles and scale tile arrive by TMA bulk copies into a
// second buffer while the previous task computes.  Slices (several only when
// x^T of the whole K does not fit) leave partial planes that a second kernel
// sums in slice order.
//
// Layout of the batch code stream (prepacked once per layer, on first use):
//   [row tile rt of 16 rows][chunk of 128 K elements][codebook t][lane'][16 B]
// Thread (g = lane/4, tq = lane%4) of a warp holds in its 16 bytes, for the 8
// mma k16 steps s of the chunk and rows g, g+8 (r = 0, 1), byte 2s+r = the code
// of codeword s*(16/v) + tq/(v/4) of row g+8r; lanes sharing a codeword (v > 4)
// share the 16 bytes (lane' = lane / (v/4)).  Within a k16 step, thread tq's
// "piece" is the 4 consecutive K elements 16s + 4tq .. +3 (piece tq % (v/4) of
// its codeword); the mma k index 2tq, 2tq+1 <-> piece elements 0, 1 and
// 2tq+8, 2tq+9 <-> 2, 3, for both A (weights) and B (x), so every product pairs
// the right weight with the right input element.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "cg_batch.h"
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


constexpr int kChunk = 128;  // K elements per code chunk (8 k16 steps)

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
    asm(  // (not volatile: a pure register op the scheduler may move)
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t word_of4(const uint4& q, int i) {
    return i == 0 ? q.x : (i == 1 ? q.y : (i == 2 ? q.z : q.w));
}

__device__ __forceinline__ void pdl_wait_b() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger_b() {
    asm volatile("griddepcontrol.launch_dependents;" :::);
}

// ---------------------------------------------------------------------------
// prepack: uint16 planes (m, rows, segs) -> batch code stream (one byte per code)
// ---------------------------------------------------------------------------
__global__ void prepack_batch_kernel(const uint16_t* __restrict__ raw, uint8_t* __restrict__ out,
                                     int64_t total, int64_t rows, int64_t segs, int m, int v,
                                     int64_t n_chunks) {
    const int lanes_u = 32 / (v / 4);       // distinct 16-byte slots per (rt, chunk, t)
    const int64_t unit = (int64_t)lanes_u * 16;
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
         o += (int64_t)gridDim.x * blockDim.x) {
        int64_t rest = o;
        const int byte = (int)(rest % 16);
        rest /= 16;
        const int lu = (int)(rest % lanes_u);
        rest /= lanes_u;
        const int t = (int)(rest % m);
        rest /= m;
        const int64_t ch = rest % n_chunks;
        const int64_t rt = rest / n_chunks;
        (void)unit;
        // lane' -> (g, codeword-in-step); byte -> (step s, row half r)
        const int lanes_per = v / 4;
        const int lane0 = lu * lanes_per;  // first lane of the group sharing these bytes
        const int g = lane0 >> 2, tq = lane0 & 3;
        const int s = byte >> 1, r = byte & 1;
        const int64_t row = rt * 16 + g + 8 * r;
        const int64_t cw = ch * (kChunk / v) + (int64_t)s * (16 / v) + tq / lanes_per;
        uint8_t val = 0;
        if (row < rows && cw < segs) val = static_cast<uint8_t>(raw[((int64_t)t * rows + row) * segs + cw]);
        out[o] = val;
    }
}

// ---------------------------------------------------------------------------
// batch scale layout: [32-row set][group][32 rows] binary16 (rows past the end 0),
// so one task's scale tile (its rows x its slice's groups) is one bulk copy
// ---------------------------------------------------------------------------
__global__ void prepack_batch_scales_kernel(const uint16_t* __restrict__ raw,
                                            uint16_t* __restrict__ out, int64_t total,
                                            int64_t rows, int64_t groups) {
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
         o += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = o & 31;
        const int64_t grp = (o >> 5) % groups;
        const int64_t rset = (o >> 5) / groups;
        const int64_t row = rset * 32 + r;
        out[o] = row < rows ? raw[row * groups + grp] : (uint16_t)0;
    }
}

template <int V, int M>
struct BShape {
    static constexpr int kPieces = V / 4;           // 4-element pieces per codeword
    static constexpr int kLanesU = 32 / kPieces;    // distinct code slots per chunk
    static constexpr int kUnit = kLanesU * 16;      // bytes per (row tile, chunk, codebook)
    static constexpr int kTileChunk = M * kUnit;    // bytes per (row tile, chunk)
};

// lane-replicated codebook: entry (t, code, piece, rep) = 8 bytes at
// (((t * kcount + code) * pieces + piece) * 16 + rep) * 8, rep = lane % 16

__device__ __forceinline__ void bmbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bmbar_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bcopy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void bmbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAITB_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAITB_%=;\n}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

struct BTask {
    int l, slice, rset;
};
// (the layer table is read from the CTA's shared-memory copy: indexed
// parameter-space loads are slow)
__device__ __forceinline__ BTask btask(const BatchLayer* sl, int n_layers, int t) {
    int l = 0;
    while (l < n_layers - 1 && t >= sl[l].n_tasks) {
        t -= sl[l].n_tasks;
        ++l;
    }
    const int rs = sl[l].n_rsets;
    return BTask{l, t / rs, t - (t / rs) * rs};
}

// one thread: the task's code tiles (2 row tiles) and scale tile into buffer `buf`
// (arguments by value: kernel parameters read through a reference in device
// code become generic loads -- ~1 us each here)
template <int V, int M>
__device__ __forceinline__ void issue_task(const BatchLayer* sl, BTask k, unsigned char* dst_codes,
                                           int tile_stride, unsigned char* dst_scl, uint64_t* bar) {
    using S = BShape<V, M>;
    const BatchLayer& L = sl[k.l];
    const int ch0 = k.slice * L.ks_chunks;
    const int nch = min(L.ks_chunks, L.n_chunks - ch0);
    const uint32_t tile_bytes = (uint32_t)(nch * S::kTileChunk);
    const int64_t grp0 = L.g_row ? 0 : (ch0 * 128) / (int)L.g_eff;  // (32-bit: K < 2^31)
    const int gis = (int)min((int64_t)L.gis, L.groups - grp0);
    const uint32_t scl_bytes = (uint32_t)gis * 64;
    int live = 0;
    for (int mt = 0; mt < 2; ++mt) live += (k.rset * 2 + mt < L.n_rt);
    bmbar_expect(bar, tile_bytes * live + scl_bytes);
    for (int mt = 0; mt < 2; ++mt) {
        const int rt = k.rset * 2 + mt;
        if (rt < L.n_rt)
            bcopy(dst_codes + mt * tile_stride,
                  L.codes + ((int64_t)rt * L.n_chunks + ch0) * S::kTileChunk, tile_bytes, bar);
    }
    bcopy(dst_scl, L.scl + ((int64_t)k.rset * L.groups + grp0) * 32, scl_bytes, bar);
}

// ---------------------------------------------------------------------------
// K4 (persistent): CTA c runs tasks [c*T/G, (c+1)*T/G) -- consecutive tasks of
// a CTA mostly share (layer, slice), so the x^T slice stays staged.
// NT = n8 tiles of the batch (n <= 8*NT).
// ---------------------------------------------------------------------------
// warps per CTA: 16 (two per scheduler more than 8: the lookup -> MMA latency
// chains need them) where the registers allow, 8 at NT = 4
template <int NT>
struct BWarps {
    static constexpr int kWarps = NT == 4 ? 8 : 16;
    static constexpr int kThreads = kWarps * 32;
};

template <int V, int M, int NT, bool SMALL>
__global__ void __launch_bounds__(BWarps<NT>::kThreads, 1)
    batch_gemm_kernel(const __grid_constant__ BatchParams p) {
    constexpr int kBatchWarps = BWarps<NT>::kWarps;
    constexpr int kBatchThreads = BWarps<NT>::kThreads;
    using S = BShape<V, M>;
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, tq = lane & 3;
    const int n = p.n;
    const int T = p.total_tasks, G = gridDim.x;
    const int t_begin = (int)((int64_t)blockIdx.x * T / G);
    const int t_end = (int)((int64_t)(blockIdx.x + 1) * T / G);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bar);
    float* red = reinterpret_cast<float*>(smem + p.off_red);
    uint16_t* xT = reinterpret_cast<uint16_t*>(smem + p.off_x);
    unsigned long long* st = p.stamps ? p.stamps + blockIdx.x * 64 : nullptr;
#define CG_BSTAMP(i) \
    if (st && tid == 0 && (i) < 64) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(st[i]));
    CG_BSTAMP(0)
    __shared__ BatchLayer sl[kMaxBatchGroup];
    if (tid < p.n_layers) sl[tid] = p.layer[tid];
    if (tid == 32) {
        bmbar_init(&bars[0]);
        bmbar_init(&bars[1]);
    }
    __syncthreads();
    const int nl = p.n_layers;
    // buffer addresses and strides into registers once (no indexed parameter loads later)
    unsigned char* const codes_buf[2] = {smem + p.off_codes[0], smem + p.off_codes[1]};
    unsigned char* const scl_buf[2] = {smem + p.off_scl[0], smem + p.off_scl[1]};
    const int tile_stride = p.code_tile_bytes;
    // the first task's weights travel before the wait on the previous kernel
    if (tid == 0 && t_begin < t_end)
        issue_task<V, M>(sl, btask(sl, nl, t_begin), codes_buf[0], tile_stride, scl_buf[0], &bars[0]);
    const int piece = tq % S::kPieces;
    const int rep = lane & 15;
    const int lu = lane / S::kPieces;
    int cur_l = -1, cur_slice = -1;
    unsigned phase = 0;
    bool waited = false;
    for (int t = t_begin; t < t_end; ++t) {
        const int buf = (t - t_begin) & 1;
        CG_BSTAMP(50 + (t - t_begin))
        const BTask k = btask(sl, nl, t);
        const BatchLayer& L = sl[k.l];
        const int ch0 = k.slice * L.ks_chunks;
        const int nch = min(L.ks_chunks, L.n_chunks - ch0);
        const int kslice = L.ks_chunks * 128;
        const int xstride = kslice + 16;  // halves: +32 B per column, conflict-free LDS.64
        if (k.l != cur_l || k.slice != cur_slice) {
            __syncthreads();  // every warp is done with the previous table / x^T
            if (k.l != cur_l) {  // lane-replicated codebook of this layer
                // raw binary16 books -> scratch (the reduction buffer), one 16-byte
                // load per thread in flight; then 16 copies of every 8-byte piece,
                // a half-warp writing one piece's 128 contiguous bytes
                const int raw_vec = (M * L.kcount * V * 2 + 15) / 16;  // (alloc padded to 16 B)
                uint4* scratch = reinterpret_cast<uint4*>(smem + p.off_red);
                for (int e = tid; e < raw_vec; e += kBatchThreads)
                    scratch[e] = __ldg(reinterpret_cast<const uint4*>(L.books) + e);
                __syncthreads();
                const int total = M * L.kcount * S::kPieces;
                const uint2* pieces = reinterpret_cast<const uint2*>(scratch);
                for (int e = tid; e < total * 16; e += kBatchThreads)
                    *reinterpret_cast<uint2*>(smem + p.off_tbl + (int64_t)e * 8) = pieces[e >> 4];
                __syncthreads();  // (scratch is the reduction buffer; the table is read below)
            }
            if (!waited) {
                pdl_wait_b();  // x may be written by the previous kernel in the stream
                waited = true;
            }
            // x^T slice: xT[c][kk] = x[k0 + kk][c_off + c].  The slice's rows of x
            // are one contiguous run; a thread reads 16-byte chunks (four in
            // flight) and scatters their halves with 2-byte stores -- for ld a
            // multiple of 8 a chunk is 8 columns of one row (a warp's stores for
            // one column cover 32 consecutive k: conflict-free), for ld = 1, 2, 4
            // it is 8/ld whole rows.
            {
                const int k0 = ch0 * 128;
                const int rows_valid = (int)min((int64_t)nch * 128, L.cols - k0);
                const int ld = p.ld;
                const int c_off = (int)(L.x - L.x0);
                const uint4* blk = reinterpret_cast<const uint4*>(L.x0 + (int64_t)k0 * ld);
                const int total = rows_valid * ld;       // halves of the run
                const int nfull = total / 8;             // whole 16-byte chunks
                // padding of the MMA tiles: columns past n (16 B at a time), rows past cols
                const int kv = nch * 16;                 // 16-byte pieces per x^T row
                for (int e = tid; e < (NT * 8 - n) * kv; e += kBatchThreads) {
                    const int c = n + e / kv, q = e - (e / kv) * kv;
                    *reinterpret_cast<uint4*>(xT + c * xstride + q * 8) = make_uint4(0u, 0u, 0u, 0u);
                }
                for (int c = 0; c < n && rows_valid < nch * 128; ++c)
                    for (int kk = rows_valid + tid; kk < nch * 128; kk += kBatchThreads)
                        xT[c * xstride + kk] = 0;
                if (ld % 8 == 0 || 8 % ld == 0) {
                    const int cpr = ld >= 8 ? ld / 8 : 1;   // chunks per row
                    const int rpc = ld >= 8 ? 1 : 8 / ld;   // rows per chunk
                    for (int q0 = tid; q0 < nfull; q0 += 4 * kBatchThreads) {
                        uint4 v4[4];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int q = q0 + j * kBatchThreads;
                            v4[j] = q < nfull ? __ldcg(blk + q) : make_uint4(0u, 0u, 0u, 0u);
                        }
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int q = q0 + j * kBatchThreads;
                            if (q >= nfull) break;
                            const uint32_t w[4] = {v4[j].x, v4[j].y, v4[j].z, v4[j].w};
                            const int kk0 = ld >= 8 ? q / cpr : q * rpc;
                            const int cb = ld >= 8 ? (q - kk0 * cpr) * 8 : 0;
#pragma unroll
                            for (int h = 0; h < 8; ++h) {
                                const int kk = ld >= 8 ? kk0 : kk0 + h / ld;
                                const int c = (ld >= 8 ? cb + h : h % ld) - c_off;
                                if (c >= 0 && c < n)
                                    xT[c * xstride + kk] = (uint16_t)(w[h >> 1] >> (16 * (h & 1)));
                            }
                        }
                    }
                    // (a run that is not a whole number of chunks: its last halves)
                    const uint16_t* xs = L.x0 + (int64_t)k0 * ld;
                    for (int e = nfull * 8 + tid; e < total; e += kBatchThreads) {
                        const int kk = e / ld, c = e - (e / ld) * ld - c_off;
                        if (c >= 0 && c < n) xT[c * xstride + kk] = xs[e];
                    }
                } else {  // other row widths: one half at a time
                    const uint16_t* xs = L.x0 + (int64_t)k0 * ld;
                    for (int e = tid; e < total; e += kBatchThreads) {
                        const int kk = e / ld, c = e - (e / ld) * ld - c_off;
                        if (c >= 0 && c < n) xT[c * xstride + kk] = __ldcg(xs + e);
                    }
                }
            }
            cur_l = k.l;
            cur_slice = k.slice;
            __syncthreads();
            CG_BSTAMP(1)
        }
        // the next task's code and scale tiles into the other buffer (its last
        // reader, the task before this one, finished at that task's end barrier)
        CG_BSTAMP(40 + (t - t_begin))
        if (tid == 0 && t + 1 < t_end)
            issue_task<V, M>(sl, btask(sl, nl, t + 1), buf ? codes_buf[0] : codes_buf[1], tile_stride,
                             buf ? scl_buf[0] : scl_buf[1], &bars[buf ^ 1]);
        CG_BSTAMP(2 + 3 * (t - t_begin))
        bmbar_wait(&bars[buf], (phase >> buf) & 1u);
        phase ^= 1u << buf;
        CG_BSTAMP(3 + 3 * (t - t_begin))

        // ---- this warp's chunks: ci = warp, warp + 8, ...
        const unsigned char* codes = buf ? codes_buf[1] : codes_buf[0];
        const uint16_t* scl = reinterpret_cast<const uint16_t*>(buf ? scl_buf[1] : scl_buf[0]);
        const int64_t grp0 = L.g_row ? 0 : (ch0 * 128) / (int)L.g_eff;  // (32-bit: K < 2^31)
        const int gis = (int)min((int64_t)L.gis, L.groups - grp0);
        // scale groups: SMALL (16/32/64 elements: spg = 1, 2 or 4 steps) close
        // inside a chunk; otherwise a group spans whole chunks (cpg of them) or the
        // whole slice (one_scale: applied once, after the last chunk)
        const int spg = L.spg;
        const bool one_scale = spg >= 8 * L.ks_chunks;
        const int cpg = spg >= 8 ? spg / 8 : 1;  // chunks per group (large groups)
        const int spg_lg = spg >= 4 ? 2 : (spg >> 1);  // (small groups: log2 spg)
        const uint32_t live0 = k.rset * 2 < L.n_rt ? 0xffffffffu : 0u;
        const uint32_t live1 = k.rset * 2 + 1 < L.n_rt ? 0xffffffffu : 0u;
        // AC accumulator copies (step s -> copy s % AC): 8 independent MMA chains
        // per warp whatever NT, so the tensor-core latency overlaps
        constexpr int AC = NT == 1 ? 4 : (NT == 2 ? 2 : 1);
        float tot[2][NT][4], acc[AC][2][NT][4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    tot[mt][nt][j] = 0.0f;
#pragma unroll
                    for (int a = 0; a < AC; ++a) acc[a][mt][nt][j] = 0.0f;
                }
        // tot += s[row, gi] * (sum of the accumulator copies); copies reset
        auto close_group = [&](int gi) {
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                const int rl = mt * 16 + g;
                const bool ok = gi < gis;
                const float s0 = ok ? __half2float(__ushort_as_half(scl[gi * 32 + rl])) : 0.0f;
                const float s1 = ok ? __half2float(__ushort_as_half(scl[gi * 32 + rl + 8])) : 0.0f;
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        float a = acc[0][mt][nt][j];
#pragma unroll
                        for (int c = 1; c < AC; ++c) a += acc[c][mt][nt][j];
                        tot[mt][nt][j] = fmaf(j < 2 ? s0 : s1, a, tot[mt][nt][j]);
#pragma unroll
                        for (int c = 0; c < AC; ++c) acc[c][mt][nt][j] = 0.0f;
                    }
            }
        };
        const uint2* x_a = reinterpret_cast<const uint2*>(xT + g * xstride + 4 * tq);
        // per-codebook lookup base: entry (t, code) of this lane's piece and copy
        const uint2* tbase[M];
#pragma unroll
        for (int t2 = 0; t2 < M; ++t2)
            tbase[t2] = reinterpret_cast<const uint2*>(smem + p.off_tbl) +
                        ((t2 * L.kcount) * S::kPieces + piece) * 16 + rep;
        constexpr int kCodeShift = S::kPieces == 1 ? 4 : 5;  // uint2 entries per code: 16 * pieces
        for (int ci = warp; ci < nch; ci += kBatchWarps) {
            // code words of the chunk (a row tile past the layer's end reads code 0)
            uint4 cw[2][M];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int t2 = 0; t2 < M; ++t2) {
                    uint4 q = *reinterpret_cast<const uint4*>(codes + mt * tile_stride +
                                                              (ci * M + t2) * S::kUnit + lu * 16);
                    const uint32_t lm = mt ? live1 : live0;
                    cw[mt][t2] = make_uint4(q.x & lm, q.y & lm, q.z & lm, q.w & lm);
                }
#pragma unroll
            for (int s = 0; s < 8; ++s) {
                uint2 bx[NT];
                const uint2* xs = x_a + (ci * 8 + s) * 4;  // 16 halves per step
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) bx[nt] = xs[nt * 8 * xstride / 4];
#pragma unroll
                for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
                    for (int t2 = 0; t2 < M; ++t2) {
                        const uint32_t w = word_of4(cw[mt][t2], s >> 1);
                        const uint32_t b0 = 2 * (s & 1);
                        const uint32_t c0 = __byte_perm(w, 0u, 0x4440u | b0);        // row g
                        const uint32_t c1 = __byte_perm(w, 0u, 0x4440u | (b0 + 1));  // row g + 8
                        const uint2 e0 = tbase[t2][c0 << kCodeShift];
                        const uint2 e1 = tbase[t2][c1 << kCodeShift];
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt)
                            mma16816(acc[s % AC][mt][nt], e0.x, e1.x, e0.y, e1.y, bx[nt].x,
                                     bx[nt].y);
                    }
                }
                if constexpr (SMALL) {  // groups of spg (1, 2, 4) steps
                    if (spg < 8 && ((s + 1) & (spg - 1)) == 0) close_group((ci * 8 + s) >> spg_lg);
                }
            }
            if (spg >= 8 && !one_scale) close_group(ci / cpg);
        }
        if (one_scale) close_group(0);
        // ---- CTA sum of the 8 warp partials (warp order: deterministic)
        constexpr int kCols = NT * 8;
        constexpr int kRed = kCols + 2;  // row stride of the partials (+8 B: rows g, g+8 in
                                         // different banks; keeps float2 alignment)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int row = mt * 16 + g + 8 * h;
                    const int col = nt * 8 + 2 * tq;
                    *reinterpret_cast<float2*>(red + (warp * 32 + row) * kRed + col) =
                        make_float2(tot[mt][nt][2 * h], tot[mt][nt][2 * h + 1]);
                }
        __syncthreads();
        const bool split = L.n_slices > 1;
        float* out = split ? L.ws + (int64_t)k.slice * L.rows * n : L.y;
        const int ldo = split ? n : p.ld;
        for (int e = tid; e < 32 * kCols; e += kBatchThreads) {
            const int row = e / kCols, col = e - (e / kCols) * kCols;
            const int64_t grow = (int64_t)k.rset * 32 + row;
            if (col >= n || grow >= L.rows) continue;
            float a = red[row * kRed + col];
#pragma unroll
            for (int w = 1; w < kBatchWarps; ++w) a += red[(w * 32 + row) * kRed + col];
            out[grow * ldo + col] = a;
        }
        __syncthreads();  // red and this buffer are free for the next task
        CG_BSTAMP(4 + 3 * (t - t_begin))
    }
    pdl_trigger_b();
#undef CG_BSTAMP
}

// y[r][c] = sum over slices (ascending) of ws[s][r][c]: fixed order, deterministic
__global__ void batch_reduce_kernel(const __grid_constant__ BatchParams p) {
    pdl_wait_b();
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (int l = 0; l < p.n_layers; ++l) {
        const BatchLayer& L = p.layer[l];
        const int64_t elems = L.rows * p.n;
        if (L.n_slices > 1) {
            for (int64_t i = e; i < elems; i += (int64_t)gridDim.x * blockDim.x) {
                float a = __ldcg(L.ws + i);
                for (int s = 1; s < L.n_slices; ++s) a += __ldcg(L.ws + (int64_t)s * elems + i);
                L.y[(i / p.n) * p.ld + (i % p.n)] = a;
            }
        }
    }
}

template <int V, int M, int NT, bool SMALL>
cudaError_t launch_batch_t(const BatchParams& bp, int grid, int smem, cudaStream_t s, bool pdl) {
    auto kern = batch_gemm_kernel<V, M, NT, SMALL>;
    static int smem_set[64] = {0};
    cudaError_t e = set_smem_once(kern, smem, smem_set);
    if (e != cudaSuccess) return e;
    bool reduce = false;
    for (int l = 0; l < bp.n_layers; ++l) reduce |= bp.layer[l].n_slices > 1;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid, 1, 1);
    cfg.blockDim = dim3(BWarps<NT>::kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    e = cudaLaunchKernelEx(&cfg, kern, bp);
    if (e != cudaSuccess || !reduce) return e;
    int64_t elems = 0;
    for (int l = 0; l < bp.n_layers; ++l)
        if (bp.layer[l].n_slices > 1 && bp.layer[l].rows * bp.n > elems) elems = bp.layer[l].rows * bp.n;
    cudaLaunchConfig_t rc = {};
    int64_t blocks = (elems + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    rc.gridDim = dim3((unsigned)(blocks < 1 ? 1 : blocks), 1, 1);
    rc.blockDim = dim3(256, 1, 1);
    rc.stream = s;
    rc.attrs = attr;
    rc.numAttrs = 1;
    return cudaLaunchKernelEx(&rc, batch_reduce_kernel, bp);
}

template <int V, int M, bool SMALL>
cudaError_t launch_batch_vms(int nt, const BatchParams& bp, int grid, int smem, cudaStream_t s,
                             bool pdl) {
    switch (nt) {
        case 1: return launch_batch_t<V, M, 1, SMALL>(bp, grid, smem, s, pdl);
        case 2: return launch_batch_t<V, M, 2, SMALL>(bp, grid, smem, s, pdl);
        case 4: return launch_batch_t<V, M, 4, SMALL>(bp, grid, smem, s, pdl);
        default: return cudaErrorInvalidConfiguration;
    }
}

// SMALL: some layer of the launch has scale groups of 16/32/64 elements
template <int V, int M>
cudaError_t launch_batch_vm(int nt, const BatchParams& bp, int grid, int smem, cudaStream_t s,
                            bool pdl) {
    bool small = false;
    for (int l = 0; l < bp.n_layers; ++l) small |= bp.layer[l].spg < 8;
    return small ? launch_batch_vms<V, M, true>(nt, bp, grid, smem, s, pdl)
                 : launch_batch_vms<V, M, false>(nt, bp, grid, smem, s, pdl);
}

}  // namespace

bool batch_supported_vm(int v, int m) { return (v == 4 || v == 8) && (m == 1 || m == 2); }

int batch_nt_for(int n) { return n <= 8 ? 1 : (n <= 16 ? 2 : 4); }

int batch_code_unit(int v) { return (32 / (v / 4)) * 16; }

// shared-memory layout of a launch whose largest layer has these sizes
int batch_layout(int v, int m, int kcount, int nt, int ks_chunks, int gis, BatchParams* bp) {
    auto up = [](int x) { return (x + 127) / 128 * 128; };
    const int tbl = m * kcount * (v / 4) * 16 * 8;
    const int xb = nt * 8 * (ks_chunks * kChunk + 16) * 2;
    const int tile = ks_chunks * m * batch_code_unit(v);  // one row tile's codes of a task
    const int codes = 2 * tile;
    const int scl = gis * 64;
    const int red = (nt == 4 ? 8 : 16) * 32 * (nt * 8 + 2) * 4;  // warps x 32 rows x padded columns
    int o = 0;
    const int off_tbl = o;
    o += up(tbl);
    const int off_x = o;
    o += up(xb);
    const int off_c0 = o;
    o += up(codes);
    const int off_c1 = o;
    o += up(codes);
    const int off_s0 = o;
    o += up(scl);
    const int off_s1 = o;
    o += up(scl);
    const int off_red = o;
    o += up(red);
    const int off_bar = o;
    o += 128;  // mbarriers of the two code/scale buffers
    if (bp) {
        bp->off_tbl = off_tbl;
        bp->off_x = off_x;
        bp->off_codes[0] = off_c0;
        bp->off_codes[1] = off_c1;
        bp->off_scl[0] = off_s0;
        bp->off_scl[1] = off_s1;
        bp->off_red = off_red;
        bp->off_bar = off_bar;
        bp->code_tile_bytes = tile;
    }
    return o;
}

int64_t batch_code_bytes(int64_t rows, int64_t cols, int v, int m) {
    const int64_t n_rt = (rows + 15) / 16;
    const int64_t n_chunks = (cols + kChunk - 1) / kChunk;
    return n_rt * n_chunks * m * (int64_t)batch_code_unit(v);
}

int64_t batch_scale_bytes(int64_t rows, int64_t groups) {
    return (rows + 31) / 32 * groups * 32 * 2;
}

cudaError_t launch_prepack_batch(const uint16_t* raw, uint8_t* out, int64_t rows, int64_t segs,
                                 int m, int v, const uint16_t* scales, int64_t groups,
                                 uint16_t* scl_out, cudaStream_t s) {
    const int64_t cols = segs * v;
    const int64_t n_chunks = (cols + kChunk - 1) / kChunk;
    const int64_t total = batch_code_bytes(rows, cols, v, m);
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    prepack_batch_kernel<<<(unsigned)blocks, 256, 0, s>>>(raw, out, total, rows, segs, m, v, n_chunks);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int64_t st = batch_scale_bytes(rows, groups) / 2;
    blocks = (st + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    prepack_batch_scales_kernel<<<(unsigned)(blocks < 1 ? 1 : blocks), 256, 0, s>>>(scales, scl_out, st,
                                                                                   rows, groups);
    return cudaGetLastError();
}

cudaError_t launch_batch_gemm(int v, int m, int nt, const BatchParams& bp, int grid, int smem,
                              cudaStream_t s, bool pdl) {
    if (v == 4 && m == 1) return launch_batch_vm<4, 1>(nt, bp, grid, smem, s, pdl);
    if (v == 4 && m == 2) return launch_batch_vm<4, 2>(nt, bp, grid, smem, s, pdl);
    if (v == 8 && m == 1) return launch_batch_vm<8, 1>(nt, bp, grid, smem, s, pdl);
    if (v == 8 && m == 2) return launch_batch_vm<8, 2>(nt, bp, grid, smem, s, pdl);
    return cudaErrorInvalidConfiguration;
}

}  // namespace cg
