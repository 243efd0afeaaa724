// Psumbook build mappings compared in isolation (diagnostics): cycles per build.
//   v0: the kernel's build_psumbook_smem (4 codes x 4 lanes per thread, all warps per sub-table)
//   v1: warp halves take alternate sub-tables, 8 codes x 4 lanes per thread, centroids hoisted
#include "../../paper_2512_17970_b200/csrc/cg_kernels.cu"
#include <cstdio>

namespace cg {
namespace {
template <int V, int M, int U, int KB>
__device__ __forceinline__ void build_v1(float* psum, const uint16_t* books16, const float* xs,
                                         int kcount, int tid) {
    using S = FusedShape<V, M, U, KB>;
    const int lane = tid & 31, warp = tid >> 5;
    const int q = lane & 7, csub = lane >> 3;
    const int c0 = csub + 4 * warp;
    constexpr int kCPT = S::kCPT;
#pragma unroll 1
    for (int t = 0; t < M; ++t) {
        const uint16_t* bk = books16 + t * kcount * V;
        float cc[kCPT][V];
#pragma unroll
        for (int i = 0; i < kCPT; ++i) load_centroid<V>(cc[i], bk + (c0 + 4 * kWarps * i) * V);
#pragma unroll 2
        for (int uu = 0; uu < U; ++uu) {
            const int j = t * U + uu;
            float2 x01[V], x23[V];
            const float4* src = reinterpret_cast<const float4*>(xs + (uu * 8 + q) * S::kXQF);
#pragma unroll
            for (int c = 0; c < V; ++c) {
                const float4 w = src[c];
                float2* d = (2 * c < V) ? &x01[2 * c] : &x23[2 * c - V];
                d[0] = make_float2(w.x, w.y);
                d[1] = make_float2(w.z, w.w);
            }
            float* dst = psum + (j >> 1) * S::kRegionFloats + (j & 1) * 32 + q * 4;
#pragma unroll
            for (int i = 0; i < kCPT; ++i) psum_entries<V>(dst + (c0 + 4 * kWarps * i) * 64, cc[i], x01, x23);
        }
    }
}

template <int V, int M, int U, int KB, int VAR>
__global__ void __launch_bounds__(kThreads, 1) bench(int iters, unsigned long long* cyc, float* chk) {
    using S = FusedShape<V, M, U, KB>;
    extern __shared__ __align__(16) unsigned char sm[];
    const uint32_t base = smem_u32(sm);
    unsigned char* al = sm + (((base + 0xffff) & ~0xffffu) - base);
    float* psum = reinterpret_cast<float*>(al);
    uint16_t* books = reinterpret_cast<uint16_t*>(al + S::kPsumBytes);
    float* xs = reinterpret_cast<float*>(books + M * S::kCodes * V);
    const int tid = threadIdx.x;
    for (int i = tid; i < M * S::kCodes * V; i += kThreads) books[i] = 0x3c00 + (i & 255);
    for (int i = tid; i < S::kXFloats; i += kThreads) xs[i] = 0.5f + (i & 7);
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (VAR == 0) build_psumbook_smem<V, M, U, KB>(psum, books, xs, S::kCodes, tid);
        else build_v1<V, M, U, KB>(psum, books, xs, S::kCodes, tid);
        __syncthreads();
    }
    long long t1 = clock64();
    if (tid == 0) cyc[blockIdx.x] = t1 - t0;
    if (blockIdx.x == 0)
        for (int i = tid; i < S::kPsumFloats; i += kThreads) chk[i] = psum[i];
}

template <int V, int M, int U, int KB, int VAR>
void run(const char* name, float* host, const float* ref) {
    using S = FusedShape<V, M, U, KB>;
    unsigned long long* cyc;
    float* chk;
    cudaMalloc(&cyc, 148 * 8);
    cudaMalloc(&chk, S::kPsumBytes);
    const int smem = 65536 + S::kPsumBytes + 32768;
    cudaFuncSetAttribute(bench<V, M, U, KB, VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 1000;
    bench<V, M, U, KB, VAR><<<148, kThreads, smem>>>(iters, cyc, chk);
    bench<V, M, U, KB, VAR><<<148, kThreads, smem>>>(iters, cyc, chk);
    unsigned long long c[148];
    cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
    cudaMemcpy(host, chk, S::kPsumBytes, cudaMemcpyDeviceToHost);
    long diff = 0;
    if (ref)
        for (int i = 0; i < S::kPsumFloats; ++i) diff += host[i] != ref[i];
    double mx = 0;
    for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
    printf("%-26s var %d: %8.1f cycles/build  diff-vs-v0 %ld  %s\n", name, VAR, mx / iters, diff,
           cudaGetErrorString(cudaGetLastError()));
}
}  // namespace
}  // namespace cg

static float g_a[65536], g_b[65536];
int main() {
    cg::run<4, 1, 4, 8, 0>("v4 m1 u4 (32K entries)", g_a, nullptr);
    cg::run<4, 1, 4, 8, 1>("v4 m1 u4 (32K entries)", g_b, g_a);
    cg::run<4, 1, 2, 8, 0>("v4 m1 u2 (16K entries)", g_a, nullptr);
    cg::run<4, 1, 2, 8, 1>("v4 m1 u2 (16K entries)", g_b, g_a);
    return 0;
}
