// Psumbook build in isolation (the product's build_psumbook_smem, v4 m1 u4: 32K
// entries), plus variants that drop the table stores or the FMAs, to find what bounds
// it.  148 CTAs x 512 threads.  nvcc -gencode arch=compute_100a,code=sm_100a -I. ...
#include "../../paper_2512_17970_b200/csrc/cg_kernels.cu"
#include <cstdio>

namespace cg {
namespace {
template <int V, int M, int U, int KB, int MODE>
__global__ void __launch_bounds__(kThreads, 1) bench_k(int iters, unsigned long long* cyc, float* sink) {
    using S = FusedShape<V, M, U, KB>;
    extern __shared__ __align__(16) unsigned char sm[];
    const uint32_t base = smem_u32(sm);
    unsigned char* al = sm + (((base + 0xffff) & ~0xffffu) - base);
    float* psum = reinterpret_cast<float*>(al);
    // the small pieces below the 64 KB-aligned table (the dynamic area starts ~1 KB in)
    uint16_t* books = reinterpret_cast<uint16_t*>(sm);
    float* xs = reinterpret_cast<float*>(books + M * S::kCodes * V + 64);
    uint16_t* xr = reinterpret_cast<uint16_t*>(xs + S::kXFloats + 64);
    const int tid = threadIdx.x;
    for (int i = tid; i < M * S::kCodes * V; i += kThreads) books[i] = 0x3c00 + (i & 255);
    for (int i = tid; i < S::kSliceSegs * V; i += kThreads) xr[i] = 0x3800 + (i & 127);
    __syncthreads();
    stage_x_raw<V, M, U, KB>(xs, xr, S::kSliceSegs * V, tid);
    __syncthreads();
    float acc = 0.f;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) build_psumbook_smem<V, M, U, KB>(psum, books, xs, S::kCodes, tid);
        if (MODE == 1) {  // stores only: same STS.128 pattern, constant data
            const int lane = tid & 31, warp = tid >> 5, q = lane & 7, csub = lane >> 3;
            for (int uu = 0; uu < U; ++uu) {
                float* dst = psum + (uu >> 1) * S::kRegionFloats + (uu & 1) * 32 + q * 4;
#pragma unroll
                for (int i = 0; i < S::kCPT; ++i) {
                    const int c = csub + 4 * warp + 64 * i;
                    *reinterpret_cast<float4*>(dst + c * 64) = make_float4(acc, acc, acc, it);
                }
            }
        }
        if (MODE == 2) {  // FFMA2 chains only (same operands, results folded into acc)
            const int lane = tid & 31, q = lane & 7;
            float cc[S::kCPT][V];
#pragma unroll
            for (int i = 0; i < S::kCPT; ++i)
#pragma unroll
                for (int k = 0; k < V; ++k) cc[i][k] = 1.0f + 0.001f * (i * V + k + it);
            for (int uu = 0; uu < U; ++uu) {
                float2 x01[V], x23[V];
                const float4* src = reinterpret_cast<const float4*>(xs + (uu * 8 + q) * S::kXQF);
#pragma unroll
                for (int c = 0; c < V; ++c) {
                    const float4 w = src[c];
                    float2* d = (2 * c < V) ? &x01[2 * c] : &x23[2 * c - V];
                    d[0] = make_float2(w.x, w.y);
                    d[1] = make_float2(w.z, w.w);
                }
                float2 a01[S::kCPT], a23[S::kCPT];
#pragma unroll
                for (int k = 0; k < V; ++k)
#pragma unroll
                    for (int i = 0; i < S::kCPT; ++i) {
                        const float2 cb = make_float2(cc[i][k], cc[i][k]);
                        a01[i] = k == 0 ? __ffma2_rn(cb, x01[0], make_float2(0.f, 0.f)) : __ffma2_rn(cb, x01[k], a01[i]);
                        a23[i] = k == 0 ? __ffma2_rn(cb, x23[0], make_float2(0.f, 0.f)) : __ffma2_rn(cb, x23[k], a23[i]);
                    }
#pragma unroll
                for (int i = 0; i < S::kCPT; ++i) acc += a01[i].x + a01[i].y * a23[i].x - a23[i].y;
            }
        }
        __syncthreads();
    }
    long long t1 = clock64();
    if (tid == 0) cyc[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * kThreads + tid] = psum[tid * 7 % 4096] + acc;
}

template <int V, int M, int U, int KB, int MODE>
void run(const char* name) {
    using S = FusedShape<V, M, U, KB>;
    unsigned long long* cyc;
    float* sink;
    cudaMalloc(&cyc, 148 * 8);
    cudaMalloc(&sink, 148 * kThreads * 4);
    const int smem = 65536 - 1024 + S::kPsumBytes;
    cudaFuncSetAttribute(bench_k<V, M, U, KB, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 1000;
    bench_k<V, M, U, KB, MODE><<<148, kThreads, smem>>>(iters, cyc, sink);
    bench_k<V, M, U, KB, MODE><<<148, kThreads, smem>>>(iters, cyc, sink);
    unsigned long long c[148];
    cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
    printf("%-30s: %8.1f cycles per build (%s)\n", name, mx / iters, cudaGetErrorString(cudaGetLastError()));
}
}  // namespace
}  // namespace cg

int main() {
    cg::run<4, 1, 4, 8, 0>("v4 m1 u4 product build");
    cg::run<4, 1, 4, 8, 1>("v4 m1 u4 stores only");
    cg::run<4, 1, 4, 8, 2>("v4 m1 u4 FFMA2 only");
    cg::run<4, 1, 2, 8, 0>("v4 m1 u2 product build");
    cg::run<8, 2, 2, 8, 0>("v8 m2 u2 product build");
    return 0;
}
