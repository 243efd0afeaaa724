// Psumbook build variants, cycles per build in isolation (diagnostics).
#include "../../paper_2512_17970_b200/csrc/cg_kernels.cu"
#include <cstdio>

namespace cg {
namespace {
__device__ __forceinline__ uint64_t ffma2(float c, uint64_t x, uint64_t a) {
    uint64_t d;
    const uint64_t cc = (uint64_t)__float_as_uint(c) | ((uint64_t)__float_as_uint(c) << 32);
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(cc), "l"(x), "l"(a));
    return d;
}

// VAR 1: packed-b64 accumulators, st.shared.v2.b64 (MOV-free?), x16 staged as now
// VAR 2: x staged as binary32 pairs (no per-use conversion)
template <int V, int M, int U, int KB, int VAR>
__device__ __forceinline__ void build_var(float* psum, const uint16_t* books16, const uint32_t* x16w,
                                          const float2* x32p, int kcount, int tid) {
    using S = FusedShape<V, M, U, KB>;
    const int lane = tid & 31, warp = tid >> 5;
    const int q = lane & 7, csub = lane >> 3, c0 = csub + 4 * warp;
    constexpr int kCPT = S::kCPT;
#pragma unroll 1
    for (int t = 0; t < M; ++t) {
        const uint16_t* bk = books16 + t * kcount * V;
        float cc[kCPT][V];
#pragma unroll
        for (int i = 0; i < kCPT; ++i) load_centroid<V>(cc[i], bk + (c0 + 4 * kWarps * i) * V);
#pragma unroll 1
        for (int uu = 0; uu < U; ++uu) {
            const int j = t * U + uu;
            uint64_t x01[V], x23[V];
            if (VAR == 2) {
                const float4* src = reinterpret_cast<const float4*>(x32p + (uu * 8 + q) * (2 * V + 2));
#pragma unroll
                for (int c = 0; c < V; ++c) {
                    const float4 w = src[c];
                    uint64_t* d = (2 * c < V) ? &x01[2 * c] : &x23[2 * c - V];
                    d[0] = (uint64_t)__float_as_uint(w.x) | ((uint64_t)__float_as_uint(w.y) << 32);
                    d[1] = (uint64_t)__float_as_uint(w.z) | ((uint64_t)__float_as_uint(w.w) << 32);
                }
            } else {
                const uint32_t* src = x16w + (uu * 8 + q) * S::kXQW;
                uint32_t w[2 * V];
#pragma unroll
                for (int i = 0; i < 2 * V; i += 4) {
                    const uint4 a = *reinterpret_cast<const uint4*>(src + i);
                    w[i] = a.x; w[i + 1] = a.y; w[i + 2] = a.z; w[i + 3] = a.w;
                }
#pragma unroll
                for (int k = 0; k < V; ++k) {
                    const float2 f01 = __half22float2(*reinterpret_cast<const __half2*>(&w[k]));
                    const float2 f23 = __half22float2(*reinterpret_cast<const __half2*>(&w[V + k]));
                    x01[k] = (uint64_t)__float_as_uint(f01.x) | ((uint64_t)__float_as_uint(f01.y) << 32);
                    x23[k] = (uint64_t)__float_as_uint(f23.x) | ((uint64_t)__float_as_uint(f23.y) << 32);
                }
            }
            float* dst = psum + (j >> 1) * S::kRegionFloats + (j & 1) * 32 + q * 4;
#pragma unroll
            for (int i = 0; i < kCPT; ++i) {
                uint64_t a01 = 0, a23 = 0;
#pragma unroll
                for (int k = 0; k < V; ++k) {
                    a01 = ffma2(cc[i][k], x01[k], a01);
                    a23 = ffma2(cc[i][k], x23[k], a23);
                }
                asm volatile("st.shared.v2.b64 [%0], {%1, %2};" ::"r"(smem_u32(dst + (c0 + 4 * kWarps * i) * 64)),
                             "l"(a01), "l"(a23) : "memory");
            }
        }
    }
}

template <int V, int M, int U, int KB, int VAR>
__global__ void __launch_bounds__(kThreads, 1) bench(int iters, unsigned long long* cyc) {
    using S = FusedShape<V, M, U, KB>;
    extern __shared__ __align__(16) unsigned char sm[];
    const uint32_t base = smem_u32(sm);
    unsigned char* al = sm + (((base + 0xffff) & ~0xffffu) - base);
    float* psum = reinterpret_cast<float*>(al);
    uint16_t* books = reinterpret_cast<uint16_t*>(al + S::kPsumBytes);
    uint16_t* x16 = books + M * S::kCodes * V;
    float2* x32p = reinterpret_cast<float2*>(x16 + S::kXBytes / 2);
    const int tid = threadIdx.x;
    for (int i = tid; i < M * S::kCodes * V; i += kThreads) books[i] = 0x3c00 + (i & 255);
    for (int i = tid; i < S::kXBytes / 2; i += kThreads) x16[i] = 0x3800 + (i & 127);
    for (int i = tid; i < U * 8 * (2 * V + 2); i += kThreads) x32p[i] = make_float2(0.5f, 0.25f);
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (VAR == 0)
            build_psumbook_smem<V, M, U, KB>(psum, books, reinterpret_cast<const uint32_t*>(x16), S::kCodes, tid);
        else
            build_var<V, M, U, KB, VAR>(psum, books, reinterpret_cast<const uint32_t*>(x16), x32p, S::kCodes, tid);
        __syncthreads();
    }
    long long t1 = clock64();
    if (tid == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int V, int M, int U, int KB, int VAR>
void run(const char* name) {
    using S = FusedShape<V, M, U, KB>;
    unsigned long long* cyc;
    cudaMalloc(&cyc, 148 * 8);
    const int smem = 65536 + S::kPsumBytes + 65536;
    cudaFuncSetAttribute(bench<V, M, U, KB, VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 2000;
    bench<V, M, U, KB, VAR><<<148, kThreads, smem>>>(iters, cyc);
    bench<V, M, U, KB, VAR><<<148, kThreads, smem>>>(iters, cyc);
    unsigned long long c[148];
    cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
    printf("%-30s var %d: %8.1f cycles/build  %s\n", name, VAR, mx / iters, cudaGetErrorString(cudaGetLastError()));
}
}  // namespace
}  // namespace cg

int main() {
    cg::run<4, 1, 2, 8, 0>("v4 m1 u2 (16K entries)");
    cg::run<4, 1, 2, 8, 1>("v4 m1 u2 (16K entries)");
    cg::run<4, 1, 2, 8, 2>("v4 m1 u2 (16K entries)");
    cg::run<4, 1, 1, 8, 0>("v4 m1 u1 (8K entries)");
    cg::run<4, 1, 1, 8, 2>("v4 m1 u1 (8K entries)");
    return 0;
}
