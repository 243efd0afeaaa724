// Micro-benchmarks of the shared-memory rates the fused kernel depends on
// (diagnostics, not product code): conflict-free LDS.32 lookups addressed by
// PRMT from random code bytes held in registers, the warp transpose-reduction
// shuffles, and STS.128 table stores.  One CTA of 512 threads per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ float lds_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(int iters, float* out, unsigned long long* cyc) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int tid = threadIdx.x, lane = tid & 31;
    uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
    base = (base + 0xffff) & ~0xffffu;
    float* tab = reinterpret_cast<float*>(sm + (base - (uint32_t)__cvta_generic_to_shared(sm)));
    for (int i = tid; i < 32768; i += 512) tab[i] = (float)(i & 1023);
    __syncthreads();
    const uint32_t lb = ((uint32_t)lane << 2) | ((base >> 16) << 8);
    uint32_t w0 = 0x9e3779b9u * (tid + 1), w1 = w0 * 747796405u + 1, w2 = w1 * 747796405u + 1,
             w3 = w2 * 747796405u + 1;
    float acc[16];
    for (int i = 0; i < 16; ++i) acc[i] = 0.f;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0 || MODE == 1) {
            // 64 lookups per iteration (16 words x 4 bytes), PRMT + LDS each
#pragma unroll
            for (int wdx = 0; wdx < 4; ++wdx) {
                const uint32_t w = wdx == 0 ? w0 : wdx == 1 ? w1 : wdx == 2 ? w2 : w3;
#pragma unroll
                for (int r = 0; r < 4; ++r) {
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        const uint32_t a = __byte_perm(w ^ (r * 0x01010101u), lb, 0x6504u | (b << 4));
                        acc[r * 4 + b] += lds_f32(a + ((r & 1) ? 65536u : 0u));
                    }
                }
            }
            if (MODE == 1) {  // + 16 shuffles (transpose-reduction)
#pragma unroll
                for (int i = 0; i < 16; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[(i + 8) & 15], 1 << (i & 3));
            }
            w0 = w0 * 1664525u + 1013904223u;
            w1 = w1 * 1664525u + 1013904223u;
            w2 = w2 * 1664525u + 1013904223u;
            w3 = w3 * 1664525u + 1013904223u;
        } else if (MODE == 2) {  // STS.128 stores, conflict-free rows (16 per iteration)
            const int q = lane & 7, csub = lane >> 3, warp = tid >> 5;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int c = (csub + 4 * warp + 64 * (i & 3)) & 255;
                float4* d = reinterpret_cast<float4*>(tab + (i >> 2) * 16384 / 2 + c * 64 + (i & 1) * 32 + q * 4);
                *d = make_float4(acc[i], acc[(i + 1) & 15], acc[(i + 2) & 15], (float)it);
                acc[i] += 1.0f;
            }
        }
    }
    long long t1 = clock64();
    float s = 0.f;
    for (int i = 0; i < 16; ++i) s += acc[i];
    out[blockIdx.x * 512 + tid] = s;
    if (tid == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
}

template <int MODE>
void run(const char* name, int iters, double per_iter_warp) {
    float* out;
    unsigned long long* cyc;
    cudaMalloc(&out, 148 * 512 * 4);
    cudaMalloc(&cyc, 148 * 8);
    const int smem = 200 * 1024;
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<MODE><<<148, 512, smem>>>(iters, out, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MODE><<<148, 512, smem>>>(iters, out, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long c[148];
    cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
    double cmax = 0;
    for (int i = 0; i < 148; ++i) cmax = c[i] > cmax ? c[i] : cmax;
    const double ops = per_iter_warp * 16.0 * iters;  // per SM
    printf("%-28s %8.3f ms  %10.0f cyc/SM  %.3f warp-ops/clk/SM  (%.2f GHz eff)\n", name, ms, cmax,
           ops / cmax, cmax / (ms * 1e6));
    cudaError_t e = cudaGetLastError();
    if (e) printf("error %s\n", cudaGetErrorString(e));
}

int main() {
    run<0>("lookup LDS.32 (per LDS)", 20000, 64);
    run<1>("lookup+16 SHFL (per LDS)", 20000, 64);
    run<2>("STS.128 (per STS)", 20000, 16);
    return 0;
}
