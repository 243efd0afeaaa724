// FP32 FMA throughput on one SM: FFMA (3-reg) vs FFMA2 (scalar-broadcast form, as in the
// Psumbook build), 16 warps, 8 independent chains per thread.  Cycles per warp-instruction
// per SMSP.  nvcc -gencode arch=compute_100a,code=sm_100a -o ffma_rate ffma_rate.cu
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512, 1) k_ffma(int iters, float* out, long long* cyc) {
    float a[8], c = threadIdx.x * 1e-3f, d = 1.0001f;
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = i;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], d, c);
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * 512 + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void __launch_bounds__(512, 1) k_ffma2(int iters, float* out, long long* cyc) {
    float2 a[8];
    float c = threadIdx.x * 1e-3f;
    float2 x = make_float2(1.0001f, 0.9999f);
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = make_float2(i, i + 1);
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(make_float2(c, c), x, a[i]);
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
    out[blockIdx.x * 512 + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    float* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 512 * 4);
    cudaMallocManaged(&cyc, 148 * 8);
    const int iters = 1000;
    for (int rep = 0; rep < 2; ++rep) {
        k_ffma<<<148, 512>>>(iters, out, cyc);
        cudaDeviceSynchronize();
        // 16 warps x (iters*16*8) instrs / 4 SMSP
        double per = (double)cyc[0] / (iters * 16.0 * 8.0 * 16 / 4);
        printf("FFMA : %.2f cycles per warp-instr per SMSP (%lld cycles)\n", per, cyc[0]);
        k_ffma2<<<148, 512>>>(iters, out, cyc);
        cudaDeviceSynchronize();
        per = (double)cyc[0] / (iters * 16.0 * 8.0 * 16 / 4);
        printf("FFMA2: %.2f cycles per warp-instr per SMSP (%lld cycles)\n", per, cyc[0]);
    }
    return 0;
}
