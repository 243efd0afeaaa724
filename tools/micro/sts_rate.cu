// Shared-memory store throughput (diagnostics): STS.32 / STS.64 / STS.128,
// conflict-free, 512 threads per SM, cycles per warp-instruction per SM.
#include <cstdio>
#include <cstdint>
template <int W>
__global__ void __launch_bounds__(512, 1) k(int iters, unsigned long long* cyc, float* out) {
    extern __shared__ __align__(16) float sm[];
    const int tid = threadIdx.x;
    float a = tid * 0.5f;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const int base = ((r * 512 + tid) * W) & (32768 - 1);
            if (W == 1) sm[base] = a;
            if (W == 2) *reinterpret_cast<float2*>(sm + base) = make_float2(a, a + 1.f);
            if (W == 4) *reinterpret_cast<float4*>(sm + base) = make_float4(a, a + 1.f, a + 2.f, a + 3.f);
            a += 1.0f;
        }
    }
    long long t1 = clock64();
    __syncthreads();
    if (tid == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * 512 + tid] = sm[tid * 3 % 32768];
}
template <int W>
void run() {
    unsigned long long* cyc;
    float* out;
    cudaMalloc(&cyc, 148 * 8);
    cudaMalloc(&out, 148 * 512 * 4);
    cudaFuncSetAttribute(k<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    const int iters = 2000;
    k<W><<<148, 512, 131072>>>(iters, cyc, out);
    k<W><<<148, 512, 131072>>>(iters, cyc, out);
    unsigned long long c[148];
    cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
    const double warp_instr = 16.0 * 16 * iters;  // per SM
    printf("STS.%d: %.3f cycles per warp-instruction per SM (%.1f B/clk)  %s\n", 32 * W, mx / warp_instr,
           warp_instr * 32 * 4 * W / mx, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    run<1>();
    run<2>();
    run<4>();
    return 0;
}
