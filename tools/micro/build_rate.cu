// Cycles per Psumbook build (build_psumbook_smem) and per x staging, in
// isolation: 148 CTAs x 512 threads, tables in shared memory (diagnostics).
#include "../../paper_2512_17970_b200/csrc/cg_kernels.cu"
#include <cstdio>

namespace cg {
namespace {
template <int V, int M, int U, int KB>
__global__ void __launch_bounds__(kThreads, 1) build_bench(int iters, unsigned long long* cyc, int mode) {
    using S = FusedShape<V, M, U, KB>;
    extern __shared__ __align__(16) unsigned char sm[];
    const uint32_t base = smem_u32(sm);
    unsigned char* al = sm + (((base + 0xffff) & ~0xffffu) - base);
    float* psum = reinterpret_cast<float*>(al);
    uint16_t* books = reinterpret_cast<uint16_t*>(al + S::kPsumBytes);
    uint16_t* x16 = books + M * S::kCodes * V;
    uint16_t* xr = x16 + S::kXBytes / 2;
    const int tid = threadIdx.x;
    for (int i = tid; i < M * S::kCodes * V; i += kThreads) books[i] = 0x3c00 + (i & 255);
    for (int i = tid; i < S::kSliceSegs * V; i += kThreads) xr[i] = 0x3800 + (i & 127);
    __syncthreads();
    stage_x_raw<V, M, U, KB>(x16, xr, S::kSliceSegs * V, tid);
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (mode & 1) stage_x_raw<V, M, U, KB>(x16, xr, S::kSliceSegs * V, tid);
        __syncthreads();
        if (mode & 2) build_psumbook_smem<V, M, U, KB>(psum, books, reinterpret_cast<const uint32_t*>(x16), S::kCodes, tid);
        __syncthreads();
    }
    long long t1 = clock64();
    if (tid == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int V, int M, int U, int KB>
void run(const char* name, int mode) {
    using S = FusedShape<V, M, U, KB>;
    unsigned long long* cyc;
    cudaMalloc(&cyc, 148 * 8);
    const int smem = 65536 + S::kPsumBytes + 65536;
    cudaFuncSetAttribute(build_bench<V, M, U, KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 2000;
    build_bench<V, M, U, KB><<<148, kThreads, smem>>>(iters, cyc, mode);
    build_bench<V, M, U, KB><<<148, kThreads, smem>>>(iters, cyc, mode);
    unsigned long long c[148];
    cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
    const double entries = (double)M * U * 32 * S::kCodes;
    printf("%-34s mode %d: %8.1f cycles/iter  (%.2f entries/clk, %s)\n", name, mode, mx / iters,
           entries / (mx / iters), cudaGetErrorString(cudaGetLastError()));
}
}  // namespace
}  // namespace cg

int main() {
    cg::run<4, 1, 2, 8>("v4 m1 u2 (16K entries)", 0);
    cg::run<4, 1, 2, 8>("v4 m1 u2 (16K entries)", 1);
    cg::run<4, 1, 2, 8>("v4 m1 u2 (16K entries)", 2);
    cg::run<4, 1, 2, 8>("v4 m1 u2 (16K entries)", 3);
    cg::run<4, 1, 4, 8>("v4 m1 u4 (32K entries)", 2);
    cg::run<8, 2, 2, 8>("v8 m2 u2 (32K entries)", 2);
    return 0;
}
