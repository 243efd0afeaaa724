// Latency of system- vs gpu-scope fences on B200 (one thread per CTA, full grid),
// idle and right after a burst of bulk L2 prefetches / global stores.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__global__ void k(unsigned long long* out, float* buf, int mode) {
    if (threadIdx.x) return;
    float* mine = buf + blockIdx.x * 65536;
    if (mode & 4)  // a burst of stores before the fences
        for (int i = 0; i < 256; ++i) mine[i * 32] = (float)i;
    if (mode & 8)  // bulk L2 prefetches in flight
        for (int i = 0; i < 8; ++i)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], 32768;" ::"l"(mine + i * 8192) : "memory");
    unsigned long long t0 = gt();
    for (int i = 0; i < 16; ++i) {
        if (mode & 1) asm volatile("fence.acq_rel.sys;" ::: "memory");
        else asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    unsigned long long t1 = gt();
    out[blockIdx.x] = (t1 - t0) / 16;
}
int main() {
    unsigned long long* out; float* buf;
    cudaMalloc(&out, 148 * 8); cudaMalloc(&buf, 148ull * 65536 * 4);
    unsigned long long h[148];
    const char* names[] = {"gpu idle", "sys idle", "", "", "gpu after stores", "sys after stores", "", "",
                           "gpu after prefetch", "sys after prefetch"};
    for (int mode : {0, 1, 4, 5, 8, 9}) {
        for (int rep = 0; rep < 3; ++rep) k<<<148, 32>>>(out, buf, mode);
        cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
        unsigned long long s = 0, mx = 0;
        for (int i = 0; i < 148; ++i) { s += h[i]; mx = h[i] > mx ? h[i] : mx; }
        printf("%-20s mean %6.0f ns per fence (max %llu)\n", names[mode], s / 148.0, mx);
    }
    return 0;
}
