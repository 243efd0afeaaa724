// How long does one thread take to ISSUE a bulk copy (cp.async.bulk global->shared)?
// Times (clock64) around expect_tx and each UBLKCP, for sources in fresh pages
// (TLB cold) and in a page just used.  nvcc -gencode arch=compute_100a,code=sm_100a -o tma_issue tma_issue.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const unsigned char* src, int64_t stride, int n, long long* out) {
    __shared__ __align__(128) unsigned char buf[16384];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x != 0) return;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    unsigned phase = 0;
    for (int i = 0; i < n; ++i) {
        const unsigned char* s = src + (int64_t)i * stride;
        long long t0 = clock64();
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(16384) : "memory");
        long long t1 = clock64();
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(buf)), "l"(s), "r"(16384), "r"(sa(&bar)) : "memory");
        long long t2 = clock64();
        asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}" ::"r"(sa(&bar)), "r"(phase) : "memory");
        phase ^= 1;
        long long t3 = clock64();
        out[i * 3 + 0] = t1 - t0;
        out[i * 3 + 1] = t2 - t1;
        out[i * 3 + 2] = t3 - t2;
    }
}

int main() {
    const int n = 16;
    unsigned char* src;
    long long* out;
    const int64_t big = 2048LL << 20;
    cudaMalloc(&src, big);
    cudaMemset(src, 1, big);
    cudaMallocManaged(&out, n * 3 * sizeof(long long));
    for (int64_t stride : {(int64_t)0, (int64_t)16384, (int64_t)(2 << 20), (int64_t)(64 << 20)}) {
        k<<<1, 32>>>(src, stride, n, out);
        cudaDeviceSynchronize();
        printf("stride %10lld: issue(expect,copy)/land cycles:", (long long)stride);
        for (int i = 0; i < n; ++i) printf(" %lld/%lld/%lld", out[3 * i], out[3 * i + 1], out[3 * i + 2]);
        printf("\n");
    }
    return 0;
}
