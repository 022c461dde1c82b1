// Probe: cost of cp.async.bulk (global -> shared, UBLKCP) per request vs size.  One thread per CTA
// issues K copies of S bytes (L2-resident source) on one mbarrier and waits; reports issue cycles
// per copy and total cycles per copy.  Grid 1 and 148.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/probes/bulk_issue_probe tools/probes/bulk_issue_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const uint8_t* src, int S, int K, int reps, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    long long ti = 0, tt = 0;
    for (int r = 0; r < reps; ++r) {
        const long long t0 = clock64();
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(&bar)), "r"(S * K) : "memory");
        for (int k = 0; k < K; ++k) {
            const uint8_t* g = src + ((size_t)(blockIdx.x * K + k) * S) % (64u << 20);
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             saddr(sm + k * S)),
                         "l"(g), "r"(S), "r"(saddr(&bar))
                         : "memory");
        }
        const long long t1 = clock64();
        asm volatile("{\n .reg .pred p;\nW:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
                         saddr(&bar)), "r"(r & 1));
        const long long t2 = clock64();
        if (r > 0) {
            ti += t1 - t0;
            tt += t2 - t0;
        }
    }
    if (blockIdx.x == 0) {
        out[0] = ti;
        out[1] = tt;
    }
}

int main() {
    uint8_t* src;
    cudaMalloc(&src, 64u << 20);
    cudaMemset(src, 1, 64u << 20);
    long long* d;
    cudaMalloc(&d, 64);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int sizes[] = {256, 2048, 8192, 16384};
    for (int grid : {1, 148})
        for (int S : sizes) {
            const int K = S >= 16384 ? 12 : 16;
            const int reps = 21;
            probe<<<grid, 32, K * S>>>(src, S, K, reps, d);
            probe<<<grid, 32, K * S>>>(src, S, K, reps, d);
            cudaError_t e = cudaDeviceSynchronize();
            long long h[2];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) {
                printf("err %s\n", cudaGetErrorString(e));
                return 1;
            }
            const double n = (double)K * (reps - 1);
            printf("grid %3d S=%6d K=%2d: issue %.1f cyc/copy, issue+land %.1f cyc/copy (%.1f B/cyc/SM)\n", grid, S, K,
                   h[0] / n, h[1] / n, S / (h[1] / n));
        }
    return 0;
}
