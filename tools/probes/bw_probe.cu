// Micro-probe: HBM streaming rate of (a) cp.async.bulk issued by one thread per CTA into a
// shared-memory ring (the chain kernel's producer pattern) vs (b) plain LDG.128 by all warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bw_probe bw_probe.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int SLOTS, int CHUNK, int PRODUCERS>
__global__ void __launch_bounds__(544, 1) bulk_ring(const uint8_t* src, size_t bytes_per_cta, unsigned long long* sink) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t* full = (uint64_t*)(sm + SLOTS * CHUNK);
    uint64_t* empty = full + SLOTS;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int i = 0; i < SLOTS; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[i])), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[i])), "r"(1));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint8_t* base = src + (size_t)blockIdx.x * bytes_per_cta;
    const int n = (int)(bytes_per_cta / CHUNK);
    if (warp == 16) {
        if (lane < PRODUCERS) {
            for (int u = lane; u < n; u += PRODUCERS) {
                const int slot = u % SLOTS;
                const unsigned ph = ((u / SLOTS) & 1) ^ 1;
                asm volatile("{ .reg .pred p; W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W%=; }" ::"r"(su32(&empty[slot])), "r"(ph) : "memory");
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[slot])), "r"(CHUNK) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(sm + slot * CHUNK)), "l"(base + (size_t)u * CHUNK), "r"(CHUNK), "r"(su32(&full[slot])) : "memory");
            }
        }
        return;
    }
    unsigned long long acc = 0;
    if (warp != 0) return;  // one consumer warp, strictly in order (no phase aliasing)
    for (int u = 0; u < n; ++u) {
        const int slot = u % SLOTS;
        const unsigned ph = (u / SLOTS) & 1;
        asm volatile("{ .reg .pred p; W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W%=; }" ::"r"(su32(&full[slot])), "r"(ph) : "memory");
        acc += ((const uint32_t*)(sm + slot * CHUNK))[lane];
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[slot])) : "memory");
    }
    if (acc == 0x123456789ull) sink[0] = acc;
}

__global__ void __launch_bounds__(512) ldg_stream(const uint4* src, size_t n16, unsigned long long* sink) {
    unsigned acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n16; i += 4 * stride) {
        uint4 a = __ldcs(src + i), b = __ldcs(src + i + stride), c = __ldcs(src + i + 2 * stride), d = __ldcs(src + i + 3 * stride);
        acc ^= a.x ^ b.y ^ c.z ^ d.w;
    }
    if (acc == 0x12345u) sink[0] = acc;
}

template <int SLOTS, int CHUNK, int PRODUCERS>
void run_bulk(const uint8_t* d, size_t total, int sms, unsigned long long* sink) {
    const size_t per = (total / sms) / CHUNK * CHUNK;
    const int smem = SLOTS * CHUNK + 2 * SLOTS * 8;
    cudaFuncSetAttribute(bulk_ring<SLOTS, CHUNK, PRODUCERS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int w = 0; w < 2; ++w) bulk_ring<SLOTS, CHUNK, PRODUCERS><<<sms, 544, smem>>>(d, per, sink);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) bulk_ring<SLOTS, CHUNK, PRODUCERS><<<sms, 544, smem>>>(d, per, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("bulk ring slots=%2d chunk=%6d producers=%d : %7.1f GB/s  (err=%s)\n", SLOTS, CHUNK, PRODUCERS,
           5.0 * per * sms / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t total = (size_t)4 << 30;
    uint8_t* d; cudaMalloc(&d, total); cudaMemset(d, 1, total);
    unsigned long long* sink; cudaMalloc(&sink, 8);
    run_bulk<11, 16384, 1>(d, total, sms, sink);
    run_bulk<11, 16384, 4>(d, total, sms, sink);
    run_bulk<22, 8192, 1>(d, total, sms, sink);
    run_bulk<22, 8192, 8>(d, total, sms, sink);
    run_bulk<44, 4096, 8>(d, total, sms, sink);
    run_bulk<6, 32768, 1>(d, total, sms, sink);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int w = 0; w < 2; ++w) ldg_stream<<<sms * 4, 512>>>((const uint4*)d, total / 16, sink);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) ldg_stream<<<sms * 4, 512>>>((const uint4*)d, total / 16, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("ldg stream: %7.1f GB/s\n", 5.0 * total / (ms * 1e-3) / 1e9);
    return 0;
}
