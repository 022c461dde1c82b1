// Probe: tcgen05.mma issue rate of kind::i8 (K = 32) vs kind::f16 (K = 16) at M = 128 for N = 64 .. 256,
// A and B from SWIZZLE_128B shared memory, one issuing thread per SM (148 CTAs), back-to-back MMAs into one
// TMEM accumulator.  The large-M MMQ question: does kind::i8 deliver more useful MACs than kind::f16 when
// the activations need two s8 limbs (two i8 MMAs per f16-equivalent product)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/probes/tc_kind_probe tools/probes/tc_kind_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t a) {
    return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

template <int N, bool I8>
__global__ void rate(int R, long long* out) {
    extern __shared__ __align__(1024) uint8_t dsm[];
    uint8_t* bt = dsm;               // 32 KB: B, N <= 256 rows x 128 B
    uint8_t* at = dsm + 32 * 1024;   // 16 KB: A, 128 rows x 128 B
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 32 * 1024; i += blockDim.x) bt[i] = (uint8_t)(i & 0x3f);
    for (int i = threadIdx.x; i < 16 * 1024; i += blockDim.x) at[i] = (uint8_t)((i * 7) & 0x3f);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(saddr(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tbase;
    if (threadIdx.x == 0) {
        // i8: D s32, A u8, B s8;  f16: D f32, A f16, B f16;  K-major A and B; N >> 3 at bit 17, M >> 4 at 24
        const uint32_t idesc = (I8 ? ((2u << 4) | (0u << 7) | (1u << 10)) : (1u << 4)) | ((uint32_t)(N >> 3) << 17) |
                               ((128u >> 4) << 24);
        const long long t0 = clock64();
        for (int k = 0; k < R; ++k) {
            const uint64_t ad = desc_sw128(saddr(at) + 32 * (k & 3));
            const uint64_t bd = desc_sw128(saddr(bt) + 32 * (k & 3));
            const uint32_t acc = k > 0;
            if (I8)
                asm volatile(
                    "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                    " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm),
                    "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
            else
                asm volatile(
                    "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                    " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm),
                    "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar))
                     : "memory");
        asm volatile(
            "{\n .reg .pred p;\nW:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n" ::"r"(
                saddr(&bar)));
        const long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
    }
}

template <int N, bool I8>
void go(long long* d) {
    const int R = 8192;
    cudaFuncSetAttribute(rate<N, I8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024 + 1024);
    rate<N, I8><<<148, 128, 48 * 1024 + 1024>>>(R, d);
    rate<N, I8><<<148, 128, 48 * 1024 + 1024>>>(R, d);
    const cudaError_t e = cudaDeviceSynchronize();
    long long h = 0;
    cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
        printf("err %s\n", cudaGetErrorString(e));
        return;
    }
    const int K = I8 ? 32 : 16;
    const double macs = 128.0 * N * K * R / h;
    printf("kind::%-3s M=128 N=%3d K=%2d: %6.1f cycles/MMA  %6.0f MACs/clk/SM  (%.0f TOPS at 1.965 GHz x 148 SMs)\n",
           I8 ? "i8" : "f16", N, K, (double)h / R, macs, 2.0 * macs * 148 * 1.965e9 / 1e12);
}

int main() {
    long long* d;
    cudaMalloc(&d, 64);
    go<64, true>(d);
    go<128, true>(d);
    go<256, true>(d);
    go<64, false>(d);
    go<128, false>(d);
    go<256, false>(d);
    return 0;
}
