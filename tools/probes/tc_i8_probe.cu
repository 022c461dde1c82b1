// Probe: tcgen05.mma kind::i8 with A (u8) in TMEM (written by tcgen05.st), B (s8) in shared memory
// (K-major SWIZZLE_128B), D (s32) in TMEM.  Checks the TMEM A layout assumption
// (lane = row, 32-bit column c = k bytes 4c..4c+3) for N = 8 and N = 16 over K = 64 (2 MMAs).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/probes/tc_i8_probe tools/probes/tc_i8_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t a) {
    return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint32_t sw128_off(int r, int j) {
    return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((j ^ (r & 7)) << 4));
}

template <int N>
__global__ void probe(const uint8_t* A, const int8_t* B, int* D, int nmma) {
    __shared__ __align__(1024) uint8_t bt[2 * 1024 * 2];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, r = threadIdx.x;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(saddr(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // B: N rows x 64 bytes of K into the SW128 tile (row = 128 B, 16-B chunks swizzled)
    for (int i = threadIdx.x; i < N * 64; i += blockDim.x) {
        const int n = i / 64, k = i % 64;
        bt[sw128_off(n, k / 16) + (k % 16)] = (uint8_t)B[n * 64 + k];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tbase;
    // A row r: 64 bytes -> 16 columns
    uint32_t a[16];
    for (int c = 0; c < 16; ++c)
        a[c] = (uint32_t)A[r * 64 + 4 * c] | ((uint32_t)A[r * 64 + 4 * c + 1] << 8) |
               ((uint32_t)A[r * 64 + 4 * c + 2] << 16) | ((uint32_t)A[r * 64 + 4 * c + 3] << 24);
    const uint32_t ta = tm + ((uint32_t)(warp * 32) << 16);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
        "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]), "r"(a[8]), "r"(a[9]),
        "r"(a[10]), "r"(a[11]), "r"(a[12]), "r"(a[13]), "r"(a[14]), "r"(a[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // D s32, A u8 (0), B s8 (1), K-major both, N, M = 128
        const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
        for (int k = 0; k < nmma; ++k) {
            const uint64_t bd = desc_sw128(saddr(bt) + 32 * k);
            const uint32_t acc = k > 0;
            asm volatile(
                "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tm + 128),
                "r"(tm + 8 * k), "l"(bd), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar))
                     : "memory");
    }
    {
        asm volatile(
            "{\n .reg .pred p;\nW:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n" ::"r"(
                saddr(&bar)));
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t v[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(ta + 128));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int n = 0; n < N; ++n) D[r * N + n] = (int)v[n];
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
    }
}

template <int N>
int run(int nmma) {
    uint8_t hA[128 * 64];
    int8_t hB[16 * 64];
    int hD[128 * 16], ref[128 * 16];
    srand(N * 7 + nmma);
    for (int i = 0; i < 128 * 64; ++i) hA[i] = (uint8_t)(rand() & 0xff);
    for (int i = 0; i < 16 * 64; ++i) hB[i] = (int8_t)(rand() & 0xff);
    for (int r = 0; r < 128; ++r)
        for (int n = 0; n < N; ++n) {
            int s = 0;
            for (int k = 0; k < 32 * nmma; ++k) s += (int)hA[r * 64 + k] * (int)hB[n * 64 + k];
            ref[r * N + n] = s;
        }
    uint8_t* dA;
    int8_t* dB;
    int* dD;
    cudaMalloc(&dA, sizeof(hA));
    cudaMalloc(&dB, sizeof(hB));
    cudaMalloc(&dD, sizeof(hD));
    cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, sizeof(hD));
    probe<N><<<1, 128>>>(dA, dB, dD, nmma);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("N=%d nmma=%d: CUDA error %s\n", N, nmma, cudaGetErrorString(e));
        return 1;
    }
    cudaMemcpy(hD, dD, sizeof(int) * 128 * N, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < 128 * N; ++i) bad += hD[i] != ref[i];
    printf("N=%d nmma=%d: %d / %d mismatches (D[0]=%d ref %d, D[1]=%d ref %d)\n", N, nmma, bad, 128 * N, hD[0], ref[0],
           hD[1], ref[1]);
    return bad != 0;
}

int main() {
    int fails = 0;
    fails += run<8>(1);
    fails += run<8>(2);
    fails += run<16>(1);
    fails += run<16>(2);
    printf(fails ? "PROBE FAILED\n" : "PROBE OK\n");
    return fails;
}
