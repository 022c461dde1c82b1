// Probe: issue rate of tcgen05.mma kind::i8 (M=128, K=32) with A from TMEM vs shared memory for
// several N, and tcgen05.st 32x32b.x64 throughput.  One CTA per SM; cycles from clock64.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/probes/tc_rate_probe tools/probes/tc_rate_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t a) {
    return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

template <int N, bool ATMEM>
__global__ void rate(int R, long long* out) {
    __shared__ __align__(1024) uint8_t bt[16 * 1024];
    __shared__ __align__(1024) uint8_t at[16 * 1024];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 16 * 1024; i += blockDim.x) bt[i] = (uint8_t)i;
    for (int i = threadIdx.x; i < 16 * 1024; i += blockDim.x) at[i] = (uint8_t)(i * 7);
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
    long long t0 = 0, t1 = 0;
    if (threadIdx.x == 0) {
        const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
        t0 = clock64();
        for (int k = 0; k < R; ++k) {
            const uint64_t bd = desc_sw128(saddr(bt) + 32 * (k & 3));
            const uint32_t acc = k > 0;
            if (ATMEM) {
                asm volatile(
                    "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                    " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tm + 256),
                    "r"(tm + 8 * (k & 31)), "l"(bd), "r"(idesc), "r"(acc));
            } else {
                const uint64_t ad = desc_sw128(saddr(at) + 32 * (k & 3));
                asm volatile(
                    "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                    " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm + 256),
                    "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar))
                     : "memory");
        asm volatile(
            "{\n .reg .pred p;\nW:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n" ::"r"(
                saddr(&bar)));
        t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
    }
    __syncthreads();
    // tcgen05.st x64 throughput: 4 warps, R stores each
    {
        uint32_t a[64];
        for (int i = 0; i < 64; ++i) a[i] = threadIdx.x * i;
        const uint32_t ta = tm + ((uint32_t)(warp * 32) << 16);
        long long s0 = clock64();
        for (int k = 0; k < R / 8; ++k) {
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
                "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,"
                "%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,"
                "%61,%62,%63,%64};" ::"r"(ta + 64 * (k & 3)),
                "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]),
                "r"(a[8]), "r"(a[9]), "r"(a[10]), "r"(a[11]), "r"(a[12]), "r"(a[13]), "r"(a[14]), "r"(a[15]),
                "r"(a[16]), "r"(a[17]), "r"(a[18]), "r"(a[19]), "r"(a[20]), "r"(a[21]), "r"(a[22]), "r"(a[23]),
                "r"(a[24]), "r"(a[25]), "r"(a[26]), "r"(a[27]), "r"(a[28]), "r"(a[29]), "r"(a[30]), "r"(a[31]),
                "r"(a[32]), "r"(a[33]), "r"(a[34]), "r"(a[35]), "r"(a[36]), "r"(a[37]), "r"(a[38]), "r"(a[39]),
                "r"(a[40]), "r"(a[41]), "r"(a[42]), "r"(a[43]), "r"(a[44]), "r"(a[45]), "r"(a[46]), "r"(a[47]),
                "r"(a[48]), "r"(a[49]), "r"(a[50]), "r"(a[51]), "r"(a[52]), "r"(a[53]), "r"(a[54]), "r"(a[55]),
                "r"(a[56]), "r"(a[57]), "r"(a[58]), "r"(a[59]), "r"(a[60]), "r"(a[61]), "r"(a[62]), "r"(a[63])
                : "memory");
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            a[k & 63] += 1;
        }
        long long s1 = clock64();
        if (blockIdx.x == 0 && threadIdx.x == 0) out[1] = s1 - s0;
        // latency of one MMA round trip (issue 8, commit, wait) repeated
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
        long long r0 = clock64();
        for (int it = 0; it < 64; ++it) {
            for (int k = 0; k < 8; ++k) {
                const uint64_t bd = desc_sw128(saddr(bt) + 32 * (k & 3));
                const uint32_t acc = k > 0;
                asm volatile(
                    "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                    " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tm + 256),
                    "r"(tm + 8 * k), "l"(bd), "r"(idesc), "r"(acc));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             saddr(&bar))
                         : "memory");
            const unsigned ph = (unsigned)(it + 1) & 1u;
            asm volatile(
                "{\n .reg .pred p;\nW2:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W2;\n}\n" ::"r"(
                    saddr(&bar)), "r"(ph));
        }
        long long r1 = clock64();
        if (blockIdx.x == 0) out[2] = r1 - r0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
    }
}

template <int N, bool AT>
void go(long long* d) {
    const int R = 4096;
    rate<N, AT><<<148, 128>>>(R, d);
    rate<N, AT><<<148, 128>>>(R, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[3];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return; }
    printf("N=%3d A=%s: %.1f cycles/MMA (%.0f MACs/clk/SM); tcgen05.st x64+wait: %.1f cycles; 8-MMA+commit round trip %.0f cycles\n",
           N, AT ? "tmem" : "smem", (double)h[0] / R, 128.0 * N * 32 * R / h[0], (double)h[1] / (R / 8), (double)h[2] / 64);
}

int main() {
    long long* d;
    cudaMalloc(&d, 64);
    go<16, true>(d);
    go<32, true>(d);
    go<64, true>(d);
    go<128, true>(d);

    go<32, false>(d);
    go<128, false>(d);

    return 0;
}
