// Probe: issue rate of tcgen05.mma kind::f16 (K = 16) for cta_group::1 (M = 128) and cta_group::2
// (M = 256 over a CTA pair), N in {64, 128, 256}, A from shared memory (SS) or from TMEM (TS).
// One cluster of 2 CTAs per TPC (74 clusters); the leader's lane 0 issues R MMAs back to back.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/probes/tc_f16_pair_probe tools/probes/tc_f16_pair_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t a) {
    return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void csync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int CG, int N, bool ATMEM, int COMMIT = 0, bool ST = false, bool LD = false, bool I8 = false>
__global__ void __cluster_dims__(2, 1, 1) rate(int R, long long* out) {
    extern __shared__ __align__(1024) uint8_t dyn[];
    uint8_t* bt = dyn;              // 32 KB: B tile (N/CG rows x 128 B per k-atom, reused)
    uint8_t* at = dyn + 32 * 1024;  // 16 KB: A tile
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar, bar2;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 48 * 1024; i += blockDim.x) dyn[i] = (uint8_t)(i * 13 >> 3) & 0x3b;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1000000;" ::"r"(saddr(&bar2)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        if (CG == 2) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(saddr(&tbase)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(saddr(&tbase)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    csync();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tbase;
    const bool issuer = threadIdx.x == 0 && (CG == 1 || rank == 0);
    if (issuer) {
        const uint32_t idesc = I8 ? ((2u << 4) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)((128 * CG) >> 4) << 24))
                                  : ((1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)((128 * CG) >> 4) << 24));
        const long long t0 = clock64();
        for (int k = 0; k < R; ++k) {
            const uint64_t bd = desc_sw128(saddr(bt) + 32 * (k & 3));
            const uint32_t acc = k > 0;
            if (ATMEM) {
                if (CG == 2)
                    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                                 " tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tm),
                                 "r"(tm + 256 + 8 * (k & 31)), "l"(bd), "r"(idesc), "r"(acc));
                else if (I8)
                    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                                 " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tm),
                                 "r"(tm + 256 + 8 * (k & 31)), "l"(bd), "r"(idesc), "r"(acc));
                else
                    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                                 " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tm),
                                 "r"(tm + 256 + 8 * (k & 31)), "l"(bd), "r"(idesc), "r"(acc));
            } else {
                const uint64_t ad = desc_sw128(saddr(at) + 32 * (k & 3));
                if (CG == 2)
                    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                                 " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm),
                                 "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
                else
                    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                                 " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm),
                                 "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
            }
            if (COMMIT && (k % COMMIT) == COMMIT - 1) {
                if (CG == 2)
                    asm volatile(
                        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                            saddr(&bar2)), "h"((uint16_t)3) : "memory");
                else
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar2))
                                 : "memory");
            }
        }
        if (CG == 2)
            asm volatile(
                "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                    saddr(&bar)), "h"((uint16_t)3) : "memory");
        else
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar))
                         : "memory");
        asm volatile("{\n .reg .pred p;\nW:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n" ::"r"(
            saddr(&bar)));
        const long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
    }
    if (LD && warp >= 4) {  // concurrent D traffic: tcgen05.ld.32x32b.x32 + wait in a loop (epilogue-like)
        const uint32_t td = tm + ((uint32_t)((warp & 3) * 32) << 16) + 128;
        uint32_t sink = 0;
        for (int k = 0; k < R / 4; ++k) {
            uint32_t v[8];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                         : "r"(td + 8 * (k & 7)));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            sink += v[0] ^ v[7];
        }
        if (sink == 0x12345) out[7] = sink;
    }
    if (ST && warp >= 4) {  // concurrent A traffic: one tcgen05.st.32x32b.x32 + wait per 4 MMAs
        uint32_t a[32];
        for (int i = 0; i < 32; ++i) a[i] = 0x3c003c00u;
        const uint32_t ta = tm + ((uint32_t)((warp & 3) * 32) << 16) + 256;
        for (int k = 0; k < R / 4; ++k) {
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
                "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta + 32 * (k & 7)),
                "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]),
                "r"(a[8]), "r"(a[9]), "r"(a[10]), "r"(a[11]), "r"(a[12]), "r"(a[13]), "r"(a[14]), "r"(a[15]),
                "r"(a[16]), "r"(a[17]), "r"(a[18]), "r"(a[19]), "r"(a[20]), "r"(a[21]), "r"(a[22]), "r"(a[23]),
                "r"(a[24]), "r"(a[25]), "r"(a[26]), "r"(a[27]), "r"(a[28]), "r"(a[29]), "r"(a[30]), "r"(a[31])
                : "memory");
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            long long w0 = clock64();
            while (clock64() - w0 < 200) {}
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    csync();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (CG == 2)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm));
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
    }
}

template <int CG, int N, bool AT, int COMMIT = 0, bool ST = false, bool LD = false, bool I8 = false>
void go(long long* d) {
    const int R = 8192;
    const int smem = 48 * 1024 + 1024;
    cudaFuncSetAttribute(rate<CG, N, AT, COMMIT, ST, LD, I8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    rate<CG, N, AT, COMMIT, ST, LD, I8><<<148, 256, smem>>>(R, d);
    rate<CG, N, AT, COMMIT, ST, LD, I8><<<148, 256, smem>>>(R, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[1];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
        printf("err %s\n", cudaGetErrorString(e));
        return;
    }
    const double macs_per_sm = 128.0 * N * 16 * R / h[0];  // per SM (the pair splits M = 256)
    printf("cta_group::%d %s M=%3d N=%3d A=%s commit/%d st=%d ld=%d: %.1f cycles/MMA, %.0f MACs/clk/SM\n", CG,
           I8 ? "i8 " : "f16", 128 * CG, N, AT ? "tmem" : "smem", COMMIT, (int)ST, (int)LD, (double)h[0] / R,
           macs_per_sm * (I8 ? 2 : 1));
}

int main() {
    long long* d;
    cudaMalloc(&d, 64);
    go<2, 128, true>(d);
    go<2, 256, true>(d);
    go<2, 256, true, 8, true, true>(d);
    go<1, 32, true, 0, false, false, true>(d);
    go<1, 32, true, 8, false, false, true>(d);
    go<1, 32, true, 8, true, false, true>(d);
    go<1, 32, true, 8, false, true, true>(d);
    go<1, 32, true, 8, true, true, true>(d);
    go<1, 128, true, 8, true, true, true>(d);
    return 0;
}
