// Micro-probe: throughput/latency of legacy mma.sync m16n8k32 u8 x s8 (IMMA.16832) and of the
// 2-bit-class LOP3 + IMMA tile loop on sm_100a.  One CTA per SM, W warps, N iterations.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
__device__ __forceinline__ void mma(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
template <int CHAINS>
__global__ void imma_tput(int iters, int* out, uint32_t seed) {
    int c[CHAINS][4] = {};
    uint32_t a = seed ^ threadIdx.x, b = seed * 3u;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < CHAINS; ++k) mma(c[k], a, a + k, a ^ k, a + 2 * k, b, b + k);
    }
    int s = 0;
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
    if (s == 0x1234567) out[0] = s;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int* out; cudaMalloc(&out, 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 4096;
    for (int warps : {1, 4, 8, 16}) {
        for (int pass = 0; pass < 2; ++pass) {
            cudaEventRecord(e0);
            imma_tput<8><<<sms, 32 * warps>>>(iters, out, 7);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
        }
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double mmas = (double)sms * warps * iters * 8;
        const double clk = 1.965e9;
        printf("warps/SM=%2d  chains=8: %.2f IMMA/clk/SM  (%.1f TOPS int8)\n", warps, mmas / (ms * 1e-3) / sms / clk,
               mmas * 16 * 8 * 32 * 2 / (ms * 1e-3) / 1e12);
    }
    for (int pass = 0; pass < 2; ++pass) {
        cudaEventRecord(e0);
        imma_tput<1><<<sms, 32>>>(iters * 8, out, 7);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("dependent chain latency: %.1f clk per IMMA\n", ms * 1e-3 * 1.965e9 / (iters * 8));
    return 0;
}
