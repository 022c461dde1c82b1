// Legacy mma.sync m16n8k32 u8.s8 issue rate on sm_100a: cycles per IMMA per SM vs warps per CTA.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/probes/imma_rate_probe.cu -o tools/probes/imma_rate_probe
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ void mma(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma4(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k64.row.col.s32.u4.s4.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__global__ void k4(int iters, int* out, long long* cyc) {
    int c[8][4] = {};
    uint32_t a = threadIdx.x * 0x01010101u, b = blockIdx.x;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) mma4(c[j], a + j, a ^ j, a + 2 * j, a, b, b + j);
    }
    __syncthreads();
    long long t1 = clock64();
    int s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int CH>
__global__ void k(int iters, int* out, long long* cyc) {
    int c[CH][4] = {};
    uint32_t a = threadIdx.x * 0x01010101u, b = blockIdx.x;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < CH; ++j) mma(c[j], a + j, a ^ j, a + 2 * j, a, b, b + j);
    }
    __syncthreads();
    long long t1 = clock64();
    int s = 0;
#pragma unroll
    for (int j = 0; j < CH; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
// IMMA interleaved with X independent integer ops per IMMA: does the IMMA block issue?
template <int X>
__global__ void kx(int iters, int* out, long long* cyc) {
    int c[4][4] = {};
    uint32_t a = threadIdx.x * 0x01010101u, b = blockIdx.x;
    uint32_t z[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) z[j] = threadIdx.x + j;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            mma(c[j], a + j, a ^ j, a + 2 * j, a, b, b + j);
#pragma unroll
            for (int x = 0; x < X; ++x) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(z[x & 7]) : "r"(a), "r"(b));
        }
    }
    __syncthreads();
    long long t1 = clock64();
    int s = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
#pragma unroll
    for (int j = 0; j < 8; ++j) s += z[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int X>
void runx(int* out, long long* cyc, int iters) {
    kx<X><<<148, 16 * 32>>>(iters, out, cyc);
    cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    const double per = (double)h[0] / ((double)iters * 4 * 4);  // per IMMA per SMSP (4 warps/SMSP)
    printf("16 warps, IMMA + %2d LOP3 each: %.2f cycles per (IMMA + %d LOP3) per SMSP\n", X, per, X);
}
int main() {
    int* out; long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
    const int iters = 2000;
    for (int warps : {1, 2, 4, 8, 16}) {
        k<8><<<148, warps * 32>>>(iters, out, cyc);
        cudaDeviceSynchronize();
        long long h[148]; cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
        const double per = (double)h[0] / ((double)iters * 8 * warps);
        printf("warps/CTA %2d (8 independent chains each): %.2f cycles per IMMA.16832 per SM  (%.1f per SMSP)\n",
               warps, per, per * (warps < 4 ? warps : 4));
    }
    for (int warps : {4, 16}) {
        k<2><<<148, warps * 32>>>(iters, out, cyc);
        cudaDeviceSynchronize();
        long long h[148]; cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
        printf("warps/CTA %2d (2 chains each): %.2f cycles per IMMA per SM\n", warps, (double)h[0] / ((double)iters * 2 * warps));
    }
    for (int warps : {4, 16}) {
        k4<<<148, warps * 32>>>(iters, out, cyc);
        cudaDeviceSynchronize();
        long long h[148]; cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
        printf("u4.s4 m16n8k64: warps/CTA %2d: %.2f cycles per IMMA per SM\n", warps, (double)h[0] / ((double)iters * 8 * warps));
    }
    runx<0>(out, cyc, iters);
    runx<2>(out, cyc, iters);
    runx<4>(out, cyc, iters);
    runx<8>(out, cyc, iters);
    runx<12>(out, cyc, iters);
    runx<16>(out, cyc, iters);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
