// Probe: the register <-> shared-memory mapping of stmatrix.m16n8.x1.trans.b8 (sm_100a), by tagging every
// source byte with (lane, byte) and dumping the 32-row window each lane's address points at.
#include <cstdio>
__global__ void k(unsigned char* out) {
    __shared__ __align__(128) unsigned char buf[32 * 32];
    for (int i = threadIdx.x; i < 1024; i += 32) buf[i] = 0xff;
    __syncwarp();
    const unsigned lane = threadIdx.x;
    const unsigned r = (lane * 4 + 0) | ((lane * 4 + 1) << 8) | ((lane * 4 + 2) << 16) | ((lane * 4 + 3) << 24);
    const unsigned a = (unsigned)__cvta_generic_to_shared(buf) + lane * 32;  // row `lane` at 32-byte pitch
    asm volatile("stmatrix.sync.aligned.m16n8.x1.trans.shared.b8 [%0], {%1};" ::"r"(a), "r"(r) : "memory");
    __syncwarp();
    for (int i = threadIdx.x; i < 1024; i += 32) out[i] = buf[i];
}
int main() {
    unsigned char* d;
    cudaMalloc(&d, 1024);
    k<<<1, 32>>>(d);
    unsigned char h[1024];
    cudaMemcpy(h, d, 1024, cudaMemcpyDeviceToHost);
    for (int row = 0; row < 32; ++row) {
        printf("row %2d:", row);
        for (int c = 0; c < 32; ++c) {
            if (h[row * 32 + c] == 0xff) printf("  .  ");
            else printf(" %2d.%d", h[row * 32 + c] / 4, h[row * 32 + c] % 4);
        }
        printf("\n");
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
