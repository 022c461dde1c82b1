// Probe: cycles per 16-row x 4096-k unit of the chain kernel's tile loop with 16 consumer warps on one
// SM, the ring pre-filled in shared memory (no HBM, no producer, no reducer): (1) chain_tile2 pairs + the
// partial stores only, (2) + per-unit mbarrier waits / arrives on barriers that are already complete.  The
// gap to the in-kernel rate (~0.38 us per unit on the critical path) is what the pipeline around the loop
// costs.   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/probes/tile_probe \
//              tools/probes/tile_probe.cu build/runtime.o
#include "../../paper_2603_27914_b200/csrc/chain.cu"
#include <cstdio>
#include <vector>

using namespace itq3;

constexpr int kProbeSlots = 10;
struct ProbeSmem {
    alignas(128) uint8_t ring[kProbeSlots][kSlotBytes];
    float part[kProbeSlots][kChainConsumerWarps][2][16];
    uint64_t full[kProbeSlots];
    uint64_t parts[kProbeSlots];
};

template <int VAR>
__global__ void __launch_bounds__(512, 1) tile_probe(int iters, long long* out, float* sink) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    ProbeSmem& sm = *reinterpret_cast<ProbeSmem*>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    for (int i = tid; i < kProbeSlots * kSlotBytes / 4; i += 512)
        reinterpret_cast<uint32_t*>(&sm.ring[0][0])[i] = (i * 2654435761u) & 0x3c00aaaau;
    if (tid == 0)
        for (int i = 0; i < kProbeSlots; ++i) {
            mbar_init(&sm.full[i], 1);
            mbar_init(&sm.parts[i], 1);
            mbar_arrive(&sm.full[i]);  // complete phase 0
        }
    __syncthreads();
    uint2 bf[8];
    for (int q = 0; q < 8; ++q) bf[q] = make_uint2(0x01020304u * (q + 1), 0x05060708u + lane);
    const float fcx = 1e-3f, corr = 0.5f;
    float acc = 0.f;
    __syncwarp();
    const long long t0 = clock64();
    int cs = 0;
    for (int it = 0; it < iters; ++it) {
        const int slot0 = cs, slot1 = cs + 1 < kProbeSlots ? cs + 1 : 0;
        cs = slot1 + 1 < kProbeSlots ? slot1 + 1 : 0;
        if (VAR == 1) {
            mbar_wait(&sm.full[slot0], 0);
            mbar_wait(&sm.full[slot1], 0);
        }
        float2 ra, rb;
        chain_tile2<false>(sm.ring[slot0], sm.ring[slot1], warp, lane, g, bf, fcx, corr, ra, rb);
        if (t < 2) {
            sm.part[slot0][warp][t][g] = ra.x;
            sm.part[slot0][warp][t][g + 8] = ra.y;
            sm.part[slot1][warp][t][g] = rb.x;
            sm.part[slot1][warp][t][g + 8] = rb.y;
        }
        __syncwarp();
        if (VAR == 1 && lane == 0 && warp == 0 && it < 0) mbar_arrive(&sm.parts[slot0]);  // (never: keeps the code)
        acc += ra.x + rb.y;
    }
    const long long t1 = clock64();
    if (lane == 0) out[warp] = (t1 - t0);
    if (acc == 12345.f) sink[tid] = acc;
}

template <int VAR>
void run(long long* d, float* sink, const char* name) {
    const int smem = (int)sizeof(ProbeSmem);
    cudaFuncSetAttribute(tile_probe<VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 2000;
    tile_probe<VAR><<<148, 512, smem>>>(iters, d, sink);
    tile_probe<VAR><<<148, 512, smem>>>(iters, d, sink);
    cudaDeviceSynchronize();
    std::vector<long long> h(16);
    cudaMemcpy(h.data(), d, 16 * 8, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (long long v : h) mx = v > mx ? v : mx;
    printf("%-34s %6.1f cycles per unit (16 warps, %d units)  [%s]\n", name, mx / (2.0 * iters), 2 * iters,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    long long* d;
    float* sink;
    cudaMalloc(&d, 64 * 8);
    cudaMalloc(&sink, 4096);
    run<0>(d, sink, "tile pairs + partial stores");
    run<1>(d, sink, "+ mbarrier waits (complete)");
    return 0;
}
