// Persistent dataflow kernel for a dependent chain of fused ITQ3_S GEMVs (decode step).
//
// One CTA per SM runs every stage of the chain in a single launch:
//   * a producer warp streams the CTA's weight units (16 rows x up to 16 256-blocks of
//     tiled 2-bit codes + f16 scales, one cp.async.bulk per field) into an NSLOT-deep shared
//     memory ring guarded by mbarriers.  Weights do not depend on activations, so the
//     stream runs ahead across stage boundaries and HBM never idles on a dependency;
//   * 16 consumer warps compute each unit with m16n8k32 u8 x s8 MMAs (same fragment
//     algebra as gemv.cu) against the stage's rotated activations held in shared memory;
//   * the 16 warps never synchronise per unit: each writes its partial for the slot and the
//     LAST warp to finish (shared-memory counter) reduces it in fixed order, finalises the
//     16-row tile (deterministic across chunks of K) and publishes it with one release
//     increment of the stage's done counter;
//   * at a stage boundary every CTA waits for done[s-1] == RT_{s-1}, then rotates the new
//     input (FWHT + fixed-point limbs, the K3 math) itself into shared memory: no extra
//     global hop for the activation.
// Co-residency of all CTAs (required by the spin waits) is guaranteed by a cooperative
// launch sized to one CTA per SM.
#include <cooperative_groups.h>

#include "common.cuh"

namespace itq3 {

constexpr int kChainConsumerWarps = 16;
constexpr int kChainThreads = 32 * (kChainConsumerWarps + 1);
constexpr int kUnitBlocks = 16;                          // 256-blocks per unit (one per consumer warp)
constexpr int kSlotCodes = kUnitBlocks * 1024;           // 16 KB
constexpr int kSlotScales = kUnitBlocks * 32;            // 512 B
constexpr int kSlotZps = kUnitBlocks * 16;               // 256 B
constexpr int kSlotBytes = kSlotCodes + kSlotScales + kSlotZps;
constexpr int kNumSlots = 8;
constexpr int kMaxChainNB = 48;                          // K up to 12288
constexpr int kMaxLimbs = 4;

struct ChainStage {
    const uint8_t* tiled;  // codes | scales | zps (itq3_repack_tiled layout)
    float* y;              // rows outputs (fp32)
    uint8_t* act;          // NB x act_block_bytes: rotated input of this stage
    int64_t rows, cols;
    int32_t NB, RT, asym, reserved;
};

__host__ __device__ inline int act_block_bytes(int L) { return 256 * L + 32; }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kChainConsumerWarps)); }

__device__ __forceinline__ void mma_u8s8_c(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                           uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

struct ChainSmem {
    uint8_t ring[kNumSlots][kSlotBytes];
    uint8_t act[kMaxChainNB * (256 * kMaxLimbs + 32)];
    float red[kNumSlots][kChainConsumerWarps][16];  // per-slot per-warp row partials (limbs combined)
    float chunkpart[kNumSlots][4][16];                  // per in-flight row tile: per-chunk row sums
    uint64_t full[kNumSlots];
    uint64_t empty[kNumSlots];
    int slotcnt[kNumSlots];
    int rtcnt[kNumSlots];
    int stage_tiles;  // row tiles of the current stage finalised by this CTA
};

constexpr int kMaxChunks = 4;

__device__ __forceinline__ int stage_rt0(int cta, int s, int G) { return (cta + 7 * s) % G; }

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Rotate 256 fp32 values (read through L2) into a compact fragment record in shared memory.
// Integer pipeline on the INT32 pipe: y -> 23-bit fixed point with the block's power-of-two
// scale s_in = 2^(ilogb(max|y|) - 21) (|y_int| < 2^22, as fine as fp32's own rounding of the
// largest elements), exact int32 butterfly (|x'| < 2^30), then x' rounded to the limb range
// |q| <= 2^(8L-2) with one more power-of-two shift k (tests/test_gpu_stack.py chain_bound).
__device__ __forceinline__ float pow2f(int e) { return __int_as_float((e + 127) << 23); }  // e in [-126, 127]

__device__ void chain_rotate_to_smem(const float* src, int L, uint8_t* img, int lane) {
    float f[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) f[e] = __ldcg(src + lane + 32 * e);
    float fmaxa = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) fmaxa = fmaxf(fmaxa, fabsf(f[e]));
#pragma unroll
    for (int o = 16; o; o >>= 1) fmaxa = fmaxf(fmaxa, __shfl_xor_sync(FULL, fmaxa, o));
    const int e_in = fmaxa > 0.f ? ilogbf(fmaxa) - 21 : 0;
    const float sc_in = pow2f(-e_in);
    int v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = __float2int_rn(f[e] * sc_in);
#pragma unroll
    for (int h = 1; h < 32; h <<= 1) {
        const bool high = (lane & h) != 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int p = __shfl_xor_sync(FULL, v[e], h);
            v[e] = high ? p - v[e] : v[e] + p;
        }
    }
#pragma unroll
    for (int hh = 1; hh < 8; hh <<= 1)
#pragma unroll
        for (int e = 0; e < 8; ++e)
            if ((e & hh) == 0) {
                const int lo = v[e], hi = v[e + hh];
                v[e] = lo + hi;
                v[e + hh] = lo - hi;
            }
    unsigned amax = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) amax = max(amax, (unsigned)abs(v[e]));
#pragma unroll
    for (int o = 16; o; o >>= 1) amax = max(amax, __shfl_xor_sync(FULL, amax, o));
    // shift k so that |q| <= 2^(8L-2) (limbs never overflow): bitlen(amax) - k <= 8L - 2
    const int bl = 32 - __clz(amax);
    const int k = max(0, bl - (8 * L - 2));
    const int ex = e_in + k;
    int Q = 0;
    const int tt = (lane & 15) >> 2, beta = lane & 3, half = lane >> 4;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        int q = k ? ((v[e] + (1 << (k - 1))) >> k) : v[e];
        Q += q;
#pragma unroll
        for (int l = 0; l < kMaxLimbs; ++l) {
            if (l < L) {
                const int lb = ((q + 128) & 255) - 128;
                q = (q - lb) >> 8;
                img[((e * L + l) * 4 + tt) * 8 + half * 4 + beta] = (uint8_t)(int8_t)lb;
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) Q += __shfl_xor_sync(FULL, Q, o);
    float* meta = reinterpret_cast<float*>(img + 256 * L);
    if (lane < L) {
        meta[2 * lane] = ldexpf(1.0f, 8 * lane + ex - 4);
        meta[2 * lane + 1] = lane == 0 ? ldexpf((float)Q, ex - 4) : 0.0f;
    }
}

// trace (optional): per (cta, stage) globaltimer stamps
//   0 stage entered, 1 input observed ready, 2 input rotated, 3 last unit of the stage reduced
__global__ void __launch_bounds__(kChainThreads, 1)
    chain_kernel(const ChainStage* __restrict__ stages, int S, const float* __restrict__ x0, int L,
                 unsigned* __restrict__ done, unsigned long long* __restrict__ trace) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    ChainSmem& sm = *reinterpret_cast<ChainSmem*>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int cta = blockIdx.x, G = gridDim.x;
    const int ab = act_block_bytes(L);

    if (tid == 0) {
        for (int i = 0; i < kNumSlots; ++i) {
            mbar_init(&sm.full[i], 1);
            mbar_init(&sm.empty[i], kChainConsumerWarps);
            sm.slotcnt[i] = 0;
            sm.rtcnt[i] = 0;
        }
        sm.stage_tiles = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == kChainConsumerWarps) {
        // ------------------------------ producer ------------------------------
        if (lane == 0) {
            int slot = 0;
            unsigned phase = 0;
            for (int s = 0; s < S; ++s) {
                const ChainStage st = stages[s];
                const uint8_t* scales = st.tiled + (int64_t)st.RT * st.NB * 1024;
                const uint8_t* zps = scales + (int64_t)st.RT * st.NB * 32;
                for (int rt = stage_rt0(cta, s, G); rt < st.RT; rt += G) {
                    for (int b0 = 0; b0 < st.NB; b0 += kUnitBlocks) {
                        const int nb = min(kUnitBlocks, st.NB - b0);
                        mbar_wait(&sm.empty[slot], phase ^ 1u);
                        const int64_t t0 = (int64_t)rt * st.NB + b0;
                        const unsigned bytes = nb * (1024 + 32 + (st.asym ? 16 : 0));
                        mbar_expect_tx(&sm.full[slot], bytes);
                        uint8_t* dst = sm.ring[slot];
                        bulk_g2s(dst, st.tiled + t0 * 1024, nb * 1024, &sm.full[slot]);
                        bulk_g2s(dst + kSlotCodes, scales + t0 * 32, nb * 32, &sm.full[slot]);
                        if (st.asym) bulk_g2s(dst + kSlotCodes + kSlotScales, zps + t0 * 16, nb * 16, &sm.full[slot]);
                        if (++slot == kNumSlots) {
                            slot = 0;
                            phase ^= 1u;
                        }
                    }
                }
            }
        }
        return;
    }

    // ------------------------------ consumers ------------------------------
    const int g = lane >> 2, t = lane & 3;
    int slot = 0;
    unsigned phase = 0;
    int unit_seq = 0;  // row-tile sequence number within the CTA (indexes chunkpart / rtcnt)
    for (int s = 0; s < S; ++s) {
        const ChainStage st = stages[s];
        int rt = stage_rt0(cta, s, G);
        if (rt >= st.RT) continue;
        if (trace && tid == 0) trace[((int64_t)cta * S + s) * 4 + 0] = globaltimer();
        // wait until every row tile of the previous stage is published, then rotate its output
        const float* xin = x0;
        if (s > 0) {
            const ChainStage pv = stages[s - 1];
            xin = pv.y;
            if (tid == 0) {
                while (ld_acquire(&done[s - 1]) < (unsigned)pv.RT) __nanosleep(20);
            }
            consumer_sync();
        }
        if (trace && tid == 0) trace[((int64_t)cta * S + s) * 4 + 1] = globaltimer();
        for (int b = warp; b < st.NB; b += kChainConsumerWarps)
            chain_rotate_to_smem(xin + 256 * b, L, sm.act + b * ab, lane);
        consumer_sync();
        if (trace && tid == 0) trace[((int64_t)cta * S + s) * 4 + 2] = globaltimer();
        const int nch = (st.NB + kUnitBlocks - 1) / kUnitBlocks;
        const int my_tiles = (st.RT - 1 - rt) / G + 1;
        for (; rt < st.RT; rt += G, ++unit_seq) {
            const int rslot = unit_seq % kNumSlots;
            for (int ch = 0; ch < nch; ++ch) {
                const int b0 = ch * kUnitBlocks;
                mbar_wait(&sm.full[slot], phase);
                const int b = b0 + warp;
                float acc[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
                if (b < st.NB) {
                    const uint8_t* ring = sm.ring[slot];
                    const uint4 wa0 = reinterpret_cast<const uint4*>(ring + warp * 1024)[lane];
                    const uint4 wa1 = reinterpret_cast<const uint4*>(ring + warp * 1024 + 512)[lane];
                    const uint32_t sc = reinterpret_cast<const uint32_t*>(ring + kSlotCodes + warp * 32)[g];
                    uint16_t zz = 0;
                    if (st.asym) zz = reinterpret_cast<const uint16_t*>(ring + kSlotCodes + kSlotScales + warp * 16)[g];
                    const uint8_t* a = sm.act + b * ab;
                    uint2 bf[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        bf[q] = g < L ? reinterpret_cast<const uint2*>(a)[(q * L + g) * 4 + t] : make_uint2(0u, 0u);
                    const float* meta = reinterpret_cast<const float*>(a + 256 * L);
                    const float f0 = 2 * t < L ? meta[4 * t] : 0.f, c0 = 2 * t < L ? meta[4 * t + 1] : 0.f;
                    const float f1 = 2 * t + 1 < L ? meta[4 * t + 2] : 0.f, c1 = 2 * t + 1 < L ? meta[4 * t + 3] : 0.f;
                    int C[4][4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) C[i][0] = C[i][1] = C[i][2] = C[i][3] = 0;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const uint32_t mk = 0x03030303u << (2 * i);
                        mma_u8s8_c(C[i], wa0.x & mk, wa0.y & mk, wa0.z & mk, wa0.w & mk, bf[i].x, bf[i].y);
                    }
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const uint32_t mk = 0x03030303u << (2 * i);
                        mma_u8s8_c(C[i], wa1.x & mk, wa1.y & mk, wa1.z & mk, wa1.w & mk, bf[4 + i].x, bf[4 + i].y);
                    }
                    int Cc[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) Cc[r] = C[0][r] + (C[1][r] >> 2) + (C[2][r] >> 4) + (C[3][r] >> 6);
                    const float d0 = f16_bits_to_f32((uint16_t)(sc & 0xffffu));
                    const float d1 = f16_bits_to_f32((uint16_t)(sc >> 16));
                    float zf0 = 1.f, zf1 = 1.f;
                    if (st.asym) {
                        zf0 = (float)(1 + (int)(int8_t)(zz & 0xff));
                        zf1 = (float)(1 + (int)(int8_t)(zz >> 8));
                    }
                    acc[0][0] = d0 * (f0 * (float)Cc[0] - zf0 * c0);
                    acc[0][1] = d0 * (f1 * (float)Cc[1] - zf0 * c1);
                    acc[1][0] = d1 * (f0 * (float)Cc[2] - zf1 * c0);
                    acc[1][1] = d1 * (f1 * (float)Cc[3] - zf1 * c1);
                }
                // combine limb columns in-warp (fixed order: quad lanes t = 0..3 via xor 1, 2), then
                // publish one partial per row; the last warp to finish the slot reduces it
                float r0 = acc[0][0] + acc[0][1], r1 = acc[1][0] + acc[1][1];
                r0 += __shfl_xor_sync(FULL, r0, 1);
                r1 += __shfl_xor_sync(FULL, r1, 1);
                r0 += __shfl_xor_sync(FULL, r0, 2);
                r1 += __shfl_xor_sync(FULL, r1, 2);
                if (t == 0) {
                    sm.red[slot][warp][g] = r0;
                    sm.red[slot][warp][g + 8] = r1;
                }
                __syncwarp();
                int last = 0;
                if (lane == 0) {
                    __threadfence_block();
                    last = atomicAdd(&sm.slotcnt[slot], 1) == kChainConsumerWarps - 1;
                }
                last = __shfl_sync(FULL, last, 0);
                if (!last) {
                    if (lane == 0) mbar_arrive(&sm.empty[slot]);
                } else {
                    __threadfence_block();
                    float rsum = 0.f;
                    if (lane < 16) {
                        float part[kChainConsumerWarps];
#pragma unroll
                        for (int w = 0; w < kChainConsumerWarps; ++w) part[w] = sm.red[slot][w][lane];
#pragma unroll
                        for (int w = 0; w < kChainConsumerWarps; ++w) rsum += part[w];
                    }
                    __syncwarp();
                    if (lane == 0) {
                        sm.slotcnt[slot] = 0;
                        mbar_arrive(&sm.empty[slot]);
                    }
                    bool final = nch == 1;
                    if (!final) {
                        if (lane < 16) sm.chunkpart[rslot][ch][lane] = rsum;
                        __syncwarp();
                        int cnt = 0;
                        if (lane == 0) {
                            __threadfence_block();
                            cnt = atomicAdd(&sm.rtcnt[rslot], 1) + 1;
                        }
                        cnt = __shfl_sync(FULL, cnt, 0);
                        if (cnt == nch) {
                            __threadfence_block();
                            final = true;
                            rsum = 0.f;
                            if (lane < 16)
                                for (int c = 0; c < nch; ++c) rsum += sm.chunkpart[rslot][c][lane];
                            if (lane == 0) sm.rtcnt[rslot] = 0;
                        }
                    }
                    if (final) {
                        const int64_t row = (int64_t)rt * 16 + lane;
                        if (lane < 16 && row < st.rows) __stcg(st.y + row, rsum);
                        __syncwarp();
                        if (lane == 0) {
                            // publish once per CTA per stage: the warp finalising the CTA's last
                            // tile fences (cumulative over the CTA's y stores) and bumps done[s]
                            __threadfence_block();
                            if (atomicAdd(&sm.stage_tiles, 1) + 1 == my_tiles) {
                                sm.stage_tiles = 0;
                                __threadfence();
                                atomicAdd(&done[s], (unsigned)my_tiles);
                                if (trace) trace[((int64_t)cta * S + s) * 4 + 3] = globaltimer();
                            }
                        }
                    }
                }
                if (++slot == kNumSlots) {
                    slot = 0;
                    phase ^= 1u;
                }
            }
        }
    }
}

}  // namespace itq3

using namespace itq3;

extern "C" int64_t itq3_chain_desc_nbytes(void) { return (int64_t)sizeof(ChainStage); }
extern "C" int itq3_chain_act_block_bytes(int limbs) { return act_block_bytes(limbs); }
extern "C" int itq3_chain_smem_bytes(void) { return (int)sizeof(ChainSmem); }

extern "C" int itq3_chain_write_desc(void* host_desc, int index, const uint8_t* tiled, float* y, uint8_t* act,
                                     int64_t rows, int64_t cols, int asymmetric, int ycnt_off) {
    if (cols % 256 || cols / 256 > kMaxChainNB) {
        set_error("chain: stage %d needs cols %% 256 == 0 and cols <= %d (got %lld)", index, 256 * kMaxChainNB,
                  (long long)cols);
        return ITQ3_E_UNSUPPORTED;
    }
    ChainStage& st = reinterpret_cast<ChainStage*>(host_desc)[index];
    st.tiled = tiled;
    st.y = y;
    st.act = act;
    st.rows = rows;
    st.cols = cols;
    st.NB = (int)(cols / 256);
    st.RT = (int)((rows + 15) / 16);
    st.asym = asymmetric;
    st.reserved = ycnt_off;
    return ITQ3_OK;
}

extern "C" int itq3_chain_run(const void* d_desc, int n_stages, const float* x0, int limbs, unsigned* d_counters,
                              int grid, void* d_trace, void* stream) {
    if (limbs < 1 || limbs > kMaxLimbs) {
        set_error("chain: limbs must be in [1, %d]", kMaxLimbs);
        return ITQ3_E_DOMAIN;
    }
    static bool attr_set = false;
    const int smem = (int)sizeof(ChainSmem);
    if (!attr_set) {
        if (cudaFuncSetAttribute(chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
            return check_launch("chain: smem attribute");
        attr_set = true;
    }
    if (grid <= 0) {
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        grid = sms;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kChainThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, chain_kernel, (const ChainStage*)d_desc, n_stages, x0, limbs,
                                             d_counters, (unsigned long long*)d_trace);
    if (e != cudaSuccess) {
        set_error("chain: launch failed: %s", cudaGetErrorString(e));
        return ITQ3_E_CUDA;
    }
    return check_launch("itq3_chain_run");
}
