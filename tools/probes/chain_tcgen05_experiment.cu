// EXPERIMENT (not built): decode chain with the multiply on tcgen05.mma kind::i8, A = class-masked
// codes written to TMEM by tcgen05.st.  Correct (tests passed) but 2.1x slower than the IMMA chain:
// each MMA (M=128, K=32) covers 4096 weights and costs >= 55.6 cycles (probe), and the 4x operand
// expansion (32 KB of A per 8 KB record) goes through tcgen05.st at ~125 B/clk; measured 1180
// cycles per record in situ.  See DESIGN.md "Why the GEMV stays on mma.sync".
// Persistent dataflow kernel for a dependent chain of fused ITQ3_S GEMVs (decode step), with
// the multiply on the 5th-generation tensor cores (tcgen05.mma kind::i8, A from TMEM).
//
// One CTA per SM runs every stage of the chain in a single cooperative launch:
//   * a producer warp streams the CTA's weight records (16 rows x 8 blocks of 256: 8 KB of
//     2-bit codes + f16 scales [+ int8 zero-points], one contiguous cp.async.bulk) into a
//     16-deep shared-memory ring guarded by mbarriers.  Weights do not depend on activations,
//     so the stream runs ahead across stage boundaries and HBM never idles on a dependency;
//   * 16 expander warps in 4 groups take the records round-robin.  A thread owns one (row,
//     block) pair of a record = one TMEM lane (lane 16j + r: block j, row r) and writes its 64
//     code bytes as 4 class-masked copies (A = byte & (3 << 2i) = c * 4^i, u8) into TMEM with one
//     tcgen05.st; the MMA warp then issues 8 x tcgen05.mma M=128 N=32 K=32 (A from TMEM, B =
//     the stage's rotated activation limbs in shared memory, s32 accumulators in TMEM).  B row
//     4j + l holds limb l of block j; D[16j + r][4j + l] is the row-r dot product with block j
//     in limb l (off-diagonal columns are unused);
//   * the same thread reads its 4 diagonal accumulators back (tcgen05.ld), folds limbs, scale and
//     zero-point, and accumulates the unit's row partial; 16 per-warp partials of each unit are
//     summed in fixed order by a reducer warp (deterministic) and stored as tagged outputs;
//   * no counters, flags or fences between stages: every output word is 64 bits = (fp32 value,
//     step epoch), stored and loaded single-copy atomically, so an expander warp simply spins
//     until the 256 x nch tags of the block it needs carry the current epoch, then rotates that
//     block (FWHT + fixed-point limbs, the K3 math) straight into the B tile.
// Co-residency of all CTAs (required by the spin waits) is guaranteed by a cooperative launch
// sized to one CTA per SM.
#include <cooperative_groups.h>

#include "common.cuh"

namespace itq3 {

constexpr int kExpWarps = 16;                       // 4 groups x 4 TMEM lane quarters
constexpr int kGroups = 4;
constexpr int kProducerWarp = 16, kMmaWarp = 17, kReducerWarp = 18;
constexpr int kChainThreads = 32 * 19;
constexpr int kUnitBlocks = 16;                      // K-chunk of a unit (2 records)
constexpr int kRecBlocks = 8;                        // blocks per record
constexpr int kRecCodes = 4 * 128 * 16;              // [chunk c][lane L][16 B] = 8 KB
constexpr int kRecBytes = kRecCodes + 256 + 128;     // + f16 scales [L] + int8 zps [L]
constexpr int kNumSlots = 16;
constexpr int kPartSlots = 8;
constexpr int kMaxChainNB = 256;                     // K up to 65536
constexpr int kMaxLimbs = 4;
constexpr int kBTile = 8192;                         // B tile of one record: 2 k-atoms x 4 KB
constexpr uint32_t kTmemCols = 512;                  // A slots: 64 cols x 4 groups; D: 32 cols x 4

struct ChainStage {
    const uint8_t* tiled;  // chain layout (itq3_repack_chain): records [RT][NR][kRecBytes]
    unsigned long long* y; // [nch][rows] tagged outputs: low 32 = fp32 bits, high 32 = step epoch
    const float* xin;      // optional: untagged fp32 input (independent stage, no dependency)
    int64_t rows, cols;
    int32_t NB, RT, asym, reserved;
};

__host__ __device__ inline int act_block_bytes(int) { return 4 * 256 + 8; }  // 4 limb rows + (fcx, corr)

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
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void expander_sync() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kExpWarps)); }

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row core groups 1024 B apart.
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
// swizzled byte offset of (row n, 16-byte chunk c) inside a K-major SW128 tile
__device__ __forceinline__ uint32_t sw128_off(int n, int c) {
    return (uint32_t)((n >> 3) * 1024 + (n & 7) * 128 + ((c ^ (n & 7)) << 4));
}

__device__ __forceinline__ float pow2f(int e) {  // exact 2^e, bit-built on the normal range
    return (e >= -126 && e <= 127) ? __int_as_float((e + 127) << 23) : ldexpf(1.0f, e);
}

__device__ __forceinline__ unsigned long long ld_u64_relaxed(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_u64_relaxed(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Wait for, and sum, one 256-block of a producing stage's tagged K-chunk partials.  Each 64-bit
// word carries its value and the step epoch in one single-copy-atomic access, so the consumer
// needs no flag, counter or fence: it spins until all 256 x nparts tags equal `epoch`.
__device__ __forceinline__ void load_tagged_block(const unsigned long long* src, int nparts, int64_t part_stride,
                                                  unsigned epoch, int lane, float (&f)[8]) {
    for (;;) {
        bool ok = true;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const unsigned long long w = ld_u64_relaxed(src + lane + 32 * e);
            ok &= (unsigned)(w >> 32) == epoch;
            f[e] = __uint_as_float((unsigned)w);
        }
        for (int c = 1; c < nparts; ++c)  // K-chunk partials, fixed order
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const unsigned long long w = ld_u64_relaxed(src + c * part_stride + lane + 32 * e);
                ok &= (unsigned)(w >> 32) == epoch;
                f[e] += __uint_as_float((unsigned)w);
            }
        if (__all_sync(FULL, ok)) return;
        __nanosleep(64);
    }
}

// Rotate one 256-block (element e = lane + 32 t in this lane's f[t]) into the B tile rows
// 4j..4j+3 of its record.  Integer pipeline: y -> 23-bit fixed point with the block's
// power-of-two scale s_in = 2^(ilogb(max|y|) - 21), exact int32 butterfly (|x'| < 2^30), then x'
// rounded to |q| <= 2^(8L-2) with one more power-of-two shift k (tests/test_gpu_stack.py
// chain_bound).  Class folding: element e pairs with the A operand c * 4^(e >> 6), so its
// activation is stored pre-scaled by 4^(3 - (e >> 6)); the four balanced base-256 limbs of
// q * 4^(3 - i) are the bytes of (qs + 0x80808080) ^ 0x80808080.  meta = (2^(ex-10), Q 2^(ex-4)).
__device__ void chain_rotate_block(const float (&fin)[8], int L, uint8_t* btile, int j, float* meta, int lane) {
    float f[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) f[e] = fin[e];
    unsigned fbits = 0;  // warp max of |f| as an integer max of the non-negative bit patterns
#pragma unroll
    for (int e = 0; e < 8; ++e) fbits = max(fbits, __float_as_uint(fabsf(f[e])));
    fbits = __reduce_max_sync(FULL, fbits);
    const float fmaxa = __uint_as_float(fbits);
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
    amax = __reduce_max_sync(FULL, amax);
    const int bl = 32 - __clz(amax);
    const int k = max(0, bl - min(8 * L - 2, 22));  // |q| <= 2^22: q * 64 fits the 4 limbs
    const int ex = e_in + k;
    int Q = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        const int q = k ? ((v[t] + (1 << (k - 1))) >> k) : v[t];
        Q += q;
        const int e = lane + 32 * t;  // element index; class i = e >> 6 = t >> 1
        const int qs = q << (2 * (3 - (t >> 1)));
        const uint32_t limbs = (uint32_t)(qs + (int)0x80808080u) ^ 0x80808080u;
        const int b = e & 127;
        uint8_t* base = btile + (e >> 7) * 4096 + (b & 15);
#pragma unroll
        for (int l = 0; l < 4; ++l) base[sw128_off(4 * j + l, b >> 4)] = (uint8_t)(limbs >> (8 * l));
    }
    Q = __reduce_add_sync(FULL, Q);
    if (lane == 0) {
        meta[0] = pow2f(ex - 10);  // 2^ex / 16 / 64 (class-folding factor)
        meta[1] = (float)Q * pow2f(ex - 4);
    }
}

// zero rows 4j..4j+3 of a record's B tile (block absent from the K-chunk)
__device__ void chain_zero_block(uint8_t* btile, int j, float* meta, int lane) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        const int idx = lane + 32 * t;  // 256 16-B... (row l, k-atom, chunk): 4 x 2 x 8 = 64 chunks
        if (idx < 64) {
            const int l = idx >> 4, ka = (idx >> 3) & 1, c = idx & 7;
            *reinterpret_cast<uint4*>(btile + ka * 4096 + sw128_off(4 * j + l, c)) = make_uint4(0, 0, 0, 0);
        }
    }
    if (lane == 0) {
        meta[0] = 0.f;
        meta[1] = 0.f;
    }
}

struct ChainSmem {
    uint8_t btile[2][kBTile];                          // B tiles of the unit's 2 records (1024-aligned)
    uint8_t ring[kNumSlots][kRecBytes];
    float meta[kUnitBlocks][2];                        // per block: (fcx, corr)
    float part[kPartSlots][kExpWarps][16];             // per-warp row partials of a unit
    uint64_t full[kNumSlots];
    uint64_t empty[kNumSlots];
    uint64_t aready[kGroups];  // group's A written to TMEM (4 warps)
    uint64_t dfull[kGroups];   // group's MMAs done (tcgen05.commit)
    uint64_t bready;           // stage's B tiles rotated (16 warps)
    uint64_t pfull[kPartSlots];
    uint64_t pfree[kPartSlots];
    uint32_t tmem_base;
};

static_assert(sizeof(ChainSmem) + 1024 <= 227 * 1024, "chain kernel shared memory exceeds the 227 KB per-CTA limit");

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Work split of stage st for CTA cta: K-chunk ch (CTAs c with c % nch == ch), and the 16-row
// tiles rt = rt0, rt0 + Gc, ... (Gc CTAs per chunk).  Returns false if the CTA is idle.
struct StageSplit {
    int nch, ch, rt0, Gc;
};
__device__ __forceinline__ bool stage_split(const ChainStage& st, int cta, int G, int s, StageSplit& sp) {
    sp.nch = (st.NB + kUnitBlocks - 1) / kUnitBlocks;
    sp.Gc = G / sp.nch;
    sp.ch = cta % sp.nch;
    const int idx = cta / sp.nch;
    if (idx >= sp.Gc) return false;
    sp.rt0 = (idx + 7 * s) % sp.Gc;
    return sp.rt0 < st.RT;
}

__global__ void chain_epoch_kernel(unsigned* epoch) { *epoch += 1; }

// trace (optional): per (cta, stage) globaltimer stamps
//   0 stage entered, 1 input observed ready, 2 input rotated, 3 own units done
__global__ void __launch_bounds__(kChainThreads, 1)
    chain_kernel(const ChainStage* __restrict__ stages, int S, const float* __restrict__ x0, int L,
                 const unsigned* __restrict__ epoch_ptr, float* __restrict__ out,
                 unsigned long long* __restrict__ trace) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    ChainSmem& sm = *reinterpret_cast<ChainSmem*>(base);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int cta = blockIdx.x, G = gridDim.x;
    const unsigned epoch = *epoch_ptr;

    if (tid == 0) {
        for (int i = 0; i < kNumSlots; ++i) {
            mbar_init(&sm.full[i], 1);
            mbar_init(&sm.empty[i], 4);  // the owning group's 4 warps
        }
        for (int g = 0; g < kGroups; ++g) {
            mbar_init(&sm.aready[g], 4);
            mbar_init(&sm.dfull[g], 1);
        }
        mbar_init(&sm.bready, kExpWarps);
        for (int i = 0; i < kPartSlots; ++i) {
            mbar_init(&sm.pfull[i], kExpWarps);
            mbar_init(&sm.pfree[i], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_base)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;

    if (warp == kReducerWarp) {
        // ------------------------------ reducer ------------------------------
        int useq = 0;
        for (int s = 0; s < S; ++s) {
            const ChainStage st = stages[s];
            StageSplit sp;
            if (!stage_split(st, cta, G, s, sp)) continue;
            const int n_units = (st.RT - 1 - sp.rt0) / sp.Gc + 1;
            unsigned long long* yout = st.y + (int64_t)sp.ch * st.rows;
            const unsigned long long tag = (unsigned long long)epoch << 32;
            for (int j = 0; j < n_units; ++j, ++useq) {
                const int ps = useq % kPartSlots;
                mbar_wait(&sm.pfull[ps], (unsigned)(useq / kPartSlots) & 1u);
                if (lane < 16) {
                    float sum = sm.part[ps][0][lane];
#pragma unroll
                    for (int w = 1; w < kExpWarps; ++w) sum += sm.part[ps][w][lane];
                    const int64_t row = (int64_t)(sp.rt0 + j * sp.Gc) * 16 + lane;
                    if (row < st.rows) st_u64_relaxed(yout + row, tag | __float_as_uint(sum));
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.pfree[ps]);
            }
        }
    } else if (warp == kProducerWarp) {
        // ------------------------------ producer ------------------------------
        if (lane == 0) {
            int rs = 0;
            for (int s = 0; s < S; ++s) {
                const ChainStage st = stages[s];
                StageSplit sp;
                if (!stage_split(st, cta, G, s, sp)) continue;
                const int NR = (st.NB + kRecBlocks - 1) / kRecBlocks;
                const int kr0 = sp.ch * (kUnitBlocks / kRecBlocks);
                const int nrec = min(kUnitBlocks / kRecBlocks, NR - kr0);
                const unsigned bytes = kRecCodes + 256 + (st.asym ? 128 : 0);
                for (int rt = sp.rt0; rt < st.RT; rt += sp.Gc)
                    for (int r = 0; r < nrec; ++r, ++rs) {
                        const int slot = rs % kNumSlots;
                        mbar_wait(&sm.empty[slot], ((unsigned)(rs / kNumSlots) & 1u) ^ 1u);
                        mbar_expect_tx(&sm.full[slot], bytes);
                        bulk_g2s(sm.ring[slot], st.tiled + ((int64_t)rt * NR + kr0 + r) * kRecBytes, bytes,
                                 &sm.full[slot]);
                    }
            }
        }
    } else if (warp == kMmaWarp) {
        // ------------------------------ MMA issuer ------------------------------
        if (lane == 0) {
            // D s32, A u8, B s8, both K-major, N = 32, M = 128
            const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
            int rs = 0, act = 0;
            const bool prof = trace != nullptr && cta == 0;
            long long m_wait_a = 0, m_wait_b = 0, m_start = clock64(), m0 = 0;
            for (int s = 0; s < S; ++s) {
                const ChainStage st = stages[s];
                StageSplit sp;
                if (!stage_split(st, cta, G, s, sp)) continue;
                const int NR = (st.NB + kRecBlocks - 1) / kRecBlocks;
                const int nrec = min(kUnitBlocks / kRecBlocks, NR - sp.ch * (kUnitBlocks / kRecBlocks));
                if (prof) m0 = clock64();
                mbar_wait(&sm.bready, (unsigned)(act++) & 1u);
                if (prof) m_wait_b += clock64() - m0;
                const int n_units = (st.RT - 1 - sp.rt0) / sp.Gc + 1;
                for (int u = 0; u < n_units; ++u)
                    for (int r = 0; r < nrec; ++r, ++rs) {
                        const int g = rs % kGroups;
                        if (prof) m0 = clock64();
                        mbar_wait(&sm.aready[g], (unsigned)(rs / kGroups) & 1u);
                        if (prof) m_wait_a += clock64() - m0;
                        tc_fence_after();
                        const uint32_t bt = smem_u32(sm.btile[r]);
                        const uint32_t ta = tmem + 64u * g, td = tmem + 256u + 32u * g;
#pragma unroll
                        for (int m = 0; m < 8; ++m) {
                            const uint64_t bd = desc_sw128(bt + (m >> 2) * 4096 + 32 * (m & 3));
                            const uint32_t acc = m > 0;
                            asm volatile(
                                "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                                " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(td),
                                "r"(ta + 8u * m), "l"(bd), "r"(idesc), "r"(acc));
                        }
                        asm volatile(
                            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                smem_u32(&sm.dfull[g]))
                            : "memory");
                    }
            }
            if (prof) {
                unsigned long long* pt = trace + (int64_t)G * S * 4 + (int64_t)S * 64;  // slot of warp 0..15 used
                pt[16 * 4 - 4 + 0] = 0;
                (void)pt;
                unsigned long long* pm = trace + (int64_t)G * S * 4;  // stage-0 row of the per-stage area
                pm[0] = m_wait_a;
                pm[1] = m_wait_b;
                pm[2] = clock64() - m_start;
                pm[3] = rs;
            }
        }
    } else {
        // ------------------------------ expanders ------------------------------
        const int g = warp >> 2, q = warp & 3;
        const int Lr = 32 * q + lane;             // TMEM lane = 16 j + r
        const int jb = Lr >> 4, r16 = Lr & 15;    // block within the record, row within the tile
        const uint32_t lane_base = (uint32_t)(32 * q) << 16;
        const uint32_t ta = tmem + lane_base + 64u * g;
        const uint32_t td = tmem + lane_base + 256u + 32u * g + 8u * q;  // cols 4 jb .. : 8 q .. 8 q + 7
        int rs = 0, useq = 0;
        const bool prof = trace != nullptr && cta == 0;
        long long c_full = 0, c_st = 0, c_d = 0, c_start = clock64(), c0 = 0;
        for (int s = 0; s < S; ++s) {
            const ChainStage st = stages[s];
            StageSplit sp;
            if (!stage_split(st, cta, G, s, sp)) continue;
            if (trace && tid == 0) trace[((int64_t)cta * S + s) * 4 + 0] = globaltimer();
            const int b0 = sp.ch * kUnitBlocks;
            const int nb = min(kUnitBlocks, st.NB - b0);
            const int nrec = (nb + kRecBlocks - 1) / kRecBlocks;
            // -- rotate block `warp` of the K-chunk into the B tile (record warp / 8, rows 4 j..)
            {
                uint8_t* bt = sm.btile[warp >> 3];
                float* meta = sm.meta[warp];
                if (warp < nb) {
                    float f[8];
                    if (s == 0 || st.xin) {
                        const float* xs = st.xin ? st.xin : x0;
#pragma unroll
                        for (int e = 0; e < 8; ++e) f[e] = __ldg(xs + 256 * (b0 + warp) + lane + 32 * e);
                    } else {
                        const ChainStage pv = stages[s - 1];
                        const int pn = (pv.NB + kUnitBlocks - 1) / kUnitBlocks;
                        load_tagged_block(pv.y + 256 * (b0 + warp), pn, pv.rows, epoch, lane, f);
                    }
                    if (trace && tid == 0) trace[((int64_t)cta * S + s) * 4 + 1] = globaltimer();
                    chain_rotate_block(f, L, bt, warp & 7, meta, lane);
                } else if (warp < kRecBlocks * nrec) {
                    chain_zero_block(bt, warp & 7, meta, lane);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.bready);
            }
            expander_sync();  // meta of every block visible to every expander
            if (trace && tid == 0) trace[((int64_t)cta * S + s) * 4 + 2] = globaltimer();
            const int n_units = (st.RT - 1 - sp.rt0) / sp.Gc + 1;
            for (int u = 0; u < n_units; ++u, ++useq) {
                float part = 0.f;
                for (int r = 0; r < nrec; ++r, ++rs) {
                    if (rs % kGroups != g) continue;
                    const int slot = rs % kNumSlots;
                    if (prof) c0 = clock64();
                    mbar_wait(&sm.full[slot], (unsigned)(rs / kNumSlots) & 1u);
                    if (prof) {
                        const long long c1 = clock64();
                        c_full += c1 - c0;
                        c0 = c1;
                    }
                    const uint8_t* rec = sm.ring[slot];
                    uint4 cw[4];
#pragma unroll
                    for (int c = 0; c < 4; ++c) cw[c] = reinterpret_cast<const uint4*>(rec + c * 2048)[Lr];
                    const float d = __half2float(__ushort_as_half(reinterpret_cast<const uint16_t*>(rec + kRecCodes)[Lr]));
                    const float zf = st.asym ? (float)(1 + (int)reinterpret_cast<const int8_t*>(rec + kRecCodes + 256)[Lr])
                                             : 1.f;
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&sm.empty[slot]);
                    // A columns: MMA m = 2 i + h covers elements 32 m .. 32 m + 31 = code bytes
                    // 32 h .. 32 h + 31 (words 8 h .. 8 h + 7) at bit pair i
                    uint32_t w[16];
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        w[4 * c] = cw[c].x;
                        w[4 * c + 1] = cw[c].y;
                        w[4 * c + 2] = cw[c].z;
                        w[4 * c + 3] = cw[c].w;
                    }
                    uint32_t a[64];
#pragma unroll
                    for (int m = 0; m < 8; ++m)
#pragma unroll
                        for (int c = 0; c < 8; ++c) a[8 * m + c] = w[8 * (m & 1) + c] & (0x03030303u << (2 * (m >> 1)));
                    asm volatile(
                        "tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
                        "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,"
                        "%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,"
                        "%61,%62,%63,%64};" ::"r"(ta),
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
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&sm.aready[g]);
                    if (prof) {
                        const long long c1 = clock64();
                        c_st += c1 - c0;
                        c0 = c1;
                    }
                    mbar_wait(&sm.dfull[g], (unsigned)(rs / kGroups) & 1u);
                    if (prof) c_d += clock64() - c0;
                    tc_fence_after();
                    uint32_t dv[8];
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                                 : "=r"(dv[0]), "=r"(dv[1]), "=r"(dv[2]), "=r"(dv[3]), "=r"(dv[4]), "=r"(dv[5]),
                                   "=r"(dv[6]), "=r"(dv[7])
                                 : "r"(td));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    tc_fence_before();
                    // this lane's block jb: columns 4 jb .. 4 jb + 3 = dv[4 (jb & 1) ..]
                    const int o = 4 * (jb & 1);
                    const int lo = (int)dv[o] + 256 * (int)dv[o + 1];  // |C| < 2^22: pairs stay below 2^31
                    const int hi = (int)dv[o + 2] + 256 * (int)dv[o + 3];
                    const float v = (float)hi * 65536.f + (float)lo;
                    const float* mt = sm.meta[kRecBlocks * r + jb];
                    part += d * (mt[0] * v - zf * mt[1]);
                }
                // rows r16 of blocks 2q (lanes 0-15) and 2q+1 (lanes 16-31)
                part += __shfl_xor_sync(FULL, part, 16);
                const int ps = useq % kPartSlots;
                mbar_wait(&sm.pfree[ps], ((unsigned)(useq / kPartSlots) & 1u) ^ 1u);
                if (lane < 16) sm.part[ps][warp][lane] = part;
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.pfull[ps]);
            }
            if (trace && tid == 0) trace[((int64_t)cta * S + s) * 4 + 3] = globaltimer();
            expander_sync();  // every group's MMAs of this stage completed: the B tiles may be rewritten
        }
        if (prof && lane == 0) {
            unsigned long long* pt = trace + (int64_t)G * S * 4 + (int64_t)S * 64 + warp * 4;
            pt[0] = c_full;
            pt[1] = c_st;
            pt[2] = c_d;
            pt[3] = clock64() - c_start;
        }
        (void)r16;
    }

    // fold the last stage's K-chunk partials into `out` (fixed order), waiting on the tags
    const ChainStage last = stages[S - 1];
    const int ln = (last.NB + kUnitBlocks - 1) / kUnitBlocks;
    for (int64_t r = (int64_t)cta * kChainThreads + tid; r < last.rows; r += (int64_t)G * kChainThreads) {
        float v;
        for (;;) {
            bool ok = true;
            unsigned long long w = ld_u64_relaxed(last.y + r);
            ok &= (unsigned)(w >> 32) == epoch;
            v = __uint_as_float((unsigned)w);
            for (int c = 1; c < ln; ++c) {
                w = ld_u64_relaxed(last.y + c * last.rows + r);
                ok &= (unsigned)(w >> 32) == epoch;
                v += __uint_as_float((unsigned)w);
            }
            if (ok) break;
            __nanosleep(64);
        }
        out[r] = v;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

// ------------------------------------------------------------------------------------------
// Chain layout: records [RT = ceil(rows/16)][NR = ceil(NB/8)][kRecBytes]; record (rt, kr):
//   codes  [c 0..3][L 0..127][16 B]  L = 16 j + r: row 16 rt + r, block 8 kr + j; chunk c holds
//          code bytes 16c .. 16c+15, code byte B holds elements B, 64+B, 128+B, 192+B of the
//          block at bit pairs 0..3 (value = stored code q + 1 in {0, 1, 2});
//   scales [L] f16 (0 for padding), zps [L] int8 (0 for symmetric / padding).
// Padding rows/blocks get code 0 and scale 0 (and zero activations), so they add nothing.
// ------------------------------------------------------------------------------------------
__global__ void repack_chain_kernel(const uint8_t* __restrict__ payload, int64_t rows, int NB, int RT, int NR,
                                    int asym, uint8_t* __restrict__ out) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // one thread per (record, L, byte B)
    const int64_t total = (int64_t)RT * NR * 128 * 64;
    if (idx >= total) return;
    const int B = (int)(idx & 63);
    const int Lr = (int)((idx >> 6) & 127);
    const int64_t rec = idx >> 13;
    const int kr = (int)(rec % NR);
    const int64_t rt = rec / NR;
    const int j = Lr >> 4, r = Lr & 15;
    const int64_t row = rt * 16 + r;
    const int kb = kr * kRecBlocks + j;
    uint8_t* o = out + rec * kRecBytes;
    uint8_t byte = 0;
    uint16_t sb = 0;
    int8_t z = 0;
    if (row < rows && kb < NB) {
        const uint8_t* p = payload + (row * NB + kb) * 100;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int e = 64 * i + B;
            const int c = ((p[e >> 3] >> (e & 7)) & 1) | (((p[32 + (e >> 3)] >> (e & 7)) & 1) << 1);
            byte |= (uint8_t)(c << (2 * i));
        }
        sb = *reinterpret_cast<const uint16_t*>(p + 96);
        if (asym) z = (int8_t)(int)f16_bits_to_f32(*reinterpret_cast<const uint16_t*>(p + 98));
    }
    o[(B >> 4) * 2048 + Lr * 16 + (B & 15)] = byte;
    if (B == 0) {
        *reinterpret_cast<uint16_t*>(o + kRecCodes + 2 * Lr) = sb;
        reinterpret_cast<int8_t*>(o + kRecCodes + 256)[Lr] = z;
    }
}

}  // namespace itq3

using namespace itq3;

extern "C" int64_t itq3_chain_desc_nbytes(void) { return (int64_t)sizeof(ChainStage); }
extern "C" int itq3_chain_act_block_bytes(int limbs) { return act_block_bytes(limbs); }
extern "C" int itq3_chain_smem_bytes(void) { return (int)sizeof(ChainSmem) + 1024; }

extern "C" int64_t itq3_chain_layout_nbytes(int64_t rows, int64_t cols) {
    const int64_t NB = cols / 256;
    return ((rows + 15) / 16) * ((NB + kRecBlocks - 1) / kRecBlocks) * kRecBytes;
}

extern "C" int itq3_repack_chain(const uint8_t* payload, int64_t rows, int64_t cols, int asymmetric, uint8_t* out,
                                 void* stream) {
    if (cols % 256 || rows <= 0) {
        set_error("chain layout: needs cols %% 256 == 0 and rows > 0 (got %lldx%lld)", (long long)rows,
                  (long long)cols);
        return ITQ3_E_UNSUPPORTED;
    }
    const int NB = (int)(cols / 256), RT = (int)((rows + 15) / 16), NR = (NB + kRecBlocks - 1) / kRecBlocks;
    const int64_t total = (int64_t)RT * NR * 128 * 64;
    repack_chain_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(payload, rows, NB, RT, NR,
                                                                                          asymmetric, out);
    return check_launch("itq3_repack_chain");
}

extern "C" int itq3_chain_write_desc(void* host_desc, int index, const uint8_t* tiled, void* y, const float* xin,
                                     int64_t rows, int64_t cols, int asymmetric, int reserved) {
    if (cols % 256 || cols / 256 > kMaxChainNB) {
        set_error("chain: stage %d needs cols %% 256 == 0 and cols <= %d (got %lld)", index, 256 * kMaxChainNB,
                  (long long)cols);
        return ITQ3_E_UNSUPPORTED;
    }
    ChainStage& st = reinterpret_cast<ChainStage*>(host_desc)[index];
    st.tiled = tiled;
    st.y = (unsigned long long*)y;
    st.xin = xin;
    st.rows = rows;
    st.cols = cols;
    st.NB = (int)(cols / 256);
    st.RT = (int)((rows + 15) / 16);
    st.asym = asymmetric;
    st.reserved = reserved;
    return ITQ3_OK;
}

extern "C" int itq3_chain_run(const void* d_desc, int n_stages, const float* x0, int limbs, unsigned* d_epoch,
                              float* out, int grid, void* d_trace, void* stream) {
    if (limbs < 1 || limbs > kMaxLimbs) {
        set_error("chain: limbs must be in [1, %d]", kMaxLimbs);
        return ITQ3_E_DOMAIN;
    }
    static bool attr_set = false;
    const int smem = (int)sizeof(ChainSmem) + 1024;
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
    chain_epoch_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(d_epoch);
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
                                             (const unsigned*)d_epoch, out, (unsigned long long*)d_trace);
    if (e != cudaSuccess) {
        set_error("chain: launch failed: %s", cudaGetErrorString(e));
        return ITQ3_E_CUDA;
    }
    return check_launch("itq3_chain_run");
}
