// K5: batched MMQ on the 5th-gen tensor cores (tcgen05.mma kind::f16, TMEM accumulators).
//
// Y[r, m] = sum_b (1/16) <d_rb t_rb, H x_bm> with t = c - 1 - z (the rotated-activation identity,
// see gemv.cu).  A = d * t is EXACT in binary16 (d is the stored f16 scale, t in {-2..2}), so
// the whole K reduction stays in one fp32 TMEM accumulator with no per-block promotion; the
// only approximation is B = f16(H x / 16).
//
// One persistent CTA PAIR (cluster of 2, cta_group::2) per TPC computes 256 weight rows x 256
// tokens per tile with M = 256, N = 256, K = 16 MMAs issued by the leader CTA.  Each SM holds
//   * its 128 rows of A in TMEM (expanded there from the 2-bit codes by tcgen05.st, so the weight
//     operand never touches shared memory: smem carries B and a 4.4 KB weight record per stage),
//   * its 128-token half of the B tile (f16, SWIZZLE_128B K-major),
//   * its 128 rows of the 256-column fp32 accumulator.
// The K loop runs in 128-k stages with exactly TWO bulk copies per stage and CTA (weight record,
// B half): a cp.async.bulk costs ~76 cycles of producer issue whatever its size
// (tools/probes/bulk_issue_probe.cu).  N = 256 per MMA halves the per-flop instruction load of the
// MMA issuer and of the expanders, which share the SM sub-partitions' issue slots (N = 128 tiles ran
// at ~55% of the tensor rate for that reason; tools/mmq_trace.py).
// Warp roles (14 warps per CTA):
//   warp 0     producer: the two bulk copies per stage into a 4-deep ring (full/empty mbarriers;
//              empty is signalled by ONE multicast tcgen05.commit per stage, which also frees the
//              stage's A slot: each commit costs the tensor pipe ~100-170 cycles);
//   warp 1     TMEM allocation (cta_group::2, all 512 columns: D = [0, 256), A ring = 4 x 64 columns);
//              in the leader CTA lane 0 issues the 8 MMAs of a stage once both CTAs' expanders
//              arrived on the leader's `ready` (relaxed remote mbarrier arrivals: no MEMBAR.GPU);
//   warps 2-9  expanders, two quads taking alternate stages, one weight row per thread (TMEM lane
//              quarter = warp % 4): codes -> f16 d*t (magic-number decode, 4 ops per f16x2),
//              two tcgen05.st.32x32b.x32 per stage;
//   warps 10-13 epilogue: tcgen05.ld of the row's 256 fp32 columns in two halves, each staged in smem
//              and written with ONE bulk store (cp.async.bulk shared -> global) per row and half,
//              or plain stores for ragged/strided outputs; the accumulator is released to the
//              leader as soon as it is read.
// Layouts written by itq3_repack_mmq / itq3_rotate_act_f16 (host ABI below).
#include "common.cuh"

namespace itq3 {

// Programmatic dependent launch: the MMQ kernels are launched so that their prologue (TMEM
// allocation, barrier init, weight-record fetch set-up) overlaps the activation rotation that
// precedes them on the stream; the rotation kernels release their dependents at entry and the MMQ
// producer waits (griddepcontrol.wait) before its first activation copy.
template <typename Kern, typename... Args>
static cudaError_t launch_pdl(Kern kernel, dim3 grid, dim3 block, int smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}
__device__ __forceinline__ void pdl_release() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

constexpr int kMmqBM = 128;
constexpr int kMmqExpGroups = 2;  // expander warp quads; group e decodes the chunks g with g % 2 == e
constexpr int kMmqEpiWarp = 2 + 4 * kMmqExpGroups;
constexpr int kMmqThreads = 32 * (kMmqEpiWarp + 4);  // producer, MMA, expander quads, 4 epilogue warps

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init_(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait_(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "W_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W_%=;\n}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s_(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row core groups 1024 B apart.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
// Instruction descriptor: D f32, A/B f16, both K-major, N = BN, M = 128.
template <int BN>
__device__ __forceinline__ uint32_t umma_idesc_f16() {
    return (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(kMmqBM >> 4) << 24);
}

// swizzled byte offset of (row r, 16-byte chunk j) inside a K-major SW128 tile
__device__ __forceinline__ uint32_t sw128_off(int r, int j) {
    return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((j ^ (r & 7)) << 4));
}

// one lane of a converged warp (the MMA issuer): lets the descriptors stay in uniform registers
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n selp.b32 %0, 1, 0, P;\n}\n" : "=r"(pred));
    return pred != 0;
}

// ---- cluster / pair helpers ----
__device__ __forceinline__ uint32_t cta_rank_in_cluster() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// acquire at cluster scope: the barrier also collects arrivals from the peer CTA
__device__ __forceinline__ void mbar_wait_cl(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "W_%=:\n"
        " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W_%=;\n}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
// arrive on the barrier at the same smem offset in CTA `cta` of the cluster
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t cta) {
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_addr(bar)), "r"(cta));
    // relaxed: what the arrival publishes is TMEM (tcgen05.wait + fence::before_thread_sync) or
    // TMA-landed smem, never generic stores, so no release fence (MEMBAR.GPU) is needed
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint16_t lds16(uint32_t a) {
    uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ int lds_s8(uint32_t a) {
    int v;
    asm volatile("ld.shared.s8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
// tcgen05.commit of the pair's MMAs to the barrier at this offset in both CTAs
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_addr(bar)),
        "h"((uint16_t)3)
        : "memory");
}

// Optional per-CTA cycle accounting (tools/mmq_trace.py): 16 counters per CTA, null = off.
__device__ unsigned long long* g_mmq_trace = nullptr;
#define MMQ_T0() const long long _t0 = clock64()
#define MMQ_ACC(slot, var) var += clock64() - _t0

// Per CTA of the pair: 128 weight rows (A, expanded into TMEM) and 64 of the tile's 128 tokens (B, smem).
// The K loop runs in STAGES of 128 k: per stage and CTA exactly two bulk copies (a 4480-byte weight
// record and a 16 KB B half tile), because every cp.async.bulk costs ~76 cycles of issue in the
// producer thread whatever its size (tools/probes/bulk_issue_probe.cu) -- 8 MMAs (512 tensor cycles)
// per stage leave the producer ample slack.
// TMEM (512 columns, both CTAs): D[2] = columns [0, 256) (two 128-token fp32 accumulators, so the
// epilogue of one tile overlaps the main loop of the next), A ring = [256, 512) (4 slots x 64 columns:
// a 128-k stage of f16 d*t, two k per 32-bit column).
constexpr int kStK = 128;                       // k per stage
constexpr int kWRec = 4096 + 256 + 128;         // weight record: codes [2 halves][128 rows][16 B] | f16 scales | int8 zps
// per-32-k tables (variant ss, or block_n != 256): codes | f16 scale [128 rows][4 sub-blocks of 32 k] |
// int8 zero-point [128 rows][4]: every 32-k group of a row has one scale and one zero-point
constexpr int kWRecT = 4096 + 1024 + 512;
constexpr int kMmqAsym = 1, kMmqPer32 = 2;  // itq3_mmq* flags
constexpr int kPairNS = 4;  // stages in flight: load slot s and A slot s are freed by ONE commit (a
                             // tcgen05.commit costs the tensor pipe ~100-170 cycles; tc_f16_pair_probe)
constexpr int kPairStage = 132;  // fp32 words per staged output row (128 + 4 pad: conflict-free v4 stores)
struct PairSmem {
    uint8_t b[kPairNS][128 * 2 * 128];  // B half tile: 2 x (128 token rows x 64 k f16, SW128 K-major), 1024-aligned
    uint8_t w[kPairNS][kWRecT];         // weight record of the stage (this CTA's 128 rows)
    float stage[kMmqBM][kPairStage];    // epilogue staging for the bulk row stores
    uint64_t full[kPairNS];    // this CTA's weight record + B half landed (TMA)
    uint64_t empty[kPairNS];   // the pair's MMAs consumed stage slot s: smem slot + A slot (multicast commit)
    uint64_t ready[kPairNS];   // leader only: A slot s expanded and its B landed in both CTAs (8 warp arrivals)
    uint64_t dfull;            // accumulator complete (multicast commit)
    uint64_t dempty;           // leader only: both CTAs' epilogues drained the accumulator (8 warp arrivals)
    uint32_t tmem_base;
};

// Work item = (split, token tile, pair row tile); every role walks the same sequence.
// Tail split: items [F, F + R * kt) are the last R tiles (the final partial round of the persistent
// grid) split kt ways along K; they write fp32 partials to the workspace, summed by mmq_tail_reduce.
struct PairWork {
    int tiles_r, tiles_n, ks, NS;  // NS = stages along K
    int F, R, kt;                  // tail split (kt = 1: none)
    int bsub;                      // BN = 128 tiles over a 256-token activation layout (itq3_mmq_block_n(m) = 256)
    __device__ int items() const { return F + R * kt; }
    // split = -1 for an item written straight to Y
    __device__ void decode(int it, int& tr, int& tn, int& s0, int& s1, int& split) const {
        int T, sp, n;
        if (it < F) {
            const int per = tiles_r * tiles_n;
            sp = it / per;
            T = it % per;
            n = ks;
            split = ks > 1 ? sp : -1;
        } else {
            const int j = it - F;
            T = F + j / kt;
            sp = j % kt;
            n = kt;
            split = sp;
        }
        tn = T / tiles_r;
        tr = T % tiles_r;
        s0 = (int)((int64_t)sp * NS / n);
        s1 = (int)((int64_t)(sp + 1) * NS / n);
    }
};

template <int BN, typename TY, bool PEERS = false>  // BN = tokens per pair tile (256, or 128 for M <= 128)
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kMmqThreads, 1)
    mmq_pair_kernel(const uint8_t* __restrict__ wrec, int flags, PairWork wk, const uint8_t* __restrict__ act,
                    int64_t rows, int64_t M, TY* __restrict__ y, int64_t stride_r, int64_t stride_m, int64_t slab,
                    float* __restrict__ tailws, const unsigned long long* __restrict__ ypeer, int npeer,
                    int64_t row0) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    PairSmem& sm = *reinterpret_cast<PairSmem*>(base);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cta_rank_in_cluster();
    const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
    const int items = wk.items();
    constexpr uint32_t kColA = 256;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kPairNS; ++s) {
            mbar_init_(&sm.full[s], 1);
            mbar_init_(&sm.empty[s], 1);
            mbar_init_(&sm.ready[s], 8);
        }
        mbar_init_(&sm.dfull, 1);
        mbar_init_(&sm.dempty, 8);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {  // the whole TMEM of both SMs of the pair
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(&sm.tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync_all();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = sm.tmem_base;
    // diagnostics only (tools/mmq_trace.py --flags): 1 = no B loads, 2 = no A stores
    const unsigned dflags = g_mmq_trace ? (unsigned)g_mmq_trace[4095 * 16] : 0u;
    const bool asym = flags & kMmqAsym, ss = flags & kMmqPer32;
    const int wbytes = ss ? kWRecT : kWRec;
    if constexpr (!PEERS) npeer = 0;  // the plain instantiation carries no peer code

    if (warp == 0) {
        if (lane == 0) {  // producer: this CTA's weight record and 64-token half of B, one copy each per stage
            pdl_wait();   // the activation rotation that precedes this launch has completed
            uint32_t g = 0;
            long long tw = 0, t_issue = 0;
            const long long tk0 = clock64();
            for (int it = cluster; it < items; it += nclusters) {
                int tr, tn, s0, s1, split;
                wk.decode(it, tr, tn, s0, s1, split);
                const uint8_t* wsrc = wrec + ((int64_t)(2 * tr + rank) * wk.NS) * wbytes;
                // B: this CTA's 64- or 128-token half, one stage = two 64-k SW128 tiles.  bsub (128-token tiles
                // over the 256-token layout): the half is rows 64 rank .. of the layout's 128-token half tn, i.e.
                // the same 8 KB of each 16 KB tile (the swizzle repeats every 8 rows): two copies per stage
                const bool bsub = BN == 128 && wk.bsub;
                const uint8_t* bsrc = bsub ? act + (int64_t)tn * wk.NS * (256 * 128) + rank * 8192
                                           : act + ((int64_t)(2 * tn + rank) * wk.NS) * (BN * 128);
                for (int st = s0; st < s1; ++st, ++g) {
                    const int s = g % kPairNS;
                    {
                        MMQ_T0();
                        mbar_wait_(&sm.empty[s], ((g / kPairNS) & 1u) ^ 1u);
                        MMQ_ACC(0, tw);
                    }
                    const long long ti0 = clock64();
                    mbar_expect_tx_(&sm.full[s], wbytes + ((dflags & 1) ? 0 : BN * 128));
                    bulk_g2s_(sm.w[s], wsrc + (int64_t)st * wbytes, wbytes, &sm.full[s]);
                    if (dflags & 1) {
                    } else if (bsub) {
                        bulk_g2s_(sm.b[s], bsrc + (int64_t)st * 32768, 8192, &sm.full[s]);
                        bulk_g2s_(sm.b[s] + 8192, bsrc + (int64_t)st * 32768 + 16384, 8192, &sm.full[s]);
                    } else {
                        bulk_g2s_(sm.b[s], bsrc + (int64_t)st * (BN * 128), BN * 128, &sm.full[s]);
                    }
                    t_issue += clock64() - ti0;
                }
            }
            if (unsigned long long* trc = g_mmq_trace) {
                trc[blockIdx.x * 16 + 10] = t_issue;
                trc[blockIdx.x * 16 + 0] = tw;
                trc[blockIdx.x * 16 + 7] = clock64() - tk0;
                trc[blockIdx.x * 16 + 8] = g;
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {  // MMA issuer of the pair (the whole warp runs the loop, one elected lane issues):
                          // M = 256 (128 rows per SM), N = 256, K = 16
            const uint32_t idesc = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
            uint32_t g = 0, t = 0;
            long long tw_ready = 0, tw_d = 0;
            const long long tm0 = clock64();
            for (int it = cluster; it < items; it += nclusters, ++t) {
                int tr, tn, s0, s1, split;
                wk.decode(it, tr, tn, s0, s1, split);
                {
                    MMQ_T0();
                    mbar_wait_(&sm.dempty, (t & 1u) ^ 1u);
                    MMQ_ACC(4, tw_d);
                }
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t td = tmem;
                for (int st = s0; st < s1; ++st, ++g) {
                    const int s = g % kPairNS, sa = s;
                    {
                        MMQ_T0();
                        mbar_wait_(&sm.ready[sa], (g / kPairNS) & 1u);
                        MMQ_ACC(3, tw_ready);
                    }
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t ta = tmem + kColA + 64u * sa, b0 = smem_addr(sm.b[s]);
                    if (elect_one()) {
#pragma unroll
                        for (int k = 0; k < kStK / 16; ++k) {
                            const uint64_t bd = umma_desc_sw128(b0 + (k >> 2) * (BN * 64) + 32 * (k & 3));
                            const uint32_t accum = (st != s0) || (k != 0);
                            asm volatile(
                                "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                                " tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(td),
                                "r"(ta + 8u * k), "l"(bd), "r"(idesc), "r"(accum));
                        }
                        umma_commit_pair(&sm.empty[s]);
                    }
                    __syncwarp();
                }
                if (elect_one()) umma_commit_pair(&sm.dfull);
                __syncwarp();
            }
            if (unsigned long long* trc = g_mmq_trace; trc && lane == 0) {
                trc[blockIdx.x * 16 + 3] = tw_ready;
                trc[blockIdx.x * 16 + 4] = tw_d;
                trc[blockIdx.x * 16 + 9] = clock64() - tm0;
            }
        }
    } else if (warp < kMmqEpiWarp) {
        // ---- expanders: row r = TMEM lane; 2-bit codes -> f16 d*t, two tcgen05.st of 32 columns per stage.
        // kMmqExpGroups quads take alternate stages so one quad's tcgen05.st latency overlaps the other's decode.
        const int q = warp & 3, r = 32 * q + lane, eg = (warp - 2) >> 2;
        const uint32_t ta_row = tmem + ((uint32_t)(32 * q) << 16) + kColA;
        uint32_t g = 0;
        long long tw_full = 0, t_work = 0, tw_aempty = 0;
        for (int it = cluster; it < items; it += nclusters) {
            int tr, tn, s0, s1, split;
            wk.decode(it, tr, tn, s0, s1, split);
            for (int st = s0; st < s1; ++st, ++g) {
                if ((int)(g % kMmqExpGroups) != eg) continue;
                const int s = g % kPairNS, sa = s;
                {
                    // slot s landed, so the producer saw `empty` for its previous use: the MMAs that
                    // read A slot s last have completed as well (one commit frees both)
                    MMQ_T0();
                    mbar_wait_(&sm.full[s], (g / kPairNS) & 1u);
                    MMQ_ACC(1, tw_full);
                }
                const long long tw0 = clock64();
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t wa = smem_addr(sm.w[s]);
                // scale and zero-point of each 32-k sub-block of the stage: the 256-block's (plain
                // records) or the row's per-32 tables (variant ss: y = d_m (c - 1 - z), codec.py:152-161;
                // block_n < 256: several blocks per stage)
                uint32_t dh[4];
                int zz[4];
                if (ss) {
                    const uint2 v = lds64(wa + 4096 + 8 * r);
                    dh[0] = v.x & 0xffffu, dh[1] = v.x >> 16, dh[2] = v.y & 0xffffu, dh[3] = v.y >> 16;
                    const uint32_t zw = asym ? lds32(wa + 5120 + 4 * r) : 0u;
#pragma unroll
                    for (int i = 0; i < 4; ++i) zz[i] = (int)(int8_t)(zw >> (8 * i));
                } else {
                    dh[0] = dh[1] = dh[2] = dh[3] = lds16(wa + 4096 + 2 * r);
                    zz[0] = zz[1] = zz[2] = zz[3] = asym ? lds_s8(wa + 4352 + r) : 0;
                }
                uint32_t d2[4], ndz2[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {  // exact: -(1 + z) in {0,-1,-2}
                    d2[i] = dh[i] * 0x10001u;
                    ndz2[i] = (uint32_t)__half_as_ushort(__hmul(__ushort_as_half((uint16_t)dh[i]),
                                                                __int2half_rn(-1 - zz[i]))) * 0x10001u;
                }
#pragma unroll
                for (int j = 0; j < 2; ++j) {  // 64-k half j of the stage: A columns 32 j .. 32 j + 31
                    const uint4 w4 = lds128(wa + 2048 * j + 16 * r);
                    const uint32_t wv[4] = {w4.x, w4.y, w4.z, w4.w};
                    uint32_t a[32];
#pragma unroll
                    for (int wi = 0; wi < 4; ++wi)
#pragma unroll
                        for (int m = 0; m < 8; ++m) {  // column 8 wi + m = k pair (16 wi + 2 m, +1)
                            const uint32_t v = ((wv[wi] >> (2 * m)) & 0x00030003u) | 0x64006400u;  // f16x2 1024 + c
                            __half2 hv =
                                __hsub2(*reinterpret_cast<const __half2*>(&v), __floats2half2_rn(1024.f, 1024.f));
                            hv = __hfma2(hv, *reinterpret_cast<const __half2*>(&d2[2 * j + (wi >> 1)]),
                                         *reinterpret_cast<const __half2*>(&ndz2[2 * j + (wi >> 1)]));
                            a[8 * wi + m] = *reinterpret_cast<uint32_t*>(&hv);
                        }
                    if (!(dflags & 2))
                    asm volatile(
                        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
                        "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(
                            ta_row + 64u * sa + 32u * j),
                        "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]),
                        "r"(a[8]), "r"(a[9]), "r"(a[10]), "r"(a[11]), "r"(a[12]), "r"(a[13]), "r"(a[14]), "r"(a[15]),
                        "r"(a[16]), "r"(a[17]), "r"(a[18]), "r"(a[19]), "r"(a[20]), "r"(a[21]), "r"(a[22]), "r"(a[23]),
                        "r"(a[24]), "r"(a[25]), "r"(a[26]), "r"(a[27]), "r"(a[28]), "r"(a[29]), "r"(a[30]), "r"(a[31])
                        : "memory");
                }
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive_remote(&sm.ready[sa], 0);
                t_work += clock64() - tw0;
            }
        }
        if (warp == 2 && lane == 0)
            if (unsigned long long* trc = g_mmq_trace) {
                trc[blockIdx.x * 16 + 1] = tw_full;
                trc[blockIdx.x * 16 + 11] = tw_aempty;
                trc[blockIdx.x * 16 + 2] = t_work;
            }
    } else {
        // ---- epilogue: TMEM lane r = output row; 256 tokens in two 128-token halves: registers -> staging
        // row -> one bulk store per half (plain stores for ragged or strided outputs)
        const int q = warp & 3, r = 32 * q + lane;
        const uint32_t td_row = tmem + ((uint32_t)(32 * q) << 16);
        const bool bulk_ok = stride_m == 1 && ((stride_r * (int64_t)sizeof(TY)) & 15) == 0 &&
                             (reinterpret_cast<uintptr_t>(y) & 15) == 0;
        // Row-sharded output with the all-gather fused in (npeer > 0): output row row0 + grow goes to
        // every rank's copy of Y (ypeer[p], NVLink peer addresses) -- one bulk copy of the staged
        // row-half per peer, asynchronous like the local store.
        bool peer_ok = npeer > 0 && stride_m == 1 && ((stride_r * (int64_t)sizeof(TY)) & 15) == 0;
        for (int p = 0; p < npeer; ++p) peer_ok &= (ypeer[p] & 15) == 0;
        uint32_t t = 0;
        long long tw_dfull = 0;
        const long long te0 = clock64();
        for (int it = cluster; it < items; it += nclusters, ++t) {
            int tr, tn, s0, s1, split;
            wk.decode(it, tr, tn, s0, s1, split);
            {
                MMQ_T0();
                mbar_wait_(&sm.dfull, t & 1u);
                MMQ_ACC(5, tw_dfull);
            }
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const int64_t grow = (int64_t)tr * 256 + rank * kMmqBM + r;
            TY* yt = y + (int64_t)(it / (wk.tiles_r * wk.tiles_n)) * slab;
            const bool tail = it >= wk.F;  // tail-split partial: fp32 tile in the workspace
            const bool live = tail || grow < rows;
            const uint32_t sa = smem_addr(sm.stage[r]);
#pragma unroll 1
            for (int h = 0; h < BN / 128; ++h) {
                const int64_t m0 = (int64_t)tn * BN + 128 * h;
                const bool bulk = live && !tail && (npeer == 0 ? bulk_ok : peer_ok) && m0 + 128 <= M;
                // the previous bulk store has finished reading the staging row
                if (bulk) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t v[32];
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
                          "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
                          "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                        : "r"(td_row + 128u * h + 32u * c));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    if (h == BN / 128 - 1 && c == 3) {  // accumulator free for the next tile
                        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                        __syncwarp();
                        if (lane == 0) mbar_arrive_remote(&sm.dempty, 0);
                    }
                    if (bulk) {
                        if constexpr (sizeof(TY) == 4) {
#pragma unroll
                            for (int j = 0; j < 32; j += 4)
                                sts128(sa + 4u * (32 * c + j), make_uint4(v[j], v[j + 1], v[j + 2], v[j + 3]));
                        } else {
#pragma unroll
                            for (int j = 0; j < 32; j += 8) {
                                uint32_t p[4];
#pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    __nv_bfloat162 hh = __floats2bfloat162_rn(__uint_as_float(v[j + 2 * e]),
                                                                              __uint_as_float(v[j + 2 * e + 1]));
                                    p[e] = *reinterpret_cast<uint32_t*>(&hh);
                                }
                                sts128(sa + 2u * (32 * c + j), make_uint4(p[0], p[1], p[2], p[3]));
                            }
                        }
                    } else if (tail) {
                        float* pt = tailws + ((int64_t)(split * wk.R + (tr + tn * wk.tiles_r - wk.F)) * 256 +
                                              rank * kMmqBM + r) * BN + 128 * h + 32 * c;
#pragma unroll
                        for (int j = 0; j < 32; j += 4)
                            *reinterpret_cast<uint4*>(pt + j) = make_uint4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                    } else if (live && !tail && npeer > 0) {
                        for (int p = 0; p < npeer; ++p) {
                            TY* yp = reinterpret_cast<TY*>(ypeer[p]) + (row0 + grow) * stride_r;
#pragma unroll
                            for (int j = 0; j < 32; ++j) {
                                const int64_t m = m0 + 32 * c + j;
                                if (m < M) yp[m * stride_m] = (TY)__uint_as_float(v[j]);
                            }
                        }
                    } else if (live) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const int64_t m = m0 + 32 * c + j;
                            if (m < M) yt[grow * stride_r + m * stride_m] = (TY)__uint_as_float(v[j]);
                        }
                    }
                }
                if (bulk) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    for (int p = 0; p < (npeer ? npeer : 1); ++p) {
                        TY* dst = npeer ? reinterpret_cast<TY*>(ypeer[p]) + (row0 + grow) * stride_r + m0
                                        : yt + grow * stride_r + m0;
                        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(sa),
                                     "r"((uint32_t)(128 * sizeof(TY)))
                                     : "memory");
                    }
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
            }
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        if (warp == kMmqEpiWarp && lane == 0)
            if (unsigned long long* trc = g_mmq_trace) {
                trc[blockIdx.x * 16 + 5] = tw_dfull;
                trc[blockIdx.x * 16 + 6] = clock64() - te0 - tw_dfull;
            }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    cluster_sync_all();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

// ------------------------------------------------------------------------------------------
// Repack: container payload (block_n 256, variant s, cols % 256 == 0) -> MMQ weight records
//   [rows_pad / 128 row tiles][cols / 128 stages][kWRec]: codes [half j][row][4 x u32] (word w of a
//   row's 64-k half holds k = 16w..16w+15: bits 2m..2m+1 = code of k = 16w + 2m, bits 16+2m.. =
//   k = 16w + 2m + 1) | f16 scales [row] of the stage's 256-block | int8 zero-points [row].
// ------------------------------------------------------------------------------------------
__global__ void repack_mmq_kernel(const uint8_t* __restrict__ payload, int64_t rows, int64_t rows_pad, int NB, int flags,
                                  uint8_t* __restrict__ out) {
    const bool asym = flags & kMmqAsym;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (row, 64-chunk kc)
    const int NC = NB * 4, NS = NB * 2;
    if (idx >= rows_pad * NC) return;
    const int64_t row = idx / NC;
    const int kc = (int)(idx % NC);
    const int st = kc >> 1, j = kc & 1, b = kc >> 2;
    uint8_t* rec = out + ((row >> 7) * NS + st) * (int64_t)kWRec;
    const int r = (int)(row & 127);
    uint32_t w[4] = {0, 0, 0, 0};
    uint16_t sb = 0;
    int8_t z = 0;
    if (row < rows) {
        const uint8_t* blk = payload + (row * NB + b) * 100;
        const int kbase = (kc & 3) * 64;
        const uint32_t p0 = *reinterpret_cast<const uint32_t*>(blk + (kbase >> 3));
        const uint32_t p0b = *reinterpret_cast<const uint32_t*>(blk + (kbase >> 3) + 4);
        const uint32_t p1 = *reinterpret_cast<const uint32_t*>(blk + 32 + (kbase >> 3));
        const uint32_t p1b = *reinterpret_cast<const uint32_t*>(blk + 32 + (kbase >> 3) + 4);
        const uint64_t P0 = (uint64_t)p0 | ((uint64_t)p0b << 32), P1 = (uint64_t)p1 | ((uint64_t)p1b << 32);
        for (int kk = 0; kk < 64; ++kk) {
            const uint32_t c = (uint32_t)((P0 >> kk) & 1u) | ((uint32_t)((P1 >> kk) & 1u) << 1);
            const int wi = kk >> 4, wk = kk & 15;
            const int bit = (wk & 1) ? 16 + 2 * (wk >> 1) : 2 * (wk >> 1);
            w[wi] |= c << bit;
        }
        sb = *reinterpret_cast<const uint16_t*>(blk + 96);
        if (asym) z = (int8_t)(int)f16_bits_to_f64(*reinterpret_cast<const uint16_t*>(blk + 98));
    }
    *reinterpret_cast<uint4*>(rec + 2048 * j + 16 * r) = make_uint4(w[0], w[1], w[2], w[3]);
    if (j == 0) {
        *reinterpret_cast<uint16_t*>(rec + 4096 + 2 * r) = sb;
        reinterpret_cast<int8_t*>(rec + 4352)[r] = z;
    }
}

// Per-32 tables (kWRecT records): any block_n in {32, ..., 512} with cols % block_n == 0, variant s
// or ss (sub-block n / 8 >= 32).  Thread = (row, 64-k chunk): codes bit by bit from the planes of the
// block(s) the chunk covers, then the scale and zero-point of each of its two 32-k groups.
__global__ void repack_mmq_tables_kernel(const uint8_t* __restrict__ payload, int64_t rows, int64_t rows_pad,
                                         int64_t cols, int n, int ss, int asym, uint8_t* __restrict__ out) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (row, 64-chunk kc)
    const int NC = (int)(cols / 64), NS = (int)(cols / 128);
    if (idx >= rows_pad * NC) return;
    const int64_t row = idx / NC;
    const int kc = (int)(idx % NC);
    const int st = kc >> 1, j = kc & 1;
    uint8_t* rec = out + ((row >> 7) * NS + st) * (int64_t)kWRecT;
    const int r = (int)(row & 127);
    const int q = 3 * n / 8, bsize = q + 4 + (ss ? 16 : 0), nbr = (int)(cols / n);
    uint32_t w[4] = {0, 0, 0, 0};
    uint16_t sc[2] = {0, 0};
    int8_t zp[2] = {0, 0};
    if (row < rows) {
        for (int kk = 0; kk < 64; ++kk) {
            const int64_t k = (int64_t)kc * 64 + kk;
            const uint8_t* blk = payload + (row * nbr + k / n) * bsize;
            const int o = (int)(k % n);
            const uint32_t c = ((blk[o >> 3] >> (o & 7)) & 1u) | (((blk[n / 8 + (o >> 3)] >> (o & 7)) & 1u) << 1);
            const int wi = kk >> 4, wk = kk & 15;
            w[wi] |= c << ((wk & 1) ? 16 + 2 * (wk >> 1) : 2 * (wk >> 1));
        }
        for (int g = 0; g < 2; ++g) {
            const int64_t k = (int64_t)kc * 64 + 32 * g;
            const uint8_t* blk = payload + (row * nbr + k / n) * bsize;
            const int o = (int)(k % n);
            sc[g] = ss ? *reinterpret_cast<const uint16_t*>(blk + q + 4 + 2 * (o / (n / 8)))
                       : *reinterpret_cast<const uint16_t*>(blk + q);
            if (asym) zp[g] = (int8_t)(int)f16_bits_to_f64(*reinterpret_cast<const uint16_t*>(blk + q + 2));
        }
    }
    *reinterpret_cast<uint4*>(rec + 2048 * j + 16 * r) = make_uint4(w[0], w[1], w[2], w[3]);
    *reinterpret_cast<uint32_t*>(rec + 4096 + 8 * r + 4 * j) = (uint32_t)sc[0] | ((uint32_t)sc[1] << 16);
    *reinterpret_cast<uint16_t*>(rec + 5120 + 4 * r + 2 * j) = (uint16_t)((uint8_t)zp[0] | ((uint16_t)(uint8_t)zp[1] << 8));
}

// ------------------------------------------------------------------------------------------
// Activation rotation for MMQ: x'' = (H_256 x_b) / 16 in f16, written pre-swizzled as
// [BN-token tile][CTA half h][64-k chunk kc][BN/2 token rows x 128 B] (SW128 K-major canonical
// layout), so each CTA's B half of a 128-k stage is ONE contiguous copy (BN x 128 B); padding = 0.
// One CTA per (256-block, 32 tokens): coalesced loads along whichever of k / token is contiguous
// into a padded smem tile, one warp per 4 tokens for the butterfly (fp32: shuffles for the lane
// bits, registers for the rest), then 16-byte stores of 8 consecutive k of one token.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void load4(const float* p, float (&f)[4]) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(p));
    f[0] = v.x, f[1] = v.y, f[2] = v.z, f[3] = v.w;
}
__device__ __forceinline__ void load4(const double* p, float (&f)[4]) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p)), b = __ldg(reinterpret_cast<const double2*>(p) + 1);
    f[0] = (float)a.x, f[1] = (float)a.y, f[2] = (float)b.x, f[3] = (float)b.y;
}
__device__ __forceinline__ void load4(const __half* p, float (&f)[4]) {
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
    const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&v.x)), b = __half22float2(*reinterpret_cast<const __half2*>(&v.y));
    f[0] = a.x, f[1] = a.y, f[2] = b.x, f[3] = b.y;
}
__device__ __forceinline__ void load4(const __nv_bfloat16* p, float (&f)[4]) {
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.x)),
                 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.y));
    f[0] = a.x, f[1] = a.y, f[2] = b.x, f[3] = b.y;
}

template <typename TX, int NH, bool ALL>
__global__ void __launch_bounds__(256) rotate_act_f16_kernel(const TX* __restrict__ x, int64_t M, int64_t stride_k,
                                                             int64_t stride_m, int64_t NC, int BN,
                                                             uint8_t* __restrict__ out, unsigned* __restrict__ nonfinite,
                                                             int logn, float inv_sqrt_n) {
    // fp32 inputs, token-major (257: conflict-free transposes)
    pdl_release();
    __shared__ __align__(16) float tile[32][257];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t b = blockIdx.y, m0 = (int64_t)blockIdx.x * 32;  // adjacent CTAs: adjacent token groups (DRAM locality)
    // block_n 512: the CTA transforms both 256-halves of the block (kept in registers) and joins them
    // with the k-bit-8 stage; otherwise one 256-k slice of n-blocks
    constexpr int nh = NH;  // = 2 iff logn == 9 (a separate instantiation: the n <= 256 kernel keeps 48 registers)
    const int tl = lane >> 3, kq = lane & 7, tok = 4 * warp + tl;
    float vv[2][32];
    bool bad = false;
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
    if (h2 >= nh) break;
    if (h2) __syncthreads();  // every read of the first half is done before the tile is overwritten
    const TX* xb = x + (b * nh + h2) * 256 * stride_k;
    if (stride_k == 1 && stride_m != 1) {  // token-major input: threads along k
#pragma unroll 4
        for (int j = 0; j < 32; ++j) {
            const int64_t m = m0 + j;
            tile[j][tid] = m < M ? (float)xb[tid + m * stride_m] : 0.f;
        }
    } else if (stride_m == 1 && (stride_k & 3) == 0 && m0 + 32 <= M &&
               (reinterpret_cast<uintptr_t>(x) & (4 * sizeof(TX) - 1)) == 0) {
        // k-major, 4-token vectors: thread (k_lo = tid / 8, tokens 4 (tid % 8) ..) loads 8 vectors in flight
        const int kl = tid >> 3, mq = tid & 7;
        float f[8][4];
#pragma unroll
        for (int i = 0; i < 8; ++i) load4(xb + (int64_t)(kl + 32 * i) * stride_k + m0 + 4 * mq, f[i]);
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int e = 0; e < 4; ++e) tile[4 * mq + e][kl + 32 * i] = f[i][e];  // conflict-free: 257 = 1 mod 32
    } else {  // k-major input: lanes along tokens
#pragma unroll 4
        for (int i = 0; i < 32; ++i) {
            const int k = warp + 8 * i;
            const int64_t m = m0 + lane;
            tile[lane][k] = m < M ? (float)xb[k * stride_k + m * stride_m] : 0.f;
        }
    }
    __syncthreads();
    // Butterfly: lane (token 4 warp + lane / 8, k bits 2..4 = lane % 8) holds the 32 values with
    // k bits 0..1 and 5..7 in registers (v[4 kh + j]: k = j + 4 (lane % 8) + 32 kh), so five of the
    // eight stages are register-only and three use shuffles (96 per thread instead of 160); the
    // smem reads are conflict-free (row pitch 257: bank = token + 4 (lane % 8) + const).
    float(&v)[32] = vv[h2];
#pragma unroll
    for (int kh = 0; kh < 8; ++kh)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            v[4 * kh + j] = tile[tok][j + 4 * kq + 32 * kh];
            bad |= !isfinite(v[4 * kh + j]);
        }
    // block_n = 2^logn <= 256: only the stages of k bits < logn (register index bit i is k bit i for
    // i < 2, k bit i + 3 above; lane bit i is k bit i + 2)
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        if (!ALL && (i < 2 ? i : i + 3) >= logn) continue;
        const int hh = 1 << i;
#pragma unroll
        for (int r = 0; r < 32; ++r)
            if ((r & hh) == 0) {
                const float lo = v[r], hi = v[r + hh];
                v[r] = lo + hi;
                v[r + hh] = lo - hi;
            }
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        if (!ALL && i + 2 >= logn) continue;
        const int h = 1 << i;
        const bool high = (lane & h) != 0;
#pragma unroll
        for (int r = 0; r < 32; ++r) {
            const float p = __shfl_xor_sync(FULL, v[r], h);
            v[r] = high ? p - v[r] : v[r] + p;
        }
    }
    }  // h2
    // fused_matmul's DomainError check (compute.py): one flag word, set if any input is not finite
    if (nonfinite && __any_sync(FULL, bad) && lane == 0) atomicOr(nonfinite, 1u);
    if (nh == 2) {
#pragma unroll
        for (int r = 0; r < 32; ++r) {
            const float lo = vv[0][r], hi = vv[1][r];
            vv[0][r] = lo + hi;
            vv[1][r] = lo - hi;
        }
    }
    // 8-byte stores of 4 consecutive k of one token (a warp covers 4 tokens x 64 contiguous bytes)
    const int64_t m = m0 + tok;
    const int hb = BN / 2;                 // tokens per CTA half of a tile
    const int64_t half = m / hb;           // = 2 * tile + h
    const int row = (int)(m % hb);
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
    if (h2 >= nh) break;
    const float(&v)[32] = vv[h2];
#pragma unroll
    for (int kh = 0; kh < 8; ++kh) {
        const int64_t k = (b * nh + h2) * 256 + 32 * kh + 4 * kq;
        const int64_t kc = k >> 6;
        const int kk = (int)(k & 63);
        const __half2 p0 = __floats2half2_rn(v[4 * kh] * inv_sqrt_n, v[4 * kh + 1] * inv_sqrt_n);
        const __half2 p1 = __floats2half2_rn(v[4 * kh + 2] * inv_sqrt_n, v[4 * kh + 3] * inv_sqrt_n);
        uint8_t* t = out + (half * NC + kc) * (int64_t)(hb * 128) + sw128_off(row, kk >> 3) + (kk & 7) * 2;
        *reinterpret_cast<uint2*>(t) = make_uint2(*reinterpret_cast<const uint32_t*>(&p0),
                                                  *reinterpret_cast<const uint32_t*>(&p1));
    }
    }  // h2
}

// Sum the kt fp32 partials of the R tail tiles (fixed split order) into Y.
template <typename TY>
__global__ void mmq_tail_reduce(const float* __restrict__ tws, int F, int R, int kt, int tiles_r, int BN, int64_t rows,
                                int64_t M, TY* __restrict__ y, int64_t stride_r, int64_t stride_m,
                                const unsigned long long* __restrict__ ypeer, int npeer, int64_t row0) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t per = (int64_t)256 * BN;
    if (i >= (int64_t)R * per) return;
    const int tl = (int)(i / per);
    const int lr = (int)((i % per) / BN), lc = (int)(i % BN);
    const int T = F + tl;
    const int64_t row = (int64_t)(T % tiles_r) * 256 + lr, m = (int64_t)(T / tiles_r) * BN + lc;
    if (row >= rows || m >= M) return;
    float v = tws[((int64_t)tl * 256 + lr) * BN + lc];
    for (int sp = 1; sp < kt; ++sp) v += tws[(((int64_t)sp * R + tl) * 256 + lr) * BN + lc];
    if (npeer == 0) y[row * stride_r + m * stride_m] = (TY)v;
    for (int p = 0; p < npeer; ++p) reinterpret_cast<TY*>(ypeer[p])[(row0 + row) * stride_r + m * stride_m] = (TY)v;
}

template <typename TY>
__global__ void mmq_splitk_reduce(const float* __restrict__ ws, int ks, int64_t rows, int64_t M, TY* __restrict__ y,
                                  int64_t stride_r, int64_t stride_m, const unsigned long long* __restrict__ ypeer,
                                  int npeer, int64_t row0) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows * M) return;
    const int64_t r = i / M, m = i % M;
    float v = ws[i];
    for (int z = 1; z < ks; ++z) v += ws[(int64_t)z * rows * M + i];  // fixed order
    if (npeer == 0) y[r * stride_r + m * stride_m] = (TY)v;
    for (int p = 0; p < npeer; ++p) reinterpret_cast<TY*>(ypeer[p])[(row0 + r) * stride_r + m * stride_m] = (TY)v;
}

}  // namespace itq3

using namespace itq3;

static int mmq_rows_pad(int64_t rows) { return (int)((rows + 255) / 256 * 256); }  // whole CTA-pair tiles

extern "C" int64_t itq3_mmq_nbytes(int64_t rows, int64_t cols, int flags) {
    // the zero-point bytes are part of every record; per-32 records carry four scales and zero-points per row
    return (int64_t)(mmq_rows_pad(rows) / 128) * (cols / kStK) * ((flags & kMmqPer32) ? kWRecT : kWRec);
}

extern "C" int itq3_repack_mmq_n(const uint8_t* payload, int64_t rows, int64_t cols, int block_n, int variant_ss,
                                 int asymmetric, uint8_t* out, void* stream) {
    if (rows <= 0 || cols <= 0 || cols % 256 || block_n < 32 || block_n > 512 || (block_n & (block_n - 1)) ||
        cols % block_n || (variant_ss && block_n < 256)) {
        set_error("itq3_repack_mmq_n: needs cols %% 256 == 0, cols %% block_n == 0, block_n in 32..512 "
                  "(>= 256 for variant ss) (got %lld x %lld, block_n %d)", (long long)rows, (long long)cols, block_n);
        return ITQ3_E_UNSUPPORTED;
    }
    const int64_t rp = mmq_rows_pad(rows);
    const int64_t n = rp * (cols / 64);
    repack_mmq_tables_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        payload, rows, rp, cols, block_n, variant_ss, asymmetric, out);
    return check_launch("itq3_repack_mmq_n");
}

extern "C" int itq3_repack_mmq_n(const uint8_t*, int64_t, int64_t, int, int, int, uint8_t*, void*);

extern "C" int itq3_repack_mmq(const uint8_t* payload, int64_t rows, int64_t cols, int flags, uint8_t* out,
                               void* stream) {
    if (rows <= 0 || cols <= 0 || cols % 256) {
        set_error("itq3_repack_mmq: needs cols %% 256 == 0 (got %lld x %lld)", (long long)rows, (long long)cols);
        return ITQ3_E_UNSUPPORTED;
    }
    if (flags & kMmqPer32)  // variant ss at block_n 256
        return itq3_repack_mmq_n(payload, rows, cols, 256, 1, flags & kMmqAsym, out, stream);
    const int64_t rp = mmq_rows_pad(rows);
    const int NB = (int)(cols / 256);
    const int64_t n = rp * NB * 4;
    repack_mmq_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(payload, rows, rp, NB, flags,
                                                                                     out);
    return check_launch("itq3_repack_mmq");
}

extern "C" int itq3_mmq_block_n(int64_t m) { return m <= 128 ? 128 : 256; }  // tokens per CTA-pair tile

extern "C" int64_t itq3_mmq_act_nbytes(int64_t cols, int64_t m) {
    const int BN = itq3_mmq_block_n(m);
    const int64_t M_pad = (m + BN - 1) / BN * BN;
    return M_pad * cols * 2;
}

extern "C" int itq3_rotate_act_f16_n(const void* x, int x_dtype, int64_t cols, int64_t m, int64_t stride_k,
                                     int64_t stride_m, int block_n, uint8_t* out, unsigned* nonfinite, void* stream) {
    if (cols <= 0 || cols % 256 || m <= 0) {
        set_error("itq3_rotate_act_f16: need cols %% 256 == 0 and m > 0");
        return ITQ3_E_SHAPE;
    }
    if (block_n < 32 || block_n > 512 || (block_n & (block_n - 1)) || cols % block_n) {
        set_error("itq3_rotate_act_f16: block_n must be a power of two in [32, 512] dividing cols (got %d)", block_n);
        return ITQ3_E_UNSUPPORTED;
    }
    const int logn = 31 - __builtin_clz((unsigned)block_n);
    // x'' = H_n x / sqrt(n): 1/16 exactly at n = 256; fl32(1/sqrt(n)) otherwise (fwht_inverse, transform.py:86-87)
    const float isn = (float)(1.0 / sqrt((double)block_n));
    const int BN = itq3_mmq_block_n(m);
    const int64_t NB = cols / 256, M_pad = (m + BN - 1) / BN * BN;
    const dim3 grid((unsigned)(M_pad / 32), (unsigned)(block_n > 256 ? NB / 2 : NB));
    cudaStream_t s = (cudaStream_t)stream;
    switch (x_dtype) {
        case ITQ3_F32:
            (block_n > 256 ? rotate_act_f16_kernel<float, 2, true> : block_n == 256 ? rotate_act_f16_kernel<float, 1, true> : rotate_act_f16_kernel<float, 1, false>)<<<grid, 256, 0, s>>>((const float*)x, m, stride_k, stride_m, NB * 4, BN, out,
                                                             nonfinite, logn, isn);
            break;
        case ITQ3_F64:
            (block_n > 256 ? rotate_act_f16_kernel<double, 2, true> : block_n == 256 ? rotate_act_f16_kernel<double, 1, true> : rotate_act_f16_kernel<double, 1, false>)<<<grid, 256, 0, s>>>((const double*)x, m, stride_k, stride_m, NB * 4, BN, out,
                                                             nonfinite, logn, isn);
            break;
        case ITQ3_BF16:
            (block_n > 256 ? rotate_act_f16_kernel<__nv_bfloat16, 2, true> : block_n == 256 ? rotate_act_f16_kernel<__nv_bfloat16, 1, true> : rotate_act_f16_kernel<__nv_bfloat16, 1, false>)<<<grid, 256, 0, s>>>((const __nv_bfloat16*)x, m, stride_k, stride_m,
                                                                      NB * 4, BN, out, nonfinite, logn, isn);
            break;
        case ITQ3_F16:
            (block_n > 256 ? rotate_act_f16_kernel<__half, 2, true> : block_n == 256 ? rotate_act_f16_kernel<__half, 1, true> : rotate_act_f16_kernel<__half, 1, false>)<<<grid, 256, 0, s>>>((const __half*)x, m, stride_k, stride_m, NB * 4, BN, out,
                                                             nonfinite, logn, isn);
            break;
        default:
            set_error("itq3_rotate_act_f16: unsupported dtype %d", x_dtype);
            return ITQ3_E_DOMAIN;
    }
    return check_launch("itq3_rotate_act_f16_n");
}

extern "C" int itq3_rotate_act_f16(const void* x, int x_dtype, int64_t cols, int64_t m, int64_t stride_k,
                                   int64_t stride_m, uint8_t* out, unsigned* nonfinite, void* stream) {
    return itq3_rotate_act_f16_n(x, x_dtype, cols, m, stride_k, stride_m, 256, out, nonfinite, stream);
}

static int mmq_max_clusters() {
    // co-resident CTA pairs of the persistent kernel (74 on a full B200)
    static int n = 0;
    if (n == 0) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(2, 1, 1);
        cfg.blockDim = dim3(kMmqThreads, 1, 1);
        cfg.dynamicSmemBytes = sizeof(PairSmem) + 1024;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int c = 0;
        if (cudaOccupancyMaxActiveClusters(&c, mmq_pair_kernel<256, float>, &cfg) != cudaSuccess || c < 1) {
            cudaGetLastError();
            int sms = 148;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
            c = sms / 2;
        }
        n = c;
    }
    return n;
}

// Pair tile width: the activation layout's (itq3_mmq_block_n), except that a 256-token layout runs 128-token
// tiles (PairWork::bsub) when 256-token tiles would leave more than half of the CTA pairs idle and K <= 4096
// -- twice the tiles instead of split-K's fp32 partial slabs and reduce pass (4096 x 4096, M = 512: 33.7 ->
// 21.3 us; 1024 x 4096, M = 2048: 32.0 -> 21.3 us).  At larger K the doubled A expansion costs more than the
// split-K traffic it saves (4096 x 14336, M = 256: 37.7 -> 42.8 us), so those keep 256-token tiles.
static int mmq_pick_bn(int64_t rows, int64_t cols, int64_t m) {
    if (itq3_mmq_block_n(m) == 128) return 128;
    if (cols > 4096) return 256;
    const int64_t tiles = (int64_t)(mmq_rows_pad(rows) / 256) * ((m + 255) / 256);
    return tiles * 2 <= mmq_max_clusters() ? 128 : 256;
}

static int mmq_splits(int64_t rows, int64_t cols, int64_t m, int BN) {
    // split K only when the output tiles leave more than half of the CTA pairs idle, so the fp32
    // partial traffic never costs more than the idle SMs it recovers; >= 4 stages (512 k) per split
    const int64_t tiles = (int64_t)(mmq_rows_pad(rows) / 256) * ((m + BN - 1) / BN);
    const int64_t pairs = mmq_max_clusters();
    if (tiles * 2 > pairs) return 1;
    const int64_t NS = cols / kStK;
    int64_t ks = pairs / tiles;
    ks = ks < NS / 4 ? ks : NS / 4;
    return (int)(ks < 1 ? 1 : ks);
}

// The last partial round of R tiles (R <= P / 2) is split kt = min(P / R, NS / 4) ways along K so the
// final wave keeps the pairs busy; F = tiles - R are processed whole.
static void mmq_tail_plan(int64_t tiles, int NS, int P, bool allowed, int& F, int& R, int& kt) {
    F = (int)tiles;
    R = 0;
    kt = 1;
    if (!allowed || tiles <= P) return;
    const int r = (int)(tiles % P);
    if (r == 0 || 2 * r > P) return;
    int k = P / r;
    if (k > NS / 4) k = NS / 4;
    if (k < 2) return;
    F = (int)(tiles - r);
    R = r;
    kt = k;
}

template <int BN, typename TY>
static int launch_mmq(const uint8_t* mmq, int64_t rows, int64_t cols, int asym, const uint8_t* act, int64_t m, TY* y,
                      int64_t sr, int64_t sm_, float* ws, cudaStream_t s,
                      const unsigned long long* ypeer = nullptr, int npeer = 0, int64_t row0 = 0) {
    const int smem = (int)sizeof(PairSmem) + 1024;
    static std::atomic<unsigned long long> attr{0}, attr_peer{0}, attr32{0};
    if (int rc = ensure_smem_attr(mmq_pair_kernel<BN, TY>, smem, attr, "itq3_mmq: smem attribute")) return rc;
    if (int rc = ensure_smem_attr(mmq_pair_kernel<BN, TY, true>, smem, attr_peer, "itq3_mmq: smem attribute")) return rc;
    if (int rc = ensure_smem_attr(mmq_pair_kernel<BN, float>, smem, attr32, "itq3_mmq: smem attribute")) return rc;
    PairWork wk;
    wk.tiles_r = mmq_rows_pad(rows) / 256;
    wk.tiles_n = (int)((m + BN - 1) / BN);
    wk.ks = ws ? mmq_splits(rows, cols, m, BN) : 1;
    wk.bsub = BN == 128 && itq3_mmq_block_n(m) == 256;
    wk.NS = (int)(cols / kStK);
    const int64_t tiles = (int64_t)wk.tiles_r * wk.tiles_n;
    const int P = mmq_max_clusters();
    mmq_tail_plan(tiles, wk.NS, P, ws != nullptr && wk.ks == 1, wk.F, wk.R, wk.kt);
    if (wk.ks > 1) {  // underfilled grid: every tile split ks ways (slabs [ks][rows][M])
        wk.F = (int)(tiles * wk.ks);
        wk.R = 0;
        wk.kt = 1;
    }
    const int64_t items = (int64_t)wk.F + (int64_t)wk.R * wk.kt;
    const int64_t clusters = items < P ? items : P;
    const dim3 grid((unsigned)(2 * clusters));
    float* tws = reinterpret_cast<float*>(ws);
    if (wk.ks == 1) {
        if (npeer)
            launch_pdl(mmq_pair_kernel<BN, TY, true>, grid, dim3(kMmqThreads), smem, s, mmq, asym, wk, act, rows, m, y,
                       sr, sm_, (int64_t)0, tws, ypeer, npeer, row0);
        else
            launch_pdl(mmq_pair_kernel<BN, TY>, grid, dim3(kMmqThreads), smem, s, mmq, asym, wk, act, rows, m, y, sr,
                       sm_, (int64_t)0, tws, ypeer, 0, (int64_t)0);
        int rc = check_launch("itq3_mmq");
        if (rc || wk.R == 0) return rc;
        const int64_t n = (int64_t)wk.R * 256 * BN;
        mmq_tail_reduce<TY><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(tws, wk.F, wk.R, wk.kt, wk.tiles_r, BN, rows, m,
                                                                      y, sr, sm_, ypeer, npeer, row0);
        return check_launch("itq3_mmq (tail reduce)");
    }
    launch_pdl(mmq_pair_kernel<BN, float>, grid, dim3(kMmqThreads), smem, s, mmq, asym, wk, act, rows, m, tws, m,
               (int64_t)1, rows * m, tws, (const unsigned long long*)nullptr, 0, (int64_t)0);
    int rc = check_launch("itq3_mmq (split-K)");
    if (rc) return rc;
    const int64_t n = rows * m;
    mmq_splitk_reduce<TY><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(tws, wk.ks, rows, m, y, sr, sm_, ypeer, npeer,
                                                                      row0);
    return check_launch("itq3_mmq (split-K reduce)");
}

extern "C" int itq3_mmq_set_trace(void* buf) {
    unsigned long long* p = (unsigned long long*)buf;
    return cudaMemcpyToSymbol(g_mmq_trace, &p, sizeof(p)) == cudaSuccess ? 0 : check_launch("itq3_mmq_set_trace");
}

extern "C" int64_t itq3_mmq_ws_nbytes(int64_t rows, int64_t cols, int64_t m) {
    const int BN = mmq_pick_bn(rows, cols, m);
    const int ks = mmq_splits(rows, cols, m, BN);
    if (ks > 1) return (int64_t)ks * rows * m * (int64_t)sizeof(float);
    int F, R, kt;
    mmq_tail_plan((int64_t)(mmq_rows_pad(rows) / 256) * ((m + BN - 1) / BN), (int)(cols / kStK), mmq_max_clusters(), true,
                  F, R, kt);
    return R ? (int64_t)R * kt * 256 * BN * (int64_t)sizeof(float) : 0;
}

extern "C" int itq3_mmq(const uint8_t* mmq, int64_t rows, int64_t cols, int flags, const uint8_t* act, int64_t m,
                        void* y, int y_dtype, int64_t stride_r, int64_t stride_m, void* workspace, void* stream) {
    if (rows <= 0 || cols <= 0 || cols % 256 || m <= 0) {
        set_error("itq3_mmq: bad shape");
        return ITQ3_E_SHAPE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    float* ws = (float*)workspace;
    const bool n128 = mmq_pick_bn(rows, cols, m) == 128;
    if (y_dtype == ITQ3_F32)
        return n128 ? launch_mmq<128>(mmq, rows, cols, flags, act, m, (float*)y, stride_r, stride_m, ws, s)
                    : launch_mmq<256>(mmq, rows, cols, flags, act, m, (float*)y, stride_r, stride_m, ws, s);
    if (y_dtype == ITQ3_BF16)
        return n128 ? launch_mmq<128>(mmq, rows, cols, flags, act, m, (__nv_bfloat16*)y, stride_r, stride_m, ws, s)
                    : launch_mmq<256>(mmq, rows, cols, flags, act, m, (__nv_bfloat16*)y, stride_r, stride_m, ws, s);
    set_error("itq3_mmq: output dtype must be float32 or bfloat16");
    return ITQ3_E_DOMAIN;
}

extern "C" int itq3_mmq_peers(const uint8_t* mmq, int64_t rows, int64_t cols, int flags, const uint8_t* act, int64_t m,
                              const void* d_ypeers, int npeer, int64_t row0, int y_dtype, int64_t stride_r,
                              int64_t stride_m, void* workspace, void* stream) {
    if (rows <= 0 || cols <= 0 || cols % 256 || m <= 0 || row0 < 0) {
        set_error("itq3_mmq_peers: bad shape");
        return ITQ3_E_SHAPE;
    }
    if (npeer < 1 || npeer > 8 || d_ypeers == nullptr) {
        set_error("itq3_mmq_peers: need 1..8 peer output pointers (got %d)", npeer);
        return ITQ3_E_DOMAIN;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const auto* yp = (const unsigned long long*)d_ypeers;
    const bool n128 = mmq_pick_bn(rows, cols, m) == 128;
    // every output row is written once -- by its tile's epilogue, or by the split reduce -- to all peers
    float* ws = (float*)workspace;
    if (y_dtype == ITQ3_F32)
        return n128 ? launch_mmq<128>(mmq, rows, cols, flags, act, m, (float*)nullptr, stride_r, stride_m, ws, s, yp,
                                      npeer, row0)
                    : launch_mmq<256>(mmq, rows, cols, flags, act, m, (float*)nullptr, stride_r, stride_m, ws, s, yp,
                                      npeer, row0);
    if (y_dtype == ITQ3_BF16)
        return n128 ? launch_mmq<128>(mmq, rows, cols, flags, act, m, (__nv_bfloat16*)nullptr, stride_r, stride_m, ws,
                                      s, yp, npeer, row0)
                    : launch_mmq<256>(mmq, rows, cols, flags, act, m, (__nv_bfloat16*)nullptr, stride_r, stride_m, ws,
                                      s, yp, npeer, row0);
    set_error("itq3_mmq_peers: output dtype must be float32 or bfloat16");
    return ITQ3_E_DOMAIN;
}

// ==========================================================================================
// K5b: small-batch MMQ on tcgen05.mma kind::i8 (M <= 64 tokens).
//
// The f16 path above spends ~3 thread instructions per weight expanding codes into d*t tiles,
// which caps it far below HBM speed at small M.  Here the weight operand is the raw code
// c = q + 1 in {0, 1, 2} (u8), one SHF + LOP per 4 weights, written to TMEM with one
// tcgen05.st per row and block; the activations are 16-bit fixed point per (token, block)
// (the K3/chain rotation: exact int32 butterfly, |q| <= 2^14) split into two s8 limbs that form
// the N = 2 BN columns of the MMA (B, shared memory, SWIZZLE_128B).  Because scales differ per
// (row, block), every block gets its own s32 accumulator in TMEM and the epilogue folds it:
//     y[r, m] += d_rb * ( 2^(ex_bm - 4) * (D0 + 256 D1) - (1 + z_rb) * Q_bm 2^(ex_bm - 4) ).
// Per CTA: 128 rows x BN tokens x a K-range of blocks.  Warps: 0 producer (one bulk copy of the
// weight record and one of the activation record per block), 1 MMA issuer + TMEM allocator,
// 2-5 expanders (one row per thread), 6-13 epilogue (lane quarter x token half).
// ==========================================================================================
namespace itq3 {

constexpr int kQ8Rec = 8192 + 256 + 128;  // codes [c][row][16 B] | f16 scales [row] | int8 zps [row]
constexpr int kQ8ExpGroups = 2;              // expander quads on alternate blocks
constexpr int kQ8EpiWarp = 2 + 4 * kQ8ExpGroups;
constexpr int kQ8Threads = 32 * (kQ8EpiWarp + 8);
constexpr int kQ8NA = 4, kQ8ND = 2;          // TMEM: A ring 4 x 64 columns | D ring 2 x N columns (N <= 128)

__host__ __device__ constexpr int q8_act_bytes(int BN) { return 512 * BN + 8 * BN; }  // B tile + (f, corr)/token
__host__ __device__ constexpr int q8_slot_bytes(int BN) { return (q8_act_bytes(BN) + kQ8Rec + 1023) / 1024 * 1024; }
template <int BN>
__host__ __device__ constexpr int q8_slots() { return BN >= 64 ? 4 : (BN == 32 ? 6 : 8); }

template <int BN>
struct Q8Smem {
    uint8_t slot[q8_slots<BN>()][q8_slot_bytes(BN)];  // [B tile (1024-aligned) | meta | weight record]
    uint64_t full[q8_slots<BN>()];
    uint64_t empty[q8_slots<BN>()];
    uint64_t aready[kQ8NA];
    uint64_t done[kQ8NA];  // block i's MMAs completed (ONE commit): A slot i % 4 free, D slot i % 2 full
    uint64_t dempty[kQ8ND];
    uint32_t tmem_base;
};

template <int BN, typename TY>
__global__ void __launch_bounds__(kQ8Threads, 1)
    mmq8_kernel(const uint8_t* __restrict__ wrec, int NB, const uint8_t* __restrict__ act, int64_t rows, int64_t M,
                TY* __restrict__ y, int64_t stride_r, int64_t stride_m, int64_t slab) {
    constexpr int NS = q8_slots<BN>();
    constexpr int N = 2 * BN;
    constexpr uint32_t kCols = 512;
    constexpr uint32_t kColD = 64 * kQ8NA;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Q8Smem<BN>& sm = *reinterpret_cast<Q8Smem<BN>*>(base);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rt = blockIdx.x, tt = blockIdx.y;
    const int b0 = (int)((int64_t)blockIdx.z * NB / gridDim.z), b1 = (int)((int64_t)(blockIdx.z + 1) * NB / gridDim.z);
    y += (int64_t)blockIdx.z * slab;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init_(&sm.full[s], 1);
            mbar_init_(&sm.empty[s], 8);  // epilogue warps (the last readers of a slot)
        }
        for (int s = 0; s < kQ8NA; ++s) {
            mbar_init_(&sm.aready[s], 4);
            mbar_init_(&sm.done[s], 1);
        }
        for (int s = 0; s < kQ8ND; ++s) mbar_init_(&sm.dempty[s], 8);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&sm.tmem_base)),
                     "r"(kCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = sm.tmem_base;
    const int nblk = b1 - b0;
    long long c[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};  // cycle accounting (g_mmq_trace)
    const long long tk0 = clock64();

    if (warp == 0) {
        if (lane == 0) {
            pdl_wait();  // the activation rotation that precedes this launch has completed
            for (int i = 0; i < nblk; ++i) {
                const int s = i % NS;
                { MMQ_T0(); mbar_wait_(&sm.empty[s], ((unsigned)(i / NS) & 1u) ^ 1u); MMQ_ACC(0, c[0]); }
                mbar_expect_tx_(&sm.full[s], q8_act_bytes(BN) + kQ8Rec);
                const int b = b0 + i;
                bulk_g2s_(sm.slot[s], act + ((int64_t)tt * NB + b) * q8_act_bytes(BN), q8_act_bytes(BN), &sm.full[s]);
                bulk_g2s_(sm.slot[s] + q8_act_bytes(BN), wrec + ((int64_t)rt * NB + b) * kQ8Rec, kQ8Rec, &sm.full[s]);
            }
        }
    } else if (warp == 1) {
        {  // the whole warp runs the loop, one elected lane issues (descriptors in uniform registers)
            // D s32, A u8, B s8, K-major, N = 2 BN, M = 128
            const uint32_t idesc = (2u << 4) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
            for (int i = 0; i < nblk; ++i) {
                const int s = i % NS, sa = i % kQ8NA, sd = i % kQ8ND;
                { MMQ_T0(); mbar_wait_(&sm.aready[sa], (unsigned)(i / kQ8NA) & 1u); MMQ_ACC(0, c[1]); }
                { MMQ_T0(); mbar_wait_(&sm.full[s], (unsigned)(i / NS) & 1u); MMQ_ACC(0, c[2]); }
                { MMQ_T0(); mbar_wait_(&sm.dempty[sd], ((unsigned)(i / kQ8ND) & 1u) ^ 1u); MMQ_ACC(0, c[3]); }
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t bt = smem_addr(sm.slot[s]);
                const uint32_t ta = tmem + 64u * sa, td = tmem + kColD + (uint32_t)N * sd;
                if (elect_one()) {
#pragma unroll
                    for (int m = 0; m < 8; ++m) {
                        const uint64_t bd = umma_desc_sw128(bt + (m >> 2) * (N * 128) + 32 * (m & 3));
                        const uint32_t acc = m > 0;
                        asm volatile(
                            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                            " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(td),
                            "r"(ta + 8u * m), "l"(bd), "r"(idesc), "r"(acc));
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                     smem_addr(&sm.done[sa]))
                                 : "memory");
                }
                __syncwarp();
            }
        }
    } else if (warp < kQ8EpiWarp) {
        // ---- expanders: row r = TMEM lane; A column 8 m + c = code word (8 (m & 1) + c) >> 2 (m >> 1) & 3s.
        // Two quads take alternate blocks so one quad's decode overlaps the other's tcgen05.st latency.
        const int q = warp & 3, r = 32 * q + lane, eg = (warp - 2) >> 2;
        const uint32_t ta_row = tmem + ((uint32_t)(32 * q) << 16);
        for (int i = eg; i < nblk; i += kQ8ExpGroups) {
            const int s = i % NS, sa = i % kQ8NA;
            { MMQ_T0(); mbar_wait_(&sm.full[s], (unsigned)(i / NS) & 1u); MMQ_ACC(0, c[5]); }
            const uint32_t rec = smem_addr(sm.slot[s]) + q8_act_bytes(BN);
            uint32_t w[16];
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                const uint4 v = lds128(rec + cc * 2048 + 16 * r);
                w[4 * cc] = v.x;
                w[4 * cc + 1] = v.y;
                w[4 * cc + 2] = v.z;
                w[4 * cc + 3] = v.w;
            }
            // A slot sa was last read by block i - 4: wait for its completion (phase of block i - 4)
            if (i >= kQ8NA) { MMQ_T0(); mbar_wait_(&sm.done[sa], (unsigned)((i - kQ8NA) / kQ8NA) & 1u); MMQ_ACC(0, c[6]); }
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {  // columns 32 hh .. 32 hh + 31 (m = 4 hh .. 4 hh + 3)
                uint32_t a[32];
#pragma unroll
                for (int mm = 0; mm < 4; ++mm)
#pragma unroll
                    for (int cc = 0; cc < 8; ++cc) {
                        const int m = 4 * hh + mm;
                        a[8 * mm + cc] = (w[8 * (m & 1) + cc] >> (2 * (m >> 1))) & 0x03030303u;
                    }
                asm volatile(
                    "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
                    "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(
                        ta_row + 64u * sa + 32u * hh),
                    "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]),
                    "r"(a[8]), "r"(a[9]), "r"(a[10]), "r"(a[11]), "r"(a[12]), "r"(a[13]), "r"(a[14]), "r"(a[15]),
                    "r"(a[16]), "r"(a[17]), "r"(a[18]), "r"(a[19]), "r"(a[20]), "r"(a[21]), "r"(a[22]), "r"(a[23]),
                    "r"(a[24]), "r"(a[25]), "r"(a[26]), "r"(a[27]), "r"(a[28]), "r"(a[29]), "r"(a[30]), "r"(a[31])
                    : "memory");
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive_(&sm.aready[sa]);
        }
    } else {
        // ---- epilogue: rows 32 q + lane, tokens [hh BN/2, (hh + 1) BN/2), drained 8 tokens at a time ----
        constexpr int H = BN / 2;
        const int q = warp & 3, hh = (warp - kQ8EpiWarp) >> 2;  // TMEM lane quarter = warp % 4
        const int r = 32 * q + lane;
        const int64_t grow = (int64_t)rt * 128 + r;
        const uint32_t td_row = tmem + ((uint32_t)(32 * q) << 16) + kColD;
        float acc[H];
#pragma unroll
        for (int j = 0; j < H; ++j) acc[j] = 0.f;
        for (int i = 0; i < nblk; ++i) {
            const int s = i % NS, sd = i % kQ8ND;
            { MMQ_T0(); mbar_wait_(&sm.done[i % kQ8NA], (unsigned)(i / kQ8NA) & 1u); MMQ_ACC(0, c[8]); }
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint8_t* slot = sm.slot[s];
            const uint32_t rec = smem_addr(slot) + q8_act_bytes(BN);
            const float d = __half2float(__ushort_as_half(lds16(rec + 8192 + 2 * r)));
            const float zf = (float)(1 + lds_s8(rec + 8192 + 256 + r));
            const float2* meta = reinterpret_cast<const float2*>(slot + 512 * BN) + hh * H;
            const uint32_t t0 = td_row + (uint32_t)N * sd + (uint32_t)(hh * H);
#pragma unroll
            for (int j0 = 0; j0 < H; j0 += 8) {
                uint32_t c0[8], c1[8];
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                             : "=r"(c0[0]), "=r"(c0[1]), "=r"(c0[2]), "=r"(c0[3]), "=r"(c0[4]), "=r"(c0[5]),
                               "=r"(c0[6]), "=r"(c0[7])
                             : "r"(t0 + j0));
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                             : "=r"(c1[0]), "=r"(c1[1]), "=r"(c1[2]), "=r"(c1[3]), "=r"(c1[4]), "=r"(c1[5]),
                               "=r"(c1[6]), "=r"(c1[7])
                             : "r"(t0 + BN + j0));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (j0 + 8 >= H) {  // last chunk read: accumulator slot free
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) mbar_arrive_(&sm.dempty[sd]);
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const float2 fc = meta[j0 + j];  // (2^(ex-4), Q 2^(ex-4)) of token hh H + j0 + j
                    const float v = (float)((int)c0[j] + 256 * (int)c1[j]);
                    acc[j0 + j] += d * (fc.x * v - zf * fc.y);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive_(&sm.empty[s]);
        }
        if (grow < rows) {
#pragma unroll
            for (int j = 0; j < H; ++j) {
                const int64_t m = (int64_t)tt * BN + hh * H + j;
                if (m < M) y[grow * stride_r + m * stride_m] = (TY)acc[j];
            }
        }
    }
    if (unsigned long long* trc = g_mmq_trace) {
        const int cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
        const long long tot = clock64() - tk0;
        if (threadIdx.x == 0) { trc[cta * 16 + 0] = c[0]; trc[cta * 16 + 10] = nblk; trc[cta * 16 + 11] = tot; }
        if (threadIdx.x == 32) { trc[cta * 16 + 1] = c[1]; trc[cta * 16 + 2] = c[2]; trc[cta * 16 + 3] = c[3]; trc[cta * 16 + 4] = tot; }
        if (threadIdx.x == 64) { trc[cta * 16 + 5] = c[5]; trc[cta * 16 + 6] = c[6]; trc[cta * 16 + 7] = tot; }
        if (threadIdx.x == 32 * kQ8EpiWarp) { trc[cta * 16 + 8] = c[8]; trc[cta * 16 + 9] = tot; }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
    }
}

// Weight records [RT][NB][kQ8Rec]: codes [c 0..3][row 0..127][16 B] (code byte B of a row holds
// elements B, 64+B, 128+B, 192+B at bit pairs 0..3, value q + 1), f16 scales [row], int8 zps [row].
__global__ void repack_mmq8_kernel(const uint8_t* __restrict__ payload, int64_t rows, int NB, int RT, int asym,
                                   uint8_t* __restrict__ out) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (record, row, byte B)
    if (idx >= (int64_t)RT * NB * 128 * 64) return;
    const int B = (int)(idx & 63), r = (int)((idx >> 6) & 127);
    const int64_t rec = idx >> 13;
    const int b = (int)(rec % NB);
    const int64_t row = (rec / NB) * 128 + r;
    uint8_t* o = out + rec * kQ8Rec;
    uint8_t byte = 0;
    uint16_t sb = 0;
    int8_t z = 0;
    if (row < rows) {
        const uint8_t* p = payload + (row * NB + b) * 100;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int e = 64 * i + B;
            const int c = ((p[e >> 3] >> (e & 7)) & 1) | (((p[32 + (e >> 3)] >> (e & 7)) & 1) << 1);
            byte |= (uint8_t)(c << (2 * i));
        }
        sb = *reinterpret_cast<const uint16_t*>(p + 96);
        if (asym) z = (int8_t)(int)f16_bits_to_f32(*reinterpret_cast<const uint16_t*>(p + 98));
    }
    o[(B >> 4) * 2048 + r * 16 + (B & 15)] = byte;
    if (B == 0) {
        *reinterpret_cast<uint16_t*>(o + 8192 + 2 * r) = sb;
        reinterpret_cast<int8_t*>(o + 8192 + 256)[r] = z;
    }
}

// Activation records [token tile][NB][q8_act_bytes(BN)]: B tile rows n = l BN + m (limb l of token
// m), 256 k bytes as 2 SW128 k-atoms of N rows; then (2^(ex-4), Q 2^(ex-4)) per token.  One warp
// per (block, token); the chain kernel's integer rotation with |q| <= 2^14 (two balanced limbs).
template <typename TX>
__global__ void rotate_act_i8_kernel(const TX* __restrict__ x, int64_t NB, int64_t M, int64_t M_pad,
                                     int64_t stride_k, int64_t stride_m, int BN, uint8_t* __restrict__ out,
                                     unsigned* __restrict__ nonfinite) {
    pdl_release();
    // CTA = (block b, 8 tokens): coalesced loads along whichever of k / token is contiguous into a
    // padded smem tile, then warp w rotates token m0 + w from it (conflict-free: pitch 257)
    __shared__ float tile[8][257];
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t b = blockIdx.x, m0 = (int64_t)blockIdx.y * 8;
    const TX* xb = x + b * 256 * stride_k;
    if (stride_k == 1 && stride_m != 1) {  // token-major: threads along k
#pragma unroll
        for (int j = 0; j < 8; ++j) tile[j][tid] = m0 + j < M ? (float)xb[tid + (m0 + j) * stride_m] : 0.f;
    } else {  // k-major: 8 consecutive tokens per k row, 32 k rows per pass
        const int j = tid & 7, kl = tid >> 3;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int k = kl + 32 * i;
            tile[j][k] = m0 + j < M ? (float)xb[k * stride_k + (m0 + j) * stride_m] : 0.f;
        }
    }
    __syncthreads();
    const int64_t m = m0 + (tid >> 5);
    const int N = 2 * BN;
    uint8_t* rec = out + ((m / BN) * NB + b) * (int64_t)(512 * BN + 8 * BN);
    const int mm = (int)(m % BN);
    int v[8];
    int ex = 0, Q = 0;
    if (m < M) {
        float f[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) f[e] = tile[tid >> 5][lane + 32 * e];
        bool bad = false;
#pragma unroll
        for (int e = 0; e < 8; ++e) bad |= !isfinite(f[e]);
        if (nonfinite && __any_sync(FULL, bad) && lane == 0) atomicOr(nonfinite, 1u);
        unsigned fb = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) fb = max(fb, __float_as_uint(fabsf(f[e])));
        fb = __reduce_max_sync(FULL, fb);
        const float fm = __uint_as_float(fb);
        const int e_in = fm > 0.f ? ilogbf(fm) - 21 : 0;
        const float sc = ldexpf(1.0f, -e_in);
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = __float2int_rn(f[e] * sc);
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
        const int k = max(0, bl - 14);
        ex = e_in + k;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            v[e] = k ? ((v[e] + (1 << (k - 1))) >> k) : v[e];
            Q += v[e];
        }
        Q = __reduce_add_sync(FULL, Q);
    } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = 0;
    }
#pragma unroll
    for (int e8 = 0; e8 < 8; ++e8) {
        const int e = lane + 32 * e8;
        const int l0 = ((v[e8] + 128) & 255) - 128;
        const int l1 = (v[e8] - l0) >> 8;
        const int kb = e & 127;
        uint8_t* atom = rec + (e >> 7) * (N * 128) + (kb & 15);
        atom[sw128_off(mm, kb >> 4)] = (uint8_t)(int8_t)l0;
        atom[sw128_off(BN + mm, kb >> 4)] = (uint8_t)(int8_t)l1;
    }
    if (lane == 0) {
        float2* meta = reinterpret_cast<float2*>(rec + 512 * BN);
        const float f = m < M ? ldexpf(1.0f, ex - 4) : 0.f;
        meta[mm] = make_float2(f, (float)Q * f);
    }
}

}  // namespace itq3

using namespace itq3;

extern "C" int itq3_mmq8_block_n(int64_t m) { return m <= 16 ? 16 : (m <= 32 ? 32 : 64); }

extern "C" int64_t itq3_mmq8_nbytes(int64_t rows, int64_t cols) {
    return (rows + 127) / 128 * (cols / 256) * (int64_t)kQ8Rec;
}

extern "C" int itq3_repack_mmq8(const uint8_t* payload, int64_t rows, int64_t cols, int asymmetric, uint8_t* out,
                                void* stream) {
    if (rows <= 0 || cols <= 0 || cols % 256) {
        set_error("itq3_repack_mmq8: needs cols %% 256 == 0 (got %lld x %lld)", (long long)rows, (long long)cols);
        return ITQ3_E_UNSUPPORTED;
    }
    const int NB = (int)(cols / 256), RT = (int)((rows + 127) / 128);
    const int64_t n = (int64_t)RT * NB * 128 * 64;
    repack_mmq8_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(payload, rows, NB, RT, asymmetric,
                                                                                      out);
    return check_launch("itq3_repack_mmq8");
}

extern "C" int64_t itq3_mmq8_act_nbytes(int64_t cols, int64_t m) {
    const int BN = itq3_mmq8_block_n(m);
    return (m + BN - 1) / BN * (cols / 256) * (int64_t)q8_act_bytes(BN);
}

extern "C" int itq3_rotate_act_i8(const void* x, int x_dtype, int64_t cols, int64_t m, int64_t stride_k,
                                  int64_t stride_m, uint8_t* out, unsigned* nonfinite, void* stream) {
    if (cols <= 0 || cols % 256 || m <= 0 || m > 64) {
        set_error("itq3_rotate_act_i8: need cols %% 256 == 0 and 0 < m <= 64");
        return ITQ3_E_SHAPE;
    }
    const int BN = itq3_mmq8_block_n(m);
    const int64_t NB = cols / 256, M_pad = (m + BN - 1) / BN * BN;
    const dim3 grid((unsigned)NB, (unsigned)(M_pad / 8));
    cudaStream_t s = (cudaStream_t)stream;
    switch (x_dtype) {
        case ITQ3_F32:
            rotate_act_i8_kernel<float><<<grid, 256, 0, s>>>((const float*)x, NB, m, M_pad, stride_k, stride_m, BN, out, nonfinite);
            break;
        case ITQ3_BF16:
            rotate_act_i8_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>((const __nv_bfloat16*)x, NB, m, M_pad, stride_k,
                                                                     stride_m, BN, out, nonfinite);
            break;
        case ITQ3_F16:
            rotate_act_i8_kernel<__half><<<grid, 256, 0, s>>>((const __half*)x, NB, m, M_pad, stride_k, stride_m, BN,
                                                              out, nonfinite);
            break;
        default:
            set_error("itq3_rotate_act_i8: unsupported dtype %d", x_dtype);
            return ITQ3_E_DOMAIN;
    }
    return check_launch("itq3_rotate_act_i8");
}

static int mmq8_splits(int64_t rows, int64_t cols, int64_t m) {
    const int BN = itq3_mmq8_block_n(m);
    const int64_t tiles = (rows + 127) / 128 * ((m + BN - 1) / BN);
    const int64_t NB = cols / 256;
    int64_t ks = 148 / tiles;                 // one wave (one CTA per SM): tiles x ks <= 148
    ks = ks < NB / 2 ? ks : NB / 2;           // >= 2 blocks per split
    return (int)(ks < 1 ? 1 : ks);
}

extern "C" int64_t itq3_mmq8_ws_nbytes(int64_t rows, int64_t cols, int64_t m) {
    const int ks = mmq8_splits(rows, cols, m);
    return ks > 1 ? (int64_t)ks * rows * m * (int64_t)sizeof(float) : 0;
}

template <int BN, typename TY>
static int launch_mmq8(const uint8_t* w, int64_t rows, int64_t cols, const uint8_t* act, int64_t m, TY* y,
                       int64_t sr, int64_t sm_, float* ws, cudaStream_t s) {
    const int smem = (int)sizeof(Q8Smem<BN>) + 1024;
    static std::atomic<unsigned long long> attr{0}, attr32{0};
    if (int rc = ensure_smem_attr(mmq8_kernel<BN, TY>, smem, attr, "itq3_mmq8: smem attribute")) return rc;
    const int NB = (int)(cols / 256);
    const int ks = ws ? mmq8_splits(rows, cols, m) : 1;
    const dim3 grid((unsigned)((rows + 127) / 128), (unsigned)((m + BN - 1) / BN), (unsigned)ks);
    if (ks == 1) {
        launch_pdl(mmq8_kernel<BN, TY>, grid, dim3(kQ8Threads), smem, s, w, NB, act, rows, m, y, sr, sm_, (int64_t)0);
        return check_launch("itq3_mmq8");
    }
    if (int rc = ensure_smem_attr(mmq8_kernel<BN, float>, smem, attr32, "itq3_mmq8: smem attribute")) return rc;
    launch_pdl(mmq8_kernel<BN, float>, grid, dim3(kQ8Threads), smem, s, w, NB, act, rows, m, ws, m, (int64_t)1,
               rows * m);
    int rc = check_launch("itq3_mmq8 (split-K)");
    if (rc) return rc;
    const int64_t n = rows * m;
    mmq_splitk_reduce<TY><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(ws, ks, rows, m, y, sr, sm_,
                                                                      (const unsigned long long*)nullptr, 0, 0);
    return check_launch("itq3_mmq8 (split-K reduce)");
}

extern "C" int itq3_mmq8(const uint8_t* w, int64_t rows, int64_t cols, const uint8_t* act, int64_t m, void* y,
                         int y_dtype, int64_t stride_r, int64_t stride_m, void* workspace, void* stream) {
    if (rows <= 0 || cols <= 0 || cols % 256 || m <= 0 || m > 64) {
        set_error("itq3_mmq8: bad shape (needs cols %% 256 == 0, 0 < m <= 64)");
        return ITQ3_E_SHAPE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const int BN = itq3_mmq8_block_n(m);
    float* ws = (float*)workspace;
    if (y_dtype == ITQ3_F32) {
        if (BN == 16) return launch_mmq8<16>(w, rows, cols, act, m, (float*)y, stride_r, stride_m, ws, s);
        if (BN == 32) return launch_mmq8<32>(w, rows, cols, act, m, (float*)y, stride_r, stride_m, ws, s);
        return launch_mmq8<64>(w, rows, cols, act, m, (float*)y, stride_r, stride_m, ws, s);
    }
    if (y_dtype == ITQ3_BF16) {
        if (BN == 16) return launch_mmq8<16>(w, rows, cols, act, m, (__nv_bfloat16*)y, stride_r, stride_m, ws, s);
        if (BN == 32) return launch_mmq8<32>(w, rows, cols, act, m, (__nv_bfloat16*)y, stride_r, stride_m, ws, s);
        return launch_mmq8<64>(w, rows, cols, act, m, (__nv_bfloat16*)y, stride_r, stride_m, ws, s);
    }
    set_error("itq3_mmq8: output dtype must be float32 or bfloat16");
    return ITQ3_E_DOMAIN;
}
