// Persistent dataflow kernel for a dependent chain of fused ITQ3_S GEMVs (decode step).
//
// One CTA per SM runs every stage of the chain in a single launch:
//   * a producer warp streams the CTA's weight units (16 rows x up to 16 256-blocks of
//     tiled 2-bit codes + f16 scales, one cp.async.bulk per field) into an NSLOT-deep shared
//     memory ring guarded by mbarriers.  Weights do not depend on activations, so the
//     stream runs ahead across stage boundaries and HBM never idles on a dependency;
//   * 16 consumer warps compute each unit with m16n8k32 u8 x s8 MMAs (same fragment
//     algebra as gemv.cu) against the stage's rotated activations held in shared memory;
//   * the 16 consumer warps take balanced contiguous tile ranges of the CTA's units (crossing
//     unit boundaries); a unit split over several warps is summed by its last segment in
//     segment order (deterministic);
//   * no counters, flags or fences between stages: every output word is 64 bits = (fp32 value,
//     step epoch), stored and loaded single-copy atomically, so a consumer warp simply spins
//     until the 256 x nch tags of the block it needs carry the current epoch, then rotates that
//     block (FWHT + fixed-point limbs, the K3 math) straight into shared memory.
// Co-residency of all CTAs (required by the spin waits) is guaranteed by a cooperative
// launch sized to one CTA per SM.
#include <cooperative_groups.h>
#include <type_traits>

#include "common.cuh"

namespace itq3 {

#ifndef CHAIN_PF_UNITS  // L2 prefetch distance of the producer, in units beyond the ring (0: off)
#define CHAIN_PF_UNITS 4
#endif

constexpr int kChainConsumerWarps = 16;
#ifndef CHAIN_REDUCERS
#define CHAIN_REDUCERS 2
#endif
// Reducer warps take alternate units (a unit's reduction sits between its last tile and its publish, and
// one warp alone falls behind).  Up to 20 warps keep 5 per SMSP, i.e. the same 96-register cap as 18.
constexpr int kChainReducers = CHAIN_REDUCERS;
constexpr int kChainThreads = 32 * (kChainConsumerWarps + 1 + kChainReducers);  // + producer + reducers
constexpr int kProducerWarp = kChainConsumerWarps, kReducerWarp = kChainConsumerWarps + 1;
constexpr int kUnitBlocks = 16;                          // 256-blocks per unit (one per consumer warp)
constexpr int kSlotCodes = kUnitBlocks * 1024;           // 16 KB
constexpr int kSlotScales = kUnitBlocks * 32;            // 512 B
constexpr int kSlotZps = kUnitBlocks * 16;               // 256 B
constexpr int kSlotBytes = kSlotCodes + kSlotScales + kSlotZps;
constexpr int kMaxChainNB = 256;                         // K up to 65536
constexpr int kMaxChainPeers = 8;                        // tensor-parallel ranks (one NVLink domain)
constexpr int kMaxLimbs = 4;

struct ChainStage {
    const uint8_t* tiled;  // codes | scales | zps (itq3_repack_tiled layout)
    unsigned long long* y; // [nch][rows] tagged outputs: low 32 = fp32 bits, high 32 = step epoch
    const float* xin;      // optional: untagged fp32 input (independent stage, no dependency)
    // Tensor-parallel stage (npeer > 0): this rank computes output rows [row0, row0 + rows) of a
    // yrows-row stage and stores each tagged word straight into all npeer ranks' copies of y
    // (ypeer[p] = rank p's y, NVLink peer pointers), so the all-gather is fused into the reducer.
    // y is then double-buffered by epoch parity ([2][nch][yrows]) so a rank already in step t+1
    // never overwrites words a slower peer still reads in step t.
    union {
        unsigned long long* const* ypeer;  // npeer > 0: the ranks' copies of y
        const unsigned long long* xres;    // decoder (npeer == 0): tagged residual stream the flag-16/64
                                           // input adds (null: the launch input x0, untagged)
    };
    unsigned long long* xout;  // flag 128: where this RMSNorm stage writes the residual it formed (tagged)
    const int32_t* work;       // optional [gridDim.x]: CTA c takes K-chunk work[c] / Gc, row tiles from
                               // work[c] % Gc (-1: idle) -- a host-balanced assignment (itq3_chain_set_work)
    int64_t rows, cols;
    int32_t NB, RT, asym, npeer;
    int32_t row0, yrows;
};

__host__ __device__ inline int act_block_bytes(int L) { return 256 * L + 32; }
constexpr int kActSmemBlock = 8 * 16 * 8 + 64;  // 4-column fragments [q][g<4][t] + 8 (factor, corr) pairs

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
// system scope: words written by peer GPUs over NVLink (tensor-parallel stages)
__device__ __forceinline__ unsigned long long ld_u64_relaxed_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_u64_relaxed_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
template <bool SYS>
__device__ __forceinline__ unsigned long long ld_tag(const unsigned long long* p) {
    return SYS ? ld_u64_relaxed_sys(p) : ld_u64_relaxed(p);
}

// Wait for, and sum, one 256-block of a producing stage's tagged K-chunk partials (this lane's elements
// el + 32 e, el = rot_lane_element(lane)).  Each 64-bit word carries its value and the step epoch in one
// single-copy-atomic access, so the consumer needs no flag, counter or fence: it spins until all
// 256 x nparts tags equal `epoch`.
template <bool SYS>
__device__ __forceinline__ void load_tagged_block(const unsigned long long* src, int nparts, int64_t part_stride,
                                                  unsigned epoch, int el, float (&f)[8]) {
    for (;;) {
        bool ok = true;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const unsigned long long w = ld_tag<SYS>(src + el + 32 * e);
            ok &= (unsigned)(w >> 32) == epoch;
            f[e] = __uint_as_float((unsigned)w);
        }
        for (int c = 1; c < nparts; ++c)  // K-chunk partials, fixed order
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const unsigned long long w = ld_tag<SYS>(src + c * part_stride + el + 32 * e);
                ok &= (unsigned)(w >> 32) == epoch;
                f[e] += __uint_as_float((unsigned)w);
            }
        if (__all_sync(FULL, ok)) return;  // no back-off: measured 0.4726 (64 ns) -> 0.4696 ms per token
    }
}

// Element layout of a rotation: lane L holds the block's elements k = rot_lane_element(L) + 32 e,
// e = 0..7, i.e. the lane bits (0, 1) and (2, 3) of k swapped.  The butterflies do not care (H_256 is a
// tensor product over the bits of k), and it puts the four bytes beta = k & 3 of every B-fragment word
// into the COLUMNS of a stmatrix.m16n8.trans.b8 source matrix: lane L = 4 c' + j holds source row c' =
// (k bits 0, 1, 4) and column pair j = k bits (2, 3); byte b of the register (limb b) goes to smem row
// 2 j + (b & 1), byte column c' + 8 (b >> 1) (tools/probes/stsm_probe.cu).  So each 128-byte chunk image
// is 8 rows (t, limb & 1) x 16 bytes (limb >> 1, h, beta), and one stmatrix.x4 writes four chunks: two
// instructions replace 32 byte stores and 24 byte shifts (tools/probes/rot_probe.cu: 1703 -> 1290 cycles
// per rotation with 16 warps, fragments identical).
__device__ __forceinline__ int rot_lane_element(int L) { return ((L & 3) << 2) | ((L >> 2) & 3) | (L & 16); }

// Rotate 256 fp32 values (this lane's elements rot_lane_element(lane) + 32 e) into the fragment image.
// Integer pipeline: y -> 23-bit fixed point with the block's power-of-two scale s_in =
// 2^(ilogb(max|y|) - 21) (|y_int| < 2^22, as fine as fp32's own rounding of the largest elements),
// exact int32 butterfly (|x'| < 2^30), then x' rounded to the limb range |q| <= 2^(8L-2) by one more
// power-of-two shift k (tests/test_gpu_stack.py chain_bound).
// MAD: butterflies as one register-operand mad each (the symmetric-only kernels).  LO: the input is H_16 y per
// 16-element group (the symmetric single-GPU kernel: its reducers store H_16 of every 16-row tile and stage
// 0 transforms x0 as it loads it), i.e. the butterflies over k bits 0-3 (lane bits 0-3) are done and only k
// bit 4 (lane bit 4) and the register bits remain.
// Output b of H_4 over a 4-lane group whose member b ^ m holds a[m]: sum_m (-1)^popc(b & (b ^ m)) a[m]
__device__ __forceinline__ float radix4_h(const float (&a)[4], int b) {
    float acc = (__popc(b) & 1) ? -a[0] : a[0];
#pragma unroll
    for (int m = 1; m < 4; ++m) acc = fmaf(a[m], (__popc(b & (b ^ m)) & 1) ? -1.0f : 1.0f, acc);
    return acc;
}

template <bool MAD = false, bool LO = false>
__device__ __forceinline__ void chain_rotate_to_smem(const float (&f)[8], int L, uint8_t* img, int lane) {
    // warp max of |f| as an integer max of the float bit patterns (sign cleared): one REDUX
    unsigned fbits = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) fbits = max(fbits, __float_as_uint(f[e]) & 0x7fffffffu);
    fbits = __reduce_max_sync(FULL, fbits);
    const int bexp = (int)(fbits >> 23);  // biased exponent of max|f|
    int e_in;
    float sc_in;
    if (bexp >= 21) {  // max|f| >= 2^-106: s_in^-1 = 2^-e_in is a normal float, built from its bits
        e_in = bexp - 148;
        sc_in = __int_as_float((127 - e_in) << 23);
    } else {
        const float fmaxa = __uint_as_float(fbits);
        e_in = fmaxa > 0.f ? ilogbf(fmaxa) - 21 : 0;
        sc_in = pow2f(-e_in);
    }
    int v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e)  // |f sc_in| < 2^22, sc_in a power of two: one FMA rounds to nearest even
        v[e] = __float_as_int(fmaf(f[e], sc_in, 12582912.0f)) - 0x4B400000;
    // the zero-point correction sum_k x'_k / 16 = v0 2^(e_in + c_sh): 256 v_0 / 16 (lane 0 holds element 0); LO:
    // H_hi of v leaves 16 sum_{k < 16} v_k (lanes 0-15 at e = 0), over 16
    int v0 = v[0];
    constexpr int c_sh = LO ? 0 : 4;
    if (LO) {
#pragma unroll
        for (int h = 1; h < 16; h <<= 1) v0 += __shfl_xor_sync(FULL, v0, h);  // |v0| < 2^26
    }
#pragma unroll
    for (int h = LO ? 16 : 1; h < 32; h <<= 1) {  // lane bits: p + v on the low lane, p - v on the high lane
        const int sg = (lane & h) ? -1 : 1;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int p = __shfl_xor_sync(FULL, v[e], h);
            if (MAD)  // an opaque +-1 multiplier keeps ptxas from splitting it into negate + add
                asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(v[e]) : "r"(v[e]), "r"(1 - ((lane & h) ? 2 : 0)), "r"(p));
            else
                v[e] = p + sg * v[e];
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
    // max |v| as max(max v, -min v) over three-input integer min / max (7 instructions, not 8 IABS + 8 max)
    const int vmx = __vimax3_s32(__vimax3_s32(v[0], v[1], v[2]), __vimax3_s32(v[3], v[4], v[5]), max(v[6], v[7]));
    const int vmn = __vimin3_s32(__vimin3_s32(v[0], v[1], v[2]), __vimin3_s32(v[3], v[4], v[5]), min(v[6], v[7]));
    unsigned amax = (unsigned)max(vmx, -vmn);
    amax = __reduce_max_sync(FULL, amax);
    // shift k so that |q| <= 2^(8L-2) (limbs never overflow): bitlen(amax) - k <= 8L - 2
    const int bl = 32 - __clz(amax);
    // (limbs = 4 gives no more than 22 bits: q 4^3 and the class differences must fit the four
    // balanced record limbs of an int32)
    const int k = max(0, bl - min(8 * L - 2, 22));
    const int ex = e_in + k;
    const int rnd = (1 << k) >> 1;
    // Class folding: chunk e = 4G + i pairs with the A operand c * 4^i (bit pair i of the code
    // bytes), so its activations are stored pre-scaled by 4^(3-i); every IMMA of a tile then
    // accumulates 64 * sum(c x') into ONE integer accumulator (no per-tile class recombination).
    // |q| <= 2^22 -> |q 4^(3-i)| <= 2^28: four balanced base-256 limbs = the bytes of
    // (qs + 0x80808080) ^ 0x80808080, all four record columns used.
    // Cumulative masks: with P_i = codes & (4^(i+1) - 1 per byte) (P_3 = the raw word, no mask),
    // sum_i (c_i 4^i) A_i = sum_i P_i (A_i - A_{i+1}) (A_4 = 0, exact in int32), so chunk e stores
    // the difference of its pre-scaled activation and the next class's: the tile needs 3 LOP3 per
    // A register group instead of 4 and produces the same integer accumulators.
    int qs[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) qs[e] = ((v[e] + rnd) >> k) << (2 * (3 - (e & 3)));
    uint32_t lw[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int dq = (e & 3) < 3 ? qs[e] - qs[e + 1] : qs[e];  // |dq| < 2^29
        lw[e] = (uint32_t)(dq + (int)0x80808080u) ^ 0x80808080u;
    }
    // lanes 8 m .. 8 m + 7 address the 8 rows of matrix m (chunk m of the first store, 4 + m of the second)
    const uint32_t a = smem_u32(img) + (lane >> 3) * 128 + (lane & 7) * 16;
    asm volatile("stmatrix.sync.aligned.m16n8.x4.trans.shared.b8 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(lw[0]),
                 "r"(lw[1]), "r"(lw[2]), "r"(lw[3])
                 : "memory");
    asm volatile("stmatrix.sync.aligned.m16n8.x4.trans.shared.b8 [%0], {%1, %2, %3, %4};" ::"r"(a + 512), "r"(lw[4]),
                 "r"(lw[5]), "r"(lw[6]), "r"(lw[7])
                 : "memory");
    float* meta = reinterpret_cast<float*>(img + 8 * 16 * 8);  // f[0..7], corr[0..7]
    if (lane < 8) {
        meta[lane] = lane < 4 ? __int_as_float((8 * lane + ex - 10 + 127) << 23) : 0.0f;  // 256^l 2^ex / 16 / 64
        // sum_k x'_k / 16 = 16 x_0 (fixed point), exact: the tile's error is then sum_k c_k (q_k 2^ex - x'_k)
        meta[8 + lane] = lane == 0 ? (float)v0 * pow2f(e_in + c_sh) : 0.0f;
    }
}

// B fragments of lane (g, t) from a rotation image: chunk q's words (limb g, t-group t, h = 0 / 1) are one
// 8-byte pair at row 2 t + (g & 1), byte 8 (g >> 1) (conflict-free: 16 lanes read 128 distinct bytes);
// columns g >= 4 are zero.
__device__ __forceinline__ void chain_load_frags(const uint8_t* img, int g, int t, uint2 (&bf)[8]) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
        bf[q] = g < 4 ? *reinterpret_cast<const uint2*>(img + q * 128 + (2 * t + (g & 1)) * 16 + 8 * (g >> 1))
                      : make_uint2(0u, 0u);
}

// One 16-row x 256-k tile of the warp's block from a ring slot: returns the (row g, row g+8)
// contributions of this lane's limb-pair columns (before the quad combine).
template <bool ASYM>  // asymmetric zero-points: a separate instantiation, so symmetric tiles skip the zp terms
__device__ __forceinline__ float2 chain_tile(const uint8_t* ring, int warp, int lane, int g, const uint2 (&bf)[8],
                                             float fcx, float corr) {
    const uint4 wa0 = reinterpret_cast<const uint4*>(ring + warp * 1024)[lane];
    const uint4 wa1 = reinterpret_cast<const uint4*>(ring + warp * 1024 + 512)[lane];
    const uint32_t sc = reinterpret_cast<const uint32_t*>(ring + kSlotCodes + warp * 32)[g];
    // ONE accumulator for both k groups (an 8-deep IMMA chain; the two units of an iteration and the
    // warps of the SMSP give the tensor pipe enough independent chains), so no group merge afterwards
    int C[4] = {0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t mk = i == 3 ? 0xffffffffu : (0x04040404u << (2 * i)) - 0x01010101u;  // cumulative
        mma_u8s8_c(C, wa0.x & mk, wa0.y & mk, wa0.z & mk, wa0.w & mk, bf[i].x, bf[i].y);
        mma_u8s8_c(C, wa1.x & mk, wa1.y & mk, wa1.z & mk, wa1.w & mk, bf[4 + i].x, bf[4 + i].y);
    }
    // columns 2t, 2t+1 = limbs 2t, 2t+1 (factors differ by 256); |C| <= 8 x 32 x 170 x 128 < 2^23, so
    // the pair combination stays below 2^31
    const float v0 = (float)(C[0] + 256 * C[1]);
    const float v1 = (float)(C[2] + 256 * C[3]);
    const float d0 = f16_bits_to_f32((uint16_t)(sc & 0xffffu));
    const float d1 = f16_bits_to_f32((uint16_t)(sc >> 16));
    if (!ASYM) return make_float2(d0 * (fcx * v0 - corr), d1 * (fcx * v1 - corr));
    const uint16_t zz = reinterpret_cast<const uint16_t*>(ring + kSlotCodes + kSlotScales + warp * 16)[g];
    const float zf0 = (float)(1 + (int)(int8_t)(zz & 0xff));
    const float zf1 = (float)(1 + (int)(int8_t)(zz >> 8));
    return make_float2(d0 * (fcx * v0 - zf0 * corr), d1 * (fcx * v1 - zf1 * corr));
}

// Two units' tiles with their IMMA chains interleaved: each IMMA's accumulator input is two MMAs back
// (the chains of one unit alone stall ~13 cycles per IMMA on the accumulator dependency -- the fixed
// stall counts ptxas puts before every dependent IMMA).  Same integer accumulators as chain_tile.
template <bool ASYM>
__device__ __forceinline__ void chain_tile2(const uint8_t* ringA, const uint8_t* ringB, int warp, int lane, int g,
                                            const uint2 (&bf)[8], float fcx, float corr, float2& ra, float2& rb) {
    const uint4 a0 = reinterpret_cast<const uint4*>(ringA + warp * 1024)[lane];
    const uint4 a1 = reinterpret_cast<const uint4*>(ringA + warp * 1024 + 512)[lane];
    const uint4 b0 = reinterpret_cast<const uint4*>(ringB + warp * 1024)[lane];
    const uint4 b1 = reinterpret_cast<const uint4*>(ringB + warp * 1024 + 512)[lane];
    int CA[4] = {0, 0, 0, 0}, CB[4] = {0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t mk = i == 3 ? 0xffffffffu : (0x04040404u << (2 * i)) - 0x01010101u;  // cumulative
        mma_u8s8_c(CA, a0.x & mk, a0.y & mk, a0.z & mk, a0.w & mk, bf[i].x, bf[i].y);
        mma_u8s8_c(CB, b0.x & mk, b0.y & mk, b0.z & mk, b0.w & mk, bf[i].x, bf[i].y);
        mma_u8s8_c(CA, a1.x & mk, a1.y & mk, a1.z & mk, a1.w & mk, bf[4 + i].x, bf[4 + i].y);
        mma_u8s8_c(CB, b1.x & mk, b1.y & mk, b1.z & mk, b1.w & mk, bf[4 + i].x, bf[4 + i].y);
    }
    const uint32_t sa = reinterpret_cast<const uint32_t*>(ringA + kSlotCodes + warp * 32)[g];
    const uint32_t sb = reinterpret_cast<const uint32_t*>(ringB + kSlotCodes + warp * 32)[g];
    const float va0 = (float)(CA[0] + 256 * CA[1]), va1 = (float)(CA[2] + 256 * CA[3]);
    const float vb0 = (float)(CB[0] + 256 * CB[1]), vb1 = (float)(CB[2] + 256 * CB[3]);
    const float da0 = f16_bits_to_f32((uint16_t)(sa & 0xffffu)), da1 = f16_bits_to_f32((uint16_t)(sa >> 16));
    const float db0 = f16_bits_to_f32((uint16_t)(sb & 0xffffu)), db1 = f16_bits_to_f32((uint16_t)(sb >> 16));
    if (!ASYM) {
        ra = make_float2(da0 * (fcx * va0 - corr), da1 * (fcx * va1 - corr));
        rb = make_float2(db0 * (fcx * vb0 - corr), db1 * (fcx * vb1 - corr));
        return;
    }
    const uint16_t za = reinterpret_cast<const uint16_t*>(ringA + kSlotCodes + kSlotScales + warp * 16)[g];
    const uint16_t zb = reinterpret_cast<const uint16_t*>(ringB + kSlotCodes + kSlotScales + warp * 16)[g];
    ra = make_float2(da0 * (fcx * va0 - (float)(1 + (int)(int8_t)(za & 0xff)) * corr),
                     da1 * (fcx * va1 - (float)(1 + (int)(int8_t)(za >> 8)) * corr));
    rb = make_float2(db0 * (fcx * vb0 - (float)(1 + (int)(int8_t)(zb & 0xff)) * corr),
                     db1 * (fcx * vb1 - (float)(1 + (int)(int8_t)(zb >> 8)) * corr));
}

// stage descriptors + this CTA's split cached in smem (global beyond) and the weight-ring depth: the
// decoder instantiation (GATED) trades one ring slot for room to cache a whole token's ~200 stages
#ifndef CHAIN_NSL
#define CHAIN_NSL 10
#endif
template <bool GATED>
struct ChainCfg {
    static constexpr int kSlots = GATED ? 9 : CHAIN_NSL;
    static constexpr int kStages = GATED ? 240 : 136;
};
constexpr int kSmemStages = ChainCfg<false>::kStages;

// ------------------------------------------------------------------------------------------------
// Decoder attention as chain stages (GATED instantiation; the decoder harness of SURVEY.md 8(f)3, not
// an ITQ3_S function).  ATTN_PART (flag 256): item (kv head, split) of nkv x S items, one per CTA;
// the 16 consumer warps read q (the kv head's G = 4 query heads), k and v from the qkv stage's tagged
// outputs, apply RoPE (rotate-half), append k / v to the KV cache at pos (split 0), score the split's
// positions (warp per position, lane = 4 dims x 4 heads), take the per-head softmax statistics and
// P V, and publish (max, sum, 4 x 128 weighted V) as tagged words.  ATTN_COMB (flag 512): CTA h < nh
// combines head h's S partials into 128 tagged attention outputs, the next stage's input.
// ------------------------------------------------------------------------------------------------
struct AttnParams {
    float* kc;           // this layer's K cache [nkv][ctx][128] (fp32)
    float* vc;           // V cache, same layout
    const float* cosb;   // [ctx][64] RoPE tables
    const float* sinb;
    const int64_t* pos;  // device position of the token
    unsigned* err;       // bit 0 set when a launch sees a position outside [0, ctx) (no cache write)
    int nh, nkv, ctx, S;
};
constexpr int kAttnG = 4, kAttnHD = 128, kAttnWords = kAttnHD + 2;  // partial record: max, sum, 128 acc
constexpr int kAttnMaxChunk = 64;  // positions per split: ceil(ctx / S) <= 64 (host-checked)

__device__ __forceinline__ void tagged_load4(const unsigned long long* p, unsigned epoch, int lane, float (&v)[4]) {
    for (;;) {
        bool ok = true;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const unsigned long long w = ld_u64_relaxed(p + lane + 32 * j);
            ok &= (unsigned)(w >> 32) == epoch;
            v[j] = __uint_as_float((unsigned)w);
        }
        if (__all_sync(FULL, ok)) return;
    }
}

// one (kv head, split) item; scratch = the consumer warps' rotation scratch (>= 12.5 KB)
__device__ void attn_part(const AttnParams& P, const unsigned long long* qkv, unsigned long long* part, int item,
                          unsigned epoch, int warp, int lane, float* scratch) {
    constexpr int HD = kAttnHD, G = kAttnG;
    float* qs = scratch;                   // [G][HD]
    float* kcur = qs + G * HD;             // [HD]
    float* vcur = kcur + HD;               // [HD]
    float* ps = vcur + HD;                 // [G][kAttnMaxChunk]
    float* red = ps + G * kAttnMaxChunk;   // [G classes][G heads][HD]
    float* stat = red + G * G * HD;        // [G][2]
    const int t = warp * 32 + lane;
    const int S = P.S, nh = P.nh, nkv = P.nkv;
    const int kvh = item / S, sp = item - kvh * S;
    const int64_t pos64 = *P.pos;
    if (pos64 < 0 || pos64 >= P.ctx) {  // beyond the KV cache: no cache write, empty partials (output 0)
        if (warp == 0 && lane == 0) atomicOr(P.err, 1u);
        const unsigned long long tag = (unsigned long long)epoch << 32;
        unsigned long long* mine = part + (int64_t)item * G * kAttnWords;
        for (int i = t; i < G * kAttnWords; i += 32 * kChainConsumerWarps)
            st_u64_relaxed(mine + i, tag | (i % kAttnWords == 0 ? __float_as_uint(-INFINITY) : 0u));
        return;
    }
    const int pos = (int)pos64;
    const int chunk = (pos + S) / S;  // ceil((pos + 1) / S)
    const int lo = sp * chunk, hi = min(pos + 1, lo + chunk), n = max(0, hi - lo);
    float* kch = P.kc + (int64_t)kvh * P.ctx * HD;
    float* vch = P.vc + (int64_t)kvh * P.ctx * HD;
    // the split's cached K and V rows (earlier tokens; the producer pulled them into L2) into registers
    // while q / k / v of this token are pending: score rows p = lo + warp + 16 i, P V rows lo + c + 4 i
    constexpr int KR = kAttnMaxChunk / kChainConsumerWarps, VR = kAttnMaxChunk / G;
    float kr[KR][4], vr[VR];
    {
#pragma unroll
        for (int i = 0; i < KR; ++i) {
            const int p = lo + warp + kChainConsumerWarps * i;
#pragma unroll
            for (int j = 0; j < 4; ++j) kr[i][j] = p < hi && p != pos ? kch[(int64_t)p * HD + lane + 32 * j] : 0.f;
        }
        const int c = t >> 7, dcol = t & (HD - 1);
#pragma unroll
        for (int i = 0; i < VR; ++i) {
            const int p = lo + c + G * i;
            vr[i] = p < hi && p != pos ? vch[(int64_t)p * HD + dcol] : 0.f;
        }
    }
    if (warp < G + 2) {
        const int base = warp < G ? (kvh * G + warp) * HD : (warp == G ? nh * HD + kvh * HD : (nh + nkv) * HD + kvh * HD);
        float c0 = 0.f, s0 = 0.f, c1 = 0.f, s1 = 0.f;
        if (warp <= G) {  // RoPE factors, loaded before the poll
            c0 = __ldg(P.cosb + (int64_t)pos * (HD / 2) + lane);
            s0 = __ldg(P.sinb + (int64_t)pos * (HD / 2) + lane);
            c1 = __ldg(P.cosb + (int64_t)pos * (HD / 2) + lane + 32);
            s1 = __ldg(P.sinb + (int64_t)pos * (HD / 2) + lane + 32);
        }
        float v[4];  // dims lane, lane + 32, lane + 64, lane + 96
        tagged_load4(qkv + base, epoch, lane, v);
        if (warp <= G) {  // RoPE: pairs (i, i + 64)
            const float a0 = v[0], b0 = v[2], a1 = v[1], b1 = v[3];
            v[0] = a0 * c0 - b0 * s0;
            v[2] = a0 * s0 + b0 * c0;
            v[1] = a1 * c1 - b1 * s1;
            v[3] = a1 * s1 + b1 * c1;
        }
        float* dst = warp < G ? qs + warp * HD : (warp == G ? kcur : vcur);
        const float sc = warp < G ? rsqrtf((float)HD) : 1.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) dst[lane + 32 * j] = v[j] * sc;
        if (warp >= G && sp == 0) {  // append k / v at pos (read back by later tokens' launches)
            float* c = warp == G ? kch : vch;
#pragma unroll
            for (int j = 0; j < 4; ++j) c[(int64_t)pos * HD + lane + 32 * j] = v[j];
        }
    }
    consumer_sync();
    float qr[G][4];
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
        for (int j = 0; j < 4; ++j) qr[g][j] = qs[g * HD + lane + 32 * j];
    // the warp's KR x G scores (positions lo + warp + 16 i beyond hi give 0 and are not stored), reduced
    // over the lanes by a transposed butterfly: each exchange halves the values a lane keeps, so the 16
    // sums take 16 shuffles in 5 dependent rounds (not 5 rounds per value); the additions pair exactly
    // as the plain butterfly's, so the sums are bit-identical
    static_assert(KR * G == 16, "the transposed reduction handles 16 values per lane");
    float d[KR * G];
#pragma unroll
    for (int i = 0; i < KR; ++i) {
        const bool cur = lo + warp + kChainConsumerWarps * i == pos;
        const float k0 = cur ? kcur[lane] : kr[i][0], k1 = cur ? kcur[lane + 32] : kr[i][1],
                    k2 = cur ? kcur[lane + 64] : kr[i][2], k3 = cur ? kcur[lane + 96] : kr[i][3];
#pragma unroll
        for (int g = 0; g < G; ++g) d[i * G + g] = qr[g][0] * k0 + qr[g][1] * k1 + qr[g][2] * k2 + qr[g][3] * k3;
    }
#pragma unroll
    for (int o = 16, w = 8; o >= 2; o >>= 1, w >>= 1) {  // lane keeps values [w * bit, w * bit + w)
        const bool up = lane & o;
#pragma unroll
        for (int j = 0; j < w; ++j) {
            const float send = up ? d[j] : d[j + w], keep = up ? d[j + w] : d[j];
            d[j] = keep + __shfl_xor_sync(FULL, send, o);
        }
    }
    d[0] += __shfl_xor_sync(FULL, d[0], 1);  // value lane >> 1 = (position i, head g) = (v >> 2, v & 3)
    {
        const int v = lane >> 1, p = lo + warp + kChainConsumerWarps * (v / G);
        if (!(lane & 1) && p < hi) ps[(v % G) * kAttnMaxChunk + p - lo] = d[0];
    }
    consumer_sync();
    if (warp < G) {
        float m = -INFINITY;
        for (int i = lane; i < n; i += 32) m = fmaxf(m, ps[warp * kAttnMaxChunk + i]);
        for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(FULL, m, o));
        float se = 0.f;
        for (int i = lane; i < n; i += 32) {
            const float e = __expf(ps[warp * kAttnMaxChunk + i] - m);
            ps[warp * kAttnMaxChunk + i] = e;
            se += e;
        }
        for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(FULL, se, o);
        if (lane == 0) {
            stat[warp * 2] = m;
            stat[warp * 2 + 1] = se;
        }
    }
    consumer_sync();
    {  // P V: thread (class c, dim d) takes positions lo + c, lo + c + G, ... for all G heads
        const int c = t >> 7, dcol = t & (HD - 1);
        float acc[G];
#pragma unroll
        for (int g = 0; g < G; ++g) acc[g] = 0.f;
#pragma unroll
        for (int k = 0; k < VR; ++k) {
            const int i = c + G * k;
            if (i >= n) break;
            const float v = lo + i == pos ? vcur[dcol] : vr[k];
#pragma unroll
            for (int g = 0; g < G; ++g) acc[g] += ps[g * kAttnMaxChunk + i] * v;
        }
#pragma unroll
        for (int g = 0; g < G; ++g) red[(c * G + g) * HD + dcol] = acc[g];
    }
    consumer_sync();
    {
        const unsigned long long tag = (unsigned long long)epoch << 32;
        const int g = t >> 7, dcol = t & (HD - 1);
        float o = 0.f;
#pragma unroll
        for (int c = 0; c < G; ++c) o += red[(c * G + g) * HD + dcol];
        unsigned long long* mine = part + ((int64_t)item * G + g) * kAttnWords;
        st_u64_relaxed(mine + 2 + dcol, tag | __float_as_uint(o));
        if (dcol == 0) {
            st_u64_relaxed(mine, tag | __float_as_uint(stat[g * 2]));
            st_u64_relaxed(mine + 1, tag | __float_as_uint(stat[g * 2 + 1]));
        }
    }
    consumer_sync();  // the scratch is free for the next item / stage
}

// head h: combine the S (<= 32) partials of its kv head into 128 tagged outputs, with all 512 consumer
// threads: thread (group q = t >> 7, dim d) loads the weighted-V words of splits q per .. q per + per - 1
// (per = ceil(S / 4) <= 8) and lane j of every warp split j's (max, sum), all in ONE poll loop -- one L2
// round trip once the partials are there -- then the four groups' sums meet in shared memory in a fixed
// order (deterministic).  scratch: >= 4 x 128 floats.
__device__ void attn_comb(const AttnParams& P, const unsigned long long* part, unsigned long long* att, int h,
                          unsigned epoch, int t, float* scratch) {
    constexpr int HD = kAttnHD, G = kAttnG, Q = 4, kPer = 8;
    const int kvh = h / G, g = h - kvh * G, S = P.S, lane = t & 31, q = t >> 7, dcol = t & (HD - 1);
    const int per = (S + Q - 1) / Q;
    const unsigned long long* base = part + ((int64_t)kvh * S * G + g) * kAttnWords;  // split j: + j G kAttnWords
    float mj = -INFINITY, sj = 0.f, a[kPer];
    for (;;) {
        bool ok = true;
        if (lane < S) {  // split statistics: lane j holds split j's (max, sum)
            const unsigned long long w0 = ld_u64_relaxed(base + (int64_t)lane * G * kAttnWords);
            const unsigned long long w1 = ld_u64_relaxed(base + (int64_t)lane * G * kAttnWords + 1);
            ok = (unsigned)(w0 >> 32) == epoch && (unsigned)(w1 >> 32) == epoch;
            mj = __uint_as_float((unsigned)w0);
            sj = __uint_as_float((unsigned)w1);
        }
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            a[u] = 0.f;
            const int j = q * per + u;
            if (u < per && j < S) {
                const unsigned long long w = ld_u64_relaxed(base + (int64_t)j * G * kAttnWords + 2 + dcol);
                ok &= (unsigned)(w >> 32) == epoch;
                a[u] = __uint_as_float((unsigned)w);
            }
        }
        if (__all_sync(FULL, ok)) break;
    }
    float m = mj;
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(FULL, m, o));
    const float fj = mj == -INFINITY ? 0.f : __expf(mj - m);  // lane j's split weight
    float num = 0.f;
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
        const int j = q * per + u;
        const float f = __shfl_sync(FULL, fj, j & 31);
        if (u < per && j < S) num += f * a[u];
    }
    scratch[q * HD + dcol] = num;
    consumer_sync();
    if (q == 0) {
        float den = 0.f;
        for (int j = 0; j < S; ++j) den += __shfl_sync(FULL, sj * fj, j);
        const float o = scratch[dcol] + scratch[HD + dcol] + scratch[2 * HD + dcol] + scratch[3 * HD + dcol];
        const float r = den > 0.f ? o / den : 0.f;  // den == 0: every split empty (position out of range)
        st_u64_relaxed(att + (int64_t)h * HD + dcol, ((unsigned long long)epoch << 32) | __float_as_uint(r));
    }
    consumer_sync();  // the scratch is free again
}


// Work split of stage st for CTA cta: K-chunk ch (CTAs c with c % nch == ch), and the row
// tiles rt = rt0, rt0 + Gc, ... (Gc CTAs per chunk); active = 0 if the CTA is idle.
struct StageSplit {
    int nch, ch, rt0, Gc, active;
};

template <bool GATED>
struct ChainSmem {
    static constexpr int NSL = ChainCfg<GATED>::kSlots, NST = ChainCfg<GATED>::kStages;
    ChainStage desc[NST];
    StageSplit split[NST];
    alignas(128) uint8_t ring[NSL][kSlotBytes];
    alignas(16) uint8_t rot[kChainConsumerWarps][kActSmemBlock];  // per-warp rotation scratch (attention scratch)
    float part[NSL][kChainConsumerWarps][2][16];        // per-warp row partials of a unit (limb pairs t = 0, 1)
    // per-warp sums of squares of the last 16 RMSNorm input stages: every stage a CTA takes part in has >= 1
    // unit, and the consumers run at most NSL < 15 units ahead of the reducers, so a buffer is never rewritten
    // before the reducers are done with it
    float normsq[16][kChainConsumerWarps];
    uint64_t full[NSL];
    uint64_t empty[NSL];
    uint64_t parts[NSL];  // 16 warps' partials of the unit in this slot are written
    int partcnt[NSL];
};

static_assert(sizeof(ChainSmem<false>) <= 227 * 1024, "chain kernel shared memory exceeds the 227 KB per-CTA limit");
static_assert(sizeof(ChainSmem<true>) <= 227 * 1024, "chain kernel shared memory exceeds the 227 KB per-CTA limit");
static_assert(ChainSmem<true>::NSL < 15, "sm.normsq reuse needs fewer ring slots than RMSNorm buffers - 1");

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ bool compute_split(const ChainStage& st, int cta, int G, int s, StageSplit& sp) {
    sp.nch = (st.NB + kUnitBlocks - 1) / kUnitBlocks;
    sp.Gc = G / sp.nch;
    sp.active = 0;
    if (st.work) {
        const int v = st.work[cta];
        if (v < 0) return false;
        sp.ch = v / sp.Gc;
        sp.rt0 = v - sp.ch * sp.Gc;
        sp.active = sp.rt0 < st.RT;
        return sp.active;
    }
    sp.ch = cta % sp.nch;
    const int idx = cta / sp.nch;
    if (idx >= sp.Gc) return false;
    sp.rt0 = (idx + 7 * s) % sp.Gc;
    sp.active = sp.rt0 < st.RT;
    return sp.active;
}
// Stage s's descriptor and this CTA's split: from the smem cache (filled at kernel start, so the
// per-stage critical path has no dependent global loads or integer divisions) or computed.
template <bool GATED>
__device__ __forceinline__ bool stage_get(const ChainSmem<GATED>& sm, const ChainStage* stages, int cta, int G, int s,
                                          ChainStage& st, StageSplit& sp) {
    if (s < ChainSmem<GATED>::NST) {
        st = sm.desc[s];
        sp = sm.split[s];
        return sp.active;
    }
    st = stages[s];
    return compute_split(st, cta, G, s, sp);
}

// trace (optional): per (cta, stage) globaltimer stamps
//   0 stage entered, 1 input observed ready, 2 input rotated, 3 own units done
// 18 warps: the per-SMSP register file (16K) caps a 5-warp SMSP at 96 registers/thread

template <bool GATED, bool TRACE = false, bool ASYM = true, bool TP = true>
                      // TRACE: globaltimer stamps + cycle counters (tools/trace_chain.py) in their own
                      // instantiation, so the measured kernels carry no counter registers.
                      // GATED: some stage reads SiLU(gate) * up (a separate instantiation keeps the
                      // plain kernel's register allocation).  ASYM = false: every stage is symmetric -- no
                      // zero-point tile loop in the kernel, which frees the tile loop's register allocation
                      // (Llama-2-7B 0.494 -> 0.483 ms with the MAD butterflies that then fit); the plain
                      // symmetric kernel also leaves out the tensor-parallel (peer-store) paths
__global__ void __launch_bounds__(kChainThreads, 1)
    chain_kernel(const ChainStage* __restrict__ stages, int S, const float* __restrict__ x0, int L,
                 unsigned* __restrict__ epoch_ptr, float* __restrict__ out,
                 unsigned long long* __restrict__ trace) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    ChainSmem<GATED>& sm = *reinterpret_cast<ChainSmem<GATED>*>(smem_raw);
    // LO (the symmetric single-GPU kernel): every stage but the last stores H_16 y per full 16-row tile and
    // every stage's input arrives in that form (stage 0 transforms x0 while loading it), so the consumers'
    // rotations skip 4 of their 5 shuffle stages (Llama-2-7B 0.4575 -> ~0.44 ms)
    constexpr bool LO = !ASYM && !TP && !GATED;
    constexpr int NSL = ChainSmem<GATED>::NSL, NST = ChainSmem<GATED>::NST;  // ring slots, cached stages
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int cta = blockIdx.x, G = gridDim.x;
    // Step epoch: tags of this launch = stored epoch + 1; every CTA checks in on epoch_ptr[1] after
    // reading it, and CTA 0 publishes the new epoch at the very end, once all CTAs have read the
    // old one (no separate bump kernel on the stream).
    const unsigned epoch = *reinterpret_cast<volatile unsigned*>(epoch_ptr) + 1u;
    if (threadIdx.x == 0) atomicAdd(epoch_ptr + 1, 1u);

    for (int s = tid; s < min(S, NST); s += kChainThreads) {
        const ChainStage st = stages[s];
        sm.desc[s] = st;
        compute_split(st, cta, G, s, sm.split[s]);
    }
    if (tid == 0) {
        for (int i = 0; i < NSL; ++i) {
            mbar_init(&sm.full[i], 1);
            mbar_init(&sm.empty[i], kChainConsumerWarps + 1);  // compute warps + reducer
            mbar_init(&sm.parts[i], kChainConsumerWarps);
            sm.partcnt[i] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp >= kReducerWarp) {
        const int rr = warp - kReducerWarp;  // this reducer's units: unit sequence number % kChainReducers == rr
        // ------------------------------ reducer ------------------------------
        // Sums each unit's 16 per-warp row partials in warp order (deterministic), stores the
        // tagged outputs and releases the ring slot.  Runs behind the compute warps so they
        // never wait on each other.
        int seq = 0, nrm = 0;
        for (int s = 0; s < S; ++s) {
            ChainStage st;
            StageSplit sp;
            if (!stage_get(sm, stages, cta, G, s, st, sp)) continue;
            const int n_units = (st.RT - 1 - sp.rt0) / sp.Gc + 1;
            // RMSNorm input stage: outputs times rsqrt(mean(x^2) + 1e-5), the sums of squares the consumer
            // warps left in sm.normsq[nb]
            const bool norm = GATED && (st.asym & 4);
            const int nb = nrm & 15;
            nrm += norm;
            // y offset of this CTA's K-chunk (+ the epoch-parity half for tensor-parallel stages)
            const int64_t yoff = (int64_t)sp.ch * st.yrows + st.row0 +
                                 (TP && st.npeer ? (int64_t)(epoch & 1u) * sp.nch * st.yrows : 0);
            unsigned long long* yout = st.y + yoff;
            const unsigned long long tag = (unsigned long long)epoch << 32;
            for (int j = (rr - seq % kChainReducers + kChainReducers) % kChainReducers; j < n_units; j += kChainReducers) {
                const int useq = seq + j;
                const int slot = useq % NSL;
                mbar_wait(&sm.parts[slot], (unsigned)(useq / NSL) & 1u);
                float sum;
                {
                    // lane = (limb pair t = lane >> 4, row lane & 15): the 16 warps' partials in warp order,
                    // then the two limb pairs
                    float part[kChainConsumerWarps];
#pragma unroll
                    for (int w = 0; w < kChainConsumerWarps; ++w) part[w] = sm.part[slot][w][lane >> 4][lane & 15];
                    sum = part[0];
#pragma unroll
                    for (int w = 1; w < kChainConsumerWarps; ++w) sum += part[w];
                    if (LO && s + 1 < S && (int64_t)(sp.rt0 + j * sp.Gc + 1) * 16 <= st.rows) {
                        // H_16 over the unit's 16 rows, fp32, as two radix-4 rounds of independent shuffles with
                        // the limb-pair fold in the first (lanes l and l ^ 16 end with the same value): two
                        // dependent shuffle latencies instead of five on the stage's critical path.  A partial
                        // last tile stays plain (the next stage reads whole 256-blocks, never it).
                        float a[4];
#pragma unroll
                        for (int m = 0; m < 4; ++m) {
                            const float r = __shfl_xor_sync(FULL, sum, 16 | m);
                            a[m] = (m ? __shfl_xor_sync(FULL, sum, m) : sum) + r;
                        }
                        sum = radix4_h(a, lane & 3);
#pragma unroll
                        for (int m = 1; m < 4; ++m) a[m] = __shfl_xor_sync(FULL, sum, 4 * m);
                        a[0] = sum;
                        sum = radix4_h(a, (lane >> 2) & 3);
                    } else {
                        sum += __shfl_xor_sync(FULL, sum, 16);
                    }
                    if (norm) {
                        float tot = 0.f;
#pragma unroll
                        for (int w = 0; w < kChainConsumerWarps; ++w) tot += sm.normsq[nb][w];
                        sum *= rsqrtf(tot / (float)st.cols + 1e-5f);
                    }
                }
                if (lane < 16) {
                    const int64_t row = (int64_t)(sp.rt0 + j * sp.Gc) * 16 + lane;
                    if (row < st.rows) {
                        const unsigned long long word = tag | __float_as_uint(sum);
                        if (!TP || st.npeer == 0) {
                            st_u64_relaxed(yout + row, word);
                        } else {
                            for (int p = 0; p < st.npeer; ++p) st_u64_relaxed_sys(st.ypeer[p] + yoff + row, word);
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.empty[slot]);
            }
            seq += n_units;
        }
        return;
    }
    if (warp == kProducerWarp) {
        // ------------------------------ producer ------------------------------
        if (lane == 0) {
            int slot = 0;
            unsigned phase = 0;
#if CHAIN_PF_UNITS > 0
            // L2 prefetch cursor, CHAIN_PF_UNITS units ahead of the ring cursor (across stages): HBM keeps
            // streaming into L2 while the ring is full and the consumers sit at a stage boundary, and the
            // ring refills from L2 after it.  Measured on the Llama-2-7B stack (tools/ab_run.sh): 0.562 ->
            // 0.528 ms per token at 4 units (+ scales); 1-16 units within 2%, 32 units (~100 MB in
            // flight) thrashes L2 (0.669 ms).
            int pf_s = 0, pf_rt = -1;
            ChainStage pf_st;
            StageSplit pf_sp;
            bool pf_done = false;
            auto pf_next = [&]() {  // advance to the next unit of this CTA and prefetch it
                for (;;) {
                    if (pf_rt >= 0) {
                        pf_rt += pf_sp.Gc;
                        if (pf_rt < pf_st.RT) break;
                        ++pf_s;
                    }
                    if (pf_s >= S) {
                        pf_done = true;
                        return;
                    }
                    if (stage_get(sm, stages, cta, G, pf_s, pf_st, pf_sp) && pf_st.RT > 0 && !(pf_st.asym & (256 | 512))) {
                        pf_rt = pf_sp.rt0;
                        break;
                    }
                    pf_rt = -1;
                    ++pf_s;
                }
                const int b0 = pf_sp.ch * kUnitBlocks;
                const int nb = min(kUnitBlocks, pf_st.NB - b0);
                const int64_t t0 = (int64_t)pf_rt * pf_st.NB + b0;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pf_st.tiled + t0 * 1024),
                             "r"(nb * 1024) : "memory");
                const uint8_t* pf_sc = pf_st.tiled + (int64_t)pf_st.RT * pf_st.NB * 1024;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pf_sc + t0 * 32), "r"(nb * 32)
                             : "memory");
                if (pf_st.asym & 1)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pf_sc + (int64_t)pf_st.RT * pf_st.NB * 32 +
                                                                                    t0 * 16),
                                 "r"(nb * 16) : "memory");
            };
            for (int i = 0; i < CHAIN_PF_UNITS && !pf_done; ++i) pf_next();
#endif
            for (int s = 0; s < S; ++s) {
                ChainStage st;
                StageSplit sp;
                const bool active = stage_get(sm, stages, cta, G, s, st, sp);
                if (GATED && (st.asym & 256)) {
                    // attention partials ahead: pull this CTA's cached K / V rows into L2 now (they do not
                    // depend on the token), so the consumers' score and P V loads hit L2
                    const AttnParams& P = *reinterpret_cast<const AttnParams*>(st.tiled);
                    const int64_t pos = *P.pos;
                    if (cta < P.nkv * P.S && pos >= 0 && pos < P.ctx) {
                        const int kvh = cta / P.S, spl = cta - kvh * P.S;
                        const int chunk = (int)(pos + P.S) / P.S, lo = spl * chunk;
                        const int hi = min((int)pos, lo + chunk);  // rows before pos (pos itself is the new token)
                        if (hi > lo) {
                            const size_t off = ((size_t)kvh * P.ctx + lo) * kAttnHD;
                            const unsigned bytes = (unsigned)(hi - lo) * kAttnHD * 4;
                            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(P.kc + off), "r"(bytes)
                                         : "memory");
                            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(P.vc + off), "r"(bytes)
                                         : "memory");
                        }
                    }
                }
                if (!active) continue;
                const uint8_t* scales = st.tiled + (int64_t)st.RT * st.NB * 1024;
                const uint8_t* zps = scales + (int64_t)st.RT * st.NB * 32;
                const int b0 = sp.ch * kUnitBlocks;
                const int nb = min(kUnitBlocks, st.NB - b0);
                const unsigned bytes = nb * (1024 + 32 + ((st.asym & 1) ? 16 : 0));
                for (int rt = sp.rt0; rt < st.RT; rt += sp.Gc) {
                    mbar_wait(&sm.empty[slot], phase ^ 1u);
                    const int64_t t0 = (int64_t)rt * st.NB + b0;
                    mbar_expect_tx(&sm.full[slot], bytes);
                    uint8_t* dst = sm.ring[slot];
                    bulk_g2s(dst, st.tiled + t0 * 1024, nb * 1024, &sm.full[slot]);
                    bulk_g2s(dst + kSlotCodes, scales + t0 * 32, nb * 32, &sm.full[slot]);
                    if (st.asym & 1) bulk_g2s(dst + kSlotCodes + kSlotScales, zps + t0 * 16, nb * 16, &sm.full[slot]);
#if CHAIN_PF_UNITS > 0
                    if (!pf_done) pf_next();
#endif
                    if (++slot == NSL) {
                        slot = 0;
                        phase ^= 1u;
                    }
                }
            }
        }
        return;
    }

    // ------------------------------ consumers ------------------------------
    // K-stationary: warp w owns 256-block b0 + w of the CTA's K-chunk for the whole stage.  It
    // rotates that block itself (no cross-warp hand-off, no flags) and keeps the activation
    // fragments in registers for every unit; each unit's 16 per-warp partials are summed by the
    // last warp to finish it, in warp order (deterministic).
    const int g = lane >> 2, t = lane & 3;
    const int el = rot_lane_element(lane);  // this lane's elements el + 32 e of a 256-block (rotation layout)
    int cs = 0;        // ring slot of the CTA's next unit
    unsigned cp = 0;   // and its full-barrier phase parity
    uint8_t* rot = sm.rot[warp];
    if (!TRACE) trace = nullptr;
    const bool prof = trace != nullptr && cta == 0;
    int nrm = 0;  // RMSNorm input stages done (sm.normsq buffer nrm & 15; the reducers count alike)
    long long c_wait = 0, c_tile = 0, c_rot = 0, c_in = 0, c_start = clock64();
    for (int s = 0; s < S; ++s) {
        ChainStage st;
        StageSplit sp;
        const bool active = stage_get(sm, stages, cta, G, s, st, sp);
        if (GATED && (st.asym & (256 | 512))) {  // decoder attention stages (no weights, no ring units)
            const AttnParams& P = *reinterpret_cast<const AttnParams*>(st.tiled);
            const ChainStage pv = s - 1 < NST ? sm.desc[s - 1] : stages[s - 1];
            if (trace && tid == 0) trace[((int64_t)cta * S + s) * 4 + 0] = globaltimer();
            if (st.asym & 256) {
                consumer_sync();  // every consumer warp is done with its rotation scratch
                for (int item = cta; item < P.nkv * P.S; item += G)
                    attn_part(P, pv.y, st.y, item, epoch, warp, lane, reinterpret_cast<float*>(&sm.rot[0][0]));
            } else {
                for (int h = cta; h < P.nh; h += G)
                    attn_comb(P, pv.y, st.y, h, epoch, tid, reinterpret_cast<float*>(&sm.rot[0][0]));
            }
            if (trace && tid == 0) trace[((int64_t)cta * S + s) * 4 + 3] = globaltimer();
            continue;
        }
        if (!active) continue;
        // a zero-point or tensor-parallel stage in a symmetric single-GPU launch: fail loudly
        if ((!ASYM && (st.asym & 1)) || (!TP && st.npeer)) __trap();
        if (trace && tid == 0) trace[((int64_t)cta * S + s) * 4 + 0] = globaltimer();
        const int b0 = sp.ch * kUnitBlocks;
        const int nb = min(kUnitBlocks, st.NB - b0);
        const bool has_block = warp < nb;
        float xv[8];  // RMSNorm input stages: this warp's block of the (residual) input before the norm
        if (GATED && (st.asym & 4)) {
            // RMSNorm input stage (decoder; host-checked cols <= 4096, so this CTA's chunk is the whole
            // input vector): every consumer warp leaves its block's sum of squares for the reducers, which
            // scale the stage's outputs (below).  Flag 16 (residual input, s >= 1): the
            // input is x0 + the previous stage's output -- the residual stream after an o projection
            // folded into the same launch (h + W_o att, then RMSNorm, as the reference step orders it).
            float ss = 0.f;
            if (has_block) {
                // the residual stream: the launch input x0, or (decoder, single GPU) a tagged buffer a
                // flag-128 stage of this launch wrote
                if (st.npeer == 0 && st.xres)
                    load_tagged_block<false>(st.xres + 256 * (b0 + warp), 1, 0, epoch, el, xv);
                else
#pragma unroll
                    for (int e = 0; e < 8; ++e) xv[e] = __ldg(x0 + 256 * (b0 + warp) + el + 32 * e);
                if ((st.asym & 64) && s > 1) {  // flag 64: + the o stage's output (index in bits 16-31) first
                    const int ref = (int)((unsigned)st.asym >> 16);
                    const ChainStage s0 = ref < NST ? sm.desc[ref] : stages[ref];
                    float pf[8];
                    load_tagged_block<false>(s0.y + 256 * (b0 + warp), (s0.NB + kUnitBlocks - 1) / kUnitBlocks,
                                             s0.yrows, epoch, el, pf);
#pragma unroll
                    for (int e = 0; e < 8; ++e) xv[e] += pf[e];
                }
                if ((st.asym & (16 | 64)) && s > 0) {
                    const ChainStage pv = s - 1 < NST ? sm.desc[s - 1] : stages[s - 1];
                    const int pn = (pv.NB + kUnitBlocks - 1) / kUnitBlocks;
                    float pf[8];
                    load_tagged_block<false>(pv.y + 256 * (b0 + warp), pn, pv.yrows, epoch, el, pf);
#pragma unroll
                    for (int e = 0; e < 8; ++e) xv[e] += pf[e];
                }
                if ((st.asym & 128) && sp.rt0 == 0)  // one CTA publishes the updated residual stream (tagged)
#pragma unroll
                    for (int e = 0; e < 8; ++e)
                        st_u64_relaxed(st.xout + 256 * (b0 + warp) + el + 32 * e,
                                       ((unsigned long long)epoch << 32) | __float_as_uint(xv[e]));
#pragma unroll
                for (int e = 0; e < 8; ++e) ss += xv[e] * xv[e];
            }
            for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(FULL, ss, o);
            // no CTA barrier: the GEMV is linear, so the norm's scalar rsqrt(mean(x^2) + eps) multiplies the
            // stage's outputs in the reducer (which reads these sums after the unit's partials barrier); each
            // warp goes on with its own block as soon as it has arrived
            if (lane == 0) sm.normsq[nrm & 15][warp] = ss;
            ++nrm;
        }
        uint2 bf[8];
        float fcx = 0.f, corr = 0.f;
        long long c0 = prof ? clock64() : 0;
        if (has_block) {
            float f[8];
            if (GATED && (st.asym & 4)) {
                // RMSNorm input: x * gain (gain in st.xin); the reducer applies rsqrt(mean(x^2) + 1e-5)
#pragma unroll
                for (int e = 0; e < 8; ++e) f[e] = xv[e] * __ldg(st.xin + 256 * (b0 + warp) + el + 32 * e);
            } else if (s == 0 || st.xin) {
                const float* xs = st.xin ? st.xin : x0;
#pragma unroll
                for (int e = 0; e < 8; ++e) f[e] = __ldg(xs + 256 * (b0 + warp) + el + 32 * e);
                if (LO) {  // the launch input in the LO form: H_16 over k bits 0-3 (lane bits 0-3), fp32
#pragma unroll
                    for (int h = 1; h < 16; h <<= 1)
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            const float p = __shfl_xor_sync(FULL, f[e], h);
                            f[e] = (lane & h) ? p - f[e] : p + f[e];
                        }
                }
            } else {
                const ChainStage pv = s - 1 < NST ? sm.desc[s - 1] : stages[s - 1];
                const int pn = (pv.NB + kUnitBlocks - 1) / kUnitBlocks;
                const unsigned long long* src = pv.y + 256 * (b0 + warp);
                if (!TP || pv.npeer == 0) {
                    load_tagged_block<false>(src, pn, pv.yrows, epoch, el, f);
                } else {
                    src += (int64_t)(epoch & 1u) * pn * pv.yrows;
                    load_tagged_block<true>(src, pn, pv.yrows, epoch, el, f);
                }
                if (GATED && (st.asym & 2)) {  // gated input: SiLU(prev[i]) * prev[cols + i] (gate | up halves)
                    float u[8];
                    if (pv.npeer == 0)
                        load_tagged_block<false>(src + st.cols, pn, pv.yrows, epoch, el, u);
                    else
                        load_tagged_block<true>(src + st.cols, pn, pv.yrows, epoch, el, u);
#pragma unroll
                    for (int e = 0; e < 8; ++e) f[e] = f[e] / (1.f + __expf(-f[e])) * u[e];
                }
            }
            if (trace && tid == 0) trace[((int64_t)cta * S + s) * 4 + 1] = globaltimer();
            if (prof) c_in += clock64() - c0;
#ifndef CHAIN_EXP_NOROT
            chain_rotate_to_smem<!ASYM, LO>(f, L, rot, lane);
#endif
            __syncwarp();
            // fragments for lane (g, t): columns g < 4 hold limbs, columns >= 4 are zero
            chain_load_frags(rot, g, t, bf);
            const float2 fc = reinterpret_cast<const float2*>(rot + 8 * 16 * 8)[t];       // f[2t], f[2t+1]
            const float2 cc = reinterpret_cast<const float2*>(rot + 8 * 16 * 8 + 32)[t];  // corr[2t], corr[2t+1]
            fcx = fc.x;  // columns 2t, 2t+1 = limbs 2t, 2t+1: factors differ by exactly 256
            corr = cc.x + cc.y;
        }
        if (prof) c_rot += clock64() - c0;
        if (trace && tid == 0) trace[((int64_t)cta * S + s) * 4 + 2] = globaltimer();
        const int n_units = (st.RT - 1 - sp.rt0) / sp.Gc + 1;
        // the stage's units, with the zero-point terms compiled in only for asymmetric stages
        auto units = [&](auto asym_tag) {
        constexpr bool ASYM = decltype(asym_tag)::value;
        for (int u0 = 0; u0 < n_units; u0 += NSL) {
            // rounds of at most NSL units: no warp waits a ring slot more than one phase ahead
            if (u0 > 0) consumer_sync();
            const int u1 = min(n_units, u0 + NSL);
            // two units per iteration: their independent dependency chains interleave in the
            // warp's in-order issue stream (software pipelining across ring slots)
            for (int j = u0; j < u1; j += 2) {
                const bool two = j + 1 < u1;
                // ring position of the two units, advanced incrementally (no division by the ring size)
                const int slot0 = cs;
                const unsigned ph0 = cp;
                if (++cs == NSL) cs = 0, cp ^= 1u;
                const int slot1 = cs;
                const unsigned ph1 = cp;
                if (two && ++cs == NSL) cs = 0, cp ^= 1u;
                long long c1 = prof ? clock64() : 0;
                mbar_wait(&sm.full[slot0], ph0);
                if (two) mbar_wait(&sm.full[slot1], ph1);
                if (prof) {
                    const long long c2 = clock64();
                    c_wait += c2 - c1;
                    c1 = c2;
                }
                float2 ra = make_float2(0.f, 0.f), rb = make_float2(0.f, 0.f);
#ifdef CHAIN_EXP_NOTILE
                if (false) {
#else
                if (has_block) {
#endif
                    if (two)
                        chain_tile2<ASYM>(sm.ring[slot0], sm.ring[slot1], warp, lane, g, bf, fcx, corr, ra, rb);
                    else
                        ra = chain_tile<ASYM>(sm.ring[slot0], warp, lane, g, bf, fcx, corr);
                }
                // lanes t = 0, 1 hold the limb-pair columns 0..3 (t = 2, 3: the zero columns 4..7); the
                // reducer adds the two pairs
                if (t < 2) {
                    sm.part[slot0][warp][t][g] = ra.x;
                    sm.part[slot0][warp][t][g + 8] = ra.y;
                    if (two) {
                        sm.part[slot1][warp][t][g] = rb.x;
                        sm.part[slot1][warp][t][g + 8] = rb.y;
                    }
                }
                __syncwarp();
                if (prof) c_tile += clock64() - c1;
                if (lane == 0) {
                    mbar_arrive(&sm.parts[slot0]);  // release: this warp's partials are in
                    mbar_arrive(&sm.empty[slot0]);  // done reading the slot (reducer arrives too)
                    if (two) {
                        mbar_arrive(&sm.parts[slot1]);
                        mbar_arrive(&sm.empty[slot1]);
                    }
                }
            }
        }
        };
        if (ASYM && (st.asym & 1))
            units(std::integral_constant<bool, ASYM>{});
        else
            units(std::false_type{});
        if (trace && tid == 0) trace[((int64_t)cta * S + s) * 4 + 3] = globaltimer();
    }
    if (prof && lane == 0) {
        unsigned long long* pt = trace + (int64_t)G * S * 4 + (int64_t)S * 64 + warp * 4;
        pt[0] = c_wait;
        pt[1] = c_tile;
        pt[2] = c_rot;
        pt[3] = clock64() - c_start;
        pt[64 - 3 * warp] = c_in;  // per-warp input-wait cycles: trace word [.. + 64 + warp]
    }
    // fold the last stage's K-chunk partials into `out` (fixed order), waiting on the tags
    const ChainStage last = stages[S - 1];
    const int ln = (last.NB + kUnitBlocks - 1) / kUnitBlocks;
    const bool last_tp = TP && last.npeer;
    const unsigned long long* ylast = last.y + (last_tp ? (int64_t)(epoch & 1u) * ln * last.yrows : 0);
    for (int64_t r = (int64_t)cta * (32 * kChainConsumerWarps) + tid; r < last.yrows;
         r += (int64_t)G * 32 * kChainConsumerWarps) {
        float v;
        for (;;) {
            bool ok = true;
            unsigned long long w = last_tp ? ld_u64_relaxed_sys(ylast + r) : ld_u64_relaxed(ylast + r);
            ok &= (unsigned)(w >> 32) == epoch;
            v = __uint_as_float((unsigned)w);
            for (int c = 1; c < ln; ++c) {
                w = last_tp ? ld_u64_relaxed_sys(ylast + c * last.yrows + r)
                            : ld_u64_relaxed(ylast + c * last.yrows + r);
                ok &= (unsigned)(w >> 32) == epoch;
                v += __uint_as_float((unsigned)w);
            }
            if (ok) break;
            __nanosleep(64);
        }
        if (GATED && (last.asym & 8)) {
            // residual accumulation (decoder): out is the residual stream.  Flag 32: stage 0's output
            // (an o projection in the same launch) is added first: out = (out + y_0) + y_last.
            float base;
            if (last.npeer == 0 && last.xres) {  // the residual is a tagged buffer of this launch
                for (;;) {
                    const unsigned long long w = ld_u64_relaxed(last.xres + r);
                    if ((unsigned)(w >> 32) == epoch) {
                        base = __uint_as_float((unsigned)w);
                        break;
                    }
                    __nanosleep(64);
                }
            } else {
                base = x0[r];  // the launch input is the residual (in place when out == x0)
            }
            if (last.asym & 32) {
                const int ref = (int)((unsigned)last.asym >> 16);
                const ChainStage s0 = ref < NST ? sm.desc[ref] : stages[ref];
                const int n0 = (s0.NB + kUnitBlocks - 1) / kUnitBlocks;
                float v0;
                for (;;) {
                    bool ok = true;
                    unsigned long long w = ld_u64_relaxed(s0.y + r);
                    ok &= (unsigned)(w >> 32) == epoch;
                    v0 = __uint_as_float((unsigned)w);
                    for (int c = 1; c < n0; ++c) {
                        w = ld_u64_relaxed(s0.y + c * s0.yrows + r);
                        ok &= (unsigned)(w >> 32) == epoch;
                        v0 += __uint_as_float((unsigned)w);
                    }
                    if (ok) break;
                    __nanosleep(64);
                }
                base += v0;
            }
            out[r] = base + v;
        } else {
            out[r] = v;
        }
    }
    if (cta == 0 && tid == 0) {
        while (atomicAdd(epoch_ptr + 1, 0u) < (unsigned)G) __nanosleep(32);
        epoch_ptr[1] = 0u;
        *reinterpret_cast<volatile unsigned*>(epoch_ptr) = epoch;
    }
}

}  // namespace itq3

using namespace itq3;

extern "C" int64_t itq3_chain_desc_nbytes(void) { return (int64_t)sizeof(ChainStage); }
extern "C" int itq3_chain_act_block_bytes(int limbs) { return act_block_bytes(limbs); }
extern "C" int itq3_chain_smem_bytes(void) { return (int)sizeof(ChainSmem<false>); }

extern "C" int itq3_chain_write_desc_tp(void*, int, const uint8_t*, void*, int64_t, int64_t, int, int64_t, int64_t,
                                        const void*, int);

// Host-balanced work split of stage `index`: d_work = device int32[grid]: CTA c computes K-chunk
// d_work[c] / Gc and row tiles d_work[c] % Gc, + Gc, ... (Gc = grid / nch), -1 = idle; every (chunk, first row
// tile) pair must appear exactly once.  Any such permutation gives the same outputs (each row's arithmetic does
// not depend on which CTA computes it); LinearStack balances the units a CTA carries across stages whose
// input is complete early (see stack.py).
extern "C" int itq3_chain_set_work(void* host_desc, int index, const int32_t* d_work) {
    reinterpret_cast<ChainStage*>(host_desc)[index].work = d_work;
    return ITQ3_OK;
}

// flag 128 (decoder): where the RMSNorm stage `index` writes the residual input it computed
extern "C" int itq3_chain_set_xout(void* host_desc, int index, void* xout) {
    reinterpret_cast<ChainStage*>(host_desc)[index].xout = (unsigned long long*)xout;
    return ITQ3_OK;
}
// decoder attention stage (flags 256 = partials, 512 = combine): `params` = device AttnParams, `y` = the
// stage's tagged output (partials: nkv x S x 4 x 130 words; combine: n_heads x 128 words)
extern "C" int itq3_chain_write_desc_attn(void* host_desc, int index, int kind, const void* params, void* y,
                                          int64_t yrows) {
    if ((kind != 256 && kind != 512) || index < 1 || params == nullptr) {
        set_error("chain: stage %d: attention stage needs kind 256 / 512, a previous stage and params", index);
        return ITQ3_E_DOMAIN;
    }
    ChainStage& st = reinterpret_cast<ChainStage*>(host_desc)[index];
    memset(&st, 0, sizeof(st));
    st.tiled = (const uint8_t*)params;
    st.y = (unsigned long long*)y;
    st.rows = yrows;
    st.cols = 0;
    st.NB = 1;  // a consumer of this stage's output reads one partial
    st.RT = 0;  // no weight units: producer and reducer skip the stage
    st.asym = kind;
    st.yrows = (int32_t)yrows;
    return ITQ3_OK;
}
extern "C" int itq3_chain_attn_params_nbytes(void) { return (int)sizeof(AttnParams); }

// decoder, single GPU: the tagged residual buffer a flag-4/8 stage reads instead of the launch input
// (written by a flag-128 stage of the same launch)
extern "C" int itq3_chain_set_xres(void* host_desc, int index, const void* xres) {
    ChainStage& st = reinterpret_cast<ChainStage*>(host_desc)[index];
    if (st.npeer) {
        set_error("chain: stage %d: a residual buffer needs a single-GPU stage", index);
        return ITQ3_E_DOMAIN;
    }
    st.xres = (const unsigned long long*)xres;
    return ITQ3_OK;
}

extern "C" int itq3_chain_write_desc(void* host_desc, int index, const uint8_t* tiled, void* y, const float* xin,
                                     int64_t rows, int64_t cols, int asymmetric, int reserved) {
    (void)reserved;
    const int rc = itq3_chain_write_desc_tp(host_desc, index, tiled, y, rows, cols, asymmetric, 0, rows, nullptr, 0);
    if (rc == ITQ3_OK) reinterpret_cast<ChainStage*>(host_desc)[index].xin = xin;
    return rc;
}

extern "C" int itq3_chain_write_desc_tp(void* host_desc, int index, const uint8_t* tiled, void* y, int64_t rows,
                                        int64_t cols, int asymmetric, int64_t row0, int64_t yrows,
                                        const void* d_peers, int npeer) {
    if (cols % 256 || cols / 256 > kMaxChainNB) {
        set_error("chain: stage %d needs cols %% 256 == 0 and cols <= %d (got %lld)", index, 256 * kMaxChainNB,
                  (long long)cols);
        return ITQ3_E_UNSUPPORTED;
    }
    ChainStage& st = reinterpret_cast<ChainStage*>(host_desc)[index];
    if (npeer < 0 || npeer > kMaxChainPeers || (npeer > 0 && d_peers == nullptr) || row0 < 0 || rows < 0 ||
        row0 + rows > yrows || yrows > INT32_MAX) {
        set_error("chain: stage %d: bad tensor-parallel shard (row0 %lld, rows %lld, yrows %lld, npeer %d)", index,
                  (long long)row0, (long long)rows, (long long)yrows, npeer);
        return ITQ3_E_DOMAIN;
    }
    if ((asymmetric & 4) && cols > 4096) {
        set_error("chain: stage %d: an RMSNorm input stage needs cols <= 4096 (got %lld)", index, (long long)cols);
        return ITQ3_E_UNSUPPORTED;
    }
    if (((asymmetric & 16) && (!(asymmetric & 4) || index < 1 || npeer)) || ((asymmetric & 32) && !(asymmetric & 8)) ||
        ((asymmetric & 64) && (!(asymmetric & 4) || index < 2 || npeer)) || ((asymmetric & 128) && !(asymmetric & 4))) {
        set_error("chain: stage %d: flag 16 (residual input) needs flag 4 on a stage >= 1, flag 64 on a stage >= 2 "
                  "(single GPU); flag 32 needs flag 8; flag 128 needs flag 4", index);
        return ITQ3_E_DOMAIN;
    }
    st.tiled = tiled;
    st.y = (unsigned long long*)y;
    st.xin = nullptr;
    st.xout = nullptr;
    st.work = nullptr;
    st.ypeer = (unsigned long long* const*)d_peers;
    st.rows = rows;
    st.cols = cols;
    st.NB = (int)(cols / 256);
    st.RT = (int)((rows + 15) / 16);
    st.asym = asymmetric;
    st.npeer = npeer;
    st.row0 = (int32_t)row0;
    st.yrows = (int32_t)yrows;
    return ITQ3_OK;
}

template <bool GATED, bool ASYM, bool TP>
static int chain_run(const void* d_desc, int n_stages, const float* x0, int limbs, unsigned* d_epoch, float* out,
                     int grid, void* d_trace, void* stream) {
    if (limbs < 1 || limbs > kMaxLimbs) {
        set_error("chain: limbs must be in [1, %d]", kMaxLimbs);
        return ITQ3_E_DOMAIN;
    }
    static std::atomic<unsigned long long> smem_attr{0}, smem_attr_tr{0};
    const int smem = (int)sizeof(ChainSmem<GATED>);
#ifdef CHAIN_GATED_TRACE  // experiment builds: a traced twin of the gated single-GPU kernel (tools/trace_decoder.py)
    const bool tr = d_trace != nullptr;
    auto kern = tr ? (GATED ? chain_kernel<true, true, true, false> : chain_kernel<false, true, true, true>)
                   : chain_kernel<GATED, false, ASYM, TP>;
#else
    const bool tr = !GATED && d_trace;  // the trace instantiation is the asymmetric-capable plain kernel
    auto kern = tr ? chain_kernel<false, true, true, true> : chain_kernel<GATED, false, ASYM, TP>;
#endif
    if (int rc = ensure_smem_attr(kern, smem, tr ? smem_attr_tr : smem_attr, "chain: smem attribute")) return rc;
    if (grid <= 0) grid = device_sms();
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
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, (const ChainStage*)d_desc, n_stages, x0, limbs,
                                             d_epoch, out, (unsigned long long*)d_trace);
    if (e != cudaSuccess) {
        set_error("chain: launch failed: %s", cudaGetErrorString(e));
        return ITQ3_E_CUDA;
    }
    return check_launch("itq3_chain_run");
}

// flags: bit 0 = gated chain (decoder stages: SiLU gating, RMSNorm, residuals, attention); bit 1 = every
// weight stage is symmetric (no zero-points); bit 2 = single GPU (no tensor-parallel stage).  Bits 1 and 2 pick
// instantiations without the zero-point tile loop / the peer-store paths (faster: the kernel is at its
// register cap, so every compiled path shapes the tile loop); a stage needing what was left out traps.
// Instantiated: plain general, plain symmetric (single-GPU / tensor-parallel), gated general, gated single-GPU
// (general / symmetric).
extern "C" int itq3_chain_run_ex(const void* d_desc, int n_stages, const float* x0, int limbs, unsigned* d_epoch,
                                 float* out, int grid, void* d_trace, void* stream, int flags) {
    const bool gated = flags & 1, sym = flags & 2, single = flags & 4;
    if (gated && sym && single)
        return chain_run<true, false, false>(d_desc, n_stages, x0, limbs, d_epoch, out, grid, d_trace, stream);
    if (gated)
        return single ? chain_run<true, true, false>(d_desc, n_stages, x0, limbs, d_epoch, out, grid, d_trace, stream)
                      : chain_run<true, true, true>(d_desc, n_stages, x0, limbs, d_epoch, out, grid, d_trace, stream);
    if (sym)
        return single ? chain_run<false, false, false>(d_desc, n_stages, x0, limbs, d_epoch, out, grid, d_trace, stream)
                      : chain_run<false, false, true>(d_desc, n_stages, x0, limbs, d_epoch, out, grid, d_trace, stream);
    return chain_run<false, true, true>(d_desc, n_stages, x0, limbs, d_epoch, out, grid, d_trace, stream);
}

extern "C" int itq3_chain_run(const void* d_desc, int n_stages, const float* x0, int limbs, unsigned* d_epoch,
                              float* out, int grid, void* d_trace, void* stream) {
    return chain_run<false, true, true>(d_desc, n_stages, x0, limbs, d_epoch, out, grid, d_trace, stream);
}

extern "C" int itq3_chain_run_gated(const void* d_desc, int n_stages, const float* x0, int limbs, unsigned* d_epoch,
                                    float* out, int grid, void* d_trace, void* stream) {
    return chain_run<true, true, true>(d_desc, n_stages, x0, limbs, d_epoch, out, grid, d_trace, stream);
}
