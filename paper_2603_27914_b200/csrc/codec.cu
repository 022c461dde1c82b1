// K1 encoder, K2 dequantiser, K7 validator and the FWHT transform (sm_100a).
//
// Bit-exactness contract: every floating-point step replays the
// reference's binary64 data flow -- radix-2 butterfly with ascending stages
// (transform.py:46-58), numpy pairwise summation (quantizer.py:85-86), correctly rounded
// sqrt / division, single-rounding binary16 (packing.py:87-101), round-half-away with the
// rounded addition (quantizer.py:152-168).  All arithmetic uses explicit _rn intrinsics so
// the compiler cannot contract or reassociate it.
//
// Thread mapping: one warp per block; element j of the block lives in lane j % 32, slot
// j / 32 ("stride layout").  Butterfly stages h < 32 are xor shuffles, h >= 32 are
// register pairs.  With that layout __ballot_sync of bit b of the stored code returns the
// little-endian plane word directly (packing.py:59-64: bit j -> byte j/8, bit j%8).
#include "common.cuh"

namespace itq3 {

// ------------------------------------------------------------------------------------------
// K1: encoder.  encode_block (codec.py:113-149) for every block of the flattened tensor.
// ------------------------------------------------------------------------------------------
constexpr int kEncWarps = 4;

template <int N, typename TIn>
__global__ void __launch_bounds__(32 * kEncWarps) encode_kernel(const TIn* __restrict__ w, int64_t numel,
                                                                int64_t n_blocks, int ss, int policy,
                                                                double coeff, int symmetric,
                                                                uint8_t* __restrict__ payload) {
    constexpr int E = N / 32;
    constexpr int M = N / kSubBlocks;  // sub-block length
    __shared__ double sm_all[kEncWarps][2 * N];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t blk = (int64_t)blockIdx.x * kEncWarps + wid;
    if (blk >= n_blocks) return;
    double* ys = sm_all[wid];
    double* sq = ys + N;

    double v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int64_t gi = blk * N + lane + 32 * e;
        v[e] = gi < numel ? (double)w[gi] : 0.0;  // zero tail pad (codec.py:175-179)
    }
    warp_butterfly<E>(v, lane);
    const double norm = __ddiv_rn(1.0, __dsqrt_rn((double)N));  // 1.0 / math.sqrt(n)
#pragma unroll
    for (int e = 0; e < E; ++e) {
        v[e] = __dmul_rn(v[e], norm);
        ys[lane + 32 * e] = v[e];
    }
    __syncwarp();
    const double mean = __ddiv_rn(warp_pairwise_sum(ys, N, lane), (double)N);

    uint8_t* out = payload + blk * block_nbytes(N, ss);
    double z = 0.0;
    double deff_e[E];
    uint16_t scale_bits;

    auto effective = [](double d_raw, uint16_t bits) {
        const double d16 = f16_bits_to_f64(bits);
        return d16 > 0.0 ? d16 : d_raw;  // codec.py:95-103
    };
    auto zero_point = [&](double d_eff) {  // codec.py:106-110
        if (symmetric) return 0.0;
        const double r = __ddiv_rn(mean, d_eff);
        return __dadd_rn(clip1(-copysign(floor(__dadd_rn(fabs(r), 0.5)), r)), 0.0);
    };

    if (!ss) {
        double d;
        if (policy == ITQ3_POLICY_MEAN_ABS) {
#pragma unroll
            for (int e = 0; e < E; ++e) sq[lane + 32 * e] = fabs(v[e]);
            __syncwarp();
            const double l1 = warp_pairwise_sum(sq, N, lane);
            d = __dmul_rn(2.0 / 3.0, __ddiv_rn(l1, (double)N));
        } else {
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const double c = __dsub_rn(v[e], mean);
                sq[lane + 32 * e] = __dmul_rn(c, c);
            }
            __syncwarp();
            const double var = __ddiv_rn(warp_pairwise_sum(sq, N, lane), (double)N);
            d = __dmul_rn(coeff, __dsqrt_rn(var));
        }
        const double d_raw = d > 0.0 ? d : 1e-8;  // EPSILON_D (quantizer.py:28,149)
        scale_bits = f64_to_f16_bits(d_raw);
        const double d_eff = effective(d_raw, scale_bits);
        z = zero_point(d_eff);
#pragma unroll
        for (int e = 0; e < E; ++e) deff_e[e] = d_eff;
    } else {
        // per-sub-block statistics (codec.py:134-149): lane s < 8 owns sub-block s
        double d_raw_s = 0.0;
        double mean_s = 0.0;
        if (lane < kSubBlocks) mean_s = __ddiv_rn(serial_pairwise_sum(ys + lane * M, M), (double)M);
        if (policy == ITQ3_POLICY_MEAN_ABS) {
#pragma unroll
            for (int e = 0; e < E; ++e) sq[lane + 32 * e] = fabs(v[e]);
        } else {
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int j = lane + 32 * e;
                const double mu = __shfl_sync(FULL, mean_s, j / M);
                const double c = __dsub_rn(v[e], mu);
                sq[j] = __dmul_rn(c, c);
            }
        }
        __syncwarp();
        if (lane < kSubBlocks) {
            double d;
            const double s = __ddiv_rn(serial_pairwise_sum(sq + lane * M, M), (double)M);
            if (policy == ITQ3_POLICY_MEAN_ABS) d = __dmul_rn(2.0 / 3.0, s);
            else d = __dmul_rn(coeff, __dsqrt_rn(s));
            d_raw_s = d > 0.0 ? d : 1e-8;
        }
        const uint16_t sub_bits = f64_to_f16_bits(d_raw_s);
        const double d_eff_s = effective(d_raw_s, sub_bits);
        // d_block = np.mean(d_raws): pairwise over 8 values, identity 0
        double r8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) r8[k] = __shfl_sync(FULL, d_raw_s, k);
        const double d_block = __ddiv_rn(serial_pairwise_sum(r8, 8), 8.0);
        scale_bits = f64_to_f16_bits(d_block);
        z = zero_point(effective(d_block, scale_bits));
#pragma unroll
        for (int e = 0; e < E; ++e) deff_e[e] = __shfl_sync(FULL, d_eff_s, (lane + 32 * e) / M);
        if (lane < kSubBlocks) {
            const int off = 3 * N / 8 + 4 + 2 * lane;
            *reinterpret_cast<uint16_t*>(out + off) = sub_bits;
        }
    }

    // ternary_quantize (quantizer.py:156-168) and pack_ternary (packing.py:59-64).
    // code = clip(round_half_away(fl(y / d)) + z, -1, 1) only depends on which side of 0.5 and 1.5
    // |fl(y / d)| falls, so a multiply by fl(1 / d) (within 2^-50 of the quotient for |q| <= 2)
    // decides every element farther than 2^-40 from those two points; the rest (and the SS
    // variant, whose scale varies per element) take the correctly rounded division.
    uint32_t c[E];
    const double inv = ss ? 0.0 : __drcp_rn(deff_e[0]);
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const double a = fabs(v[e]) * inv;
        double code;
        if (!ss && fabs(a - 0.5) > 0x1p-40 && fabs(a - 1.5) > 0x1p-40) {
            const double rr = a >= 1.5 ? 2.0 : (a >= 0.5 ? 1.0 : 0.0);
            code = clip1(__dadd_rn(copysign(rr, v[e]), z));
        } else {
            const double q = __ddiv_rn(v[e], deff_e[e]);
            code = clip1(__dadd_rn(round_half_away(q), z));
        }
        c[e] = (uint32_t)((int)code + 1);
    }
#pragma unroll
    for (int b = 0; b < 3; ++b) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const uint32_t word = __ballot_sync(FULL, (c[e] >> b) & 1u);
            if (lane == ((b * E + e) & 31)) *reinterpret_cast<uint32_t*>(out + b * (N / 8) + 4 * e) = word;
        }
    }
    if (lane == 0) {
        *reinterpret_cast<uint16_t*>(out + 3 * N / 8) = scale_bits;
        *reinterpret_cast<uint16_t*>(out + 3 * N / 8 + 2) = f64_to_f16_bits(z);
    }
}

// ------------------------------------------------------------------------------------------
// K7: validation (deserialize_block / unpack_ternary checks, packing.py:67-84,171-197)
// ------------------------------------------------------------------------------------------
__global__ void validate_kernel(const uint8_t* __restrict__ payload, int64_t n_blocks, int N, int ss,
                                uint32_t mask, unsigned long long* first_bad) {
    const int lane = threadIdx.x & 31;
    const int64_t blk = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (blk >= n_blocks) return;
    const uint8_t* p = payload + blk * block_nbytes(N, ss);
    const int W = N / 32;  // words per plane (1..16)
    unsigned long long key = ~0ull;
    if ((mask & ITQ3_CHECK_PLANES) && lane < W) {
        const uint32_t p0 = *reinterpret_cast<const uint32_t*>(p + 4 * lane);
        const uint32_t p1 = *reinterpret_cast<const uint32_t*>(p + N / 8 + 4 * lane);
        const uint32_t p2 = *reinterpret_cast<const uint32_t*>(p + N / 4 + 4 * lane);
        const uint32_t bad = p2 | (p0 & p1);
        if (bad) key = ((unsigned long long)blk << 16) | (unsigned long long)(32 * lane + __ffs(bad) - 1);
    }
    if (lane == 0) {
        const uint16_t sb = *reinterpret_cast<const uint16_t*>(p + 3 * N / 8);
        const uint16_t zb = *reinterpret_cast<const uint16_t*>(p + 3 * N / 8 + 2);
        unsigned long long k2 = ~0ull;
        if ((mask & ITQ3_CHECK_SCALE_NAN) && (sb & 0x7fff) > 0x7c00) k2 = 1;
        else if ((mask & ITQ3_CHECK_ZP) && !(zb == 0 || zb == 0x8000 || zb == 0x3C00 || zb == 0xBC00)) k2 = 2;
        else if ((mask & ITQ3_CHECK_ZP_FINITE) && (zb & 0x7c00) == 0x7c00) k2 = 4;
        if (k2 == ~0ull && ss && (mask & ITQ3_CHECK_SUB_NAN)) {
            for (int s = 0; s < kSubBlocks; ++s) {
                const uint16_t b = *reinterpret_cast<const uint16_t*>(p + 3 * N / 8 + 4 + 2 * s);
                if ((b & 0x7fff) > 0x7c00) { k2 = 3; break; }
            }
        }
        if (k2 != ~0ull) {
            const unsigned long long kk = ((unsigned long long)blk << 16) | (k2 << 10);
            key = kk < key ? kk : key;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(FULL, key, o);
        key = other < key ? other : key;
    }
    if (lane == 0 && key != ~0ull) atomicMin(first_bad, key);
}

// K7 fast path (block_n 256, variant s): one THREAD per 100-byte block.  The warp stages its 32
// consecutive blocks (3200 contiguous bytes) with 16-byte coalesced loads into shared memory, each
// thread checks its own block from there (25 words, stride 25: conflict-free), and only offenders
// touch the atomic -- no shuffles, so the pass runs at HBM speed.
__global__ void __launch_bounds__(256) validate256_kernel(const uint8_t* __restrict__ payload, int64_t n_blocks,
                                                          uint32_t mask, unsigned long long* first_bad) {
    __shared__ uint32_t stage[8][32 * 25];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t blk0 = ((int64_t)blockIdx.x * 8 + w) * 32;
    if (blk0 >= n_blocks) return;
    const int nb = (int)(n_blocks - blk0 < 32 ? n_blocks - blk0 : 32);
    const uint8_t* src = payload + blk0 * 100;
    uint32_t* st = stage[w];
    if (nb == 32 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
#pragma unroll
        for (int i = 0; i < 7; ++i) {
            const int c = lane + 32 * i;  // 16-byte chunk of the warp's 3200 bytes
            if (c < 200) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(src) + c);
                st[4 * c] = v.x, st[4 * c + 1] = v.y, st[4 * c + 2] = v.z, st[4 * c + 3] = v.w;
            }
        }
    } else {
        for (int c = lane; c < nb * 25; c += 32) st[c] = __ldg(reinterpret_cast<const uint32_t*>(src) + c);
    }
    __syncwarp();
    if (lane >= nb) return;
    const uint32_t* b = st + 25 * lane;
    const int64_t blk = blk0 + lane;
    unsigned long long key = ~0ull;
    if (mask & ITQ3_CHECK_PLANES) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t bad = b[16 + i] | (b[i] & b[8 + i]);
            if (bad) {
                key = ((unsigned long long)blk << 16) | (unsigned long long)(32 * i + __ffs(bad) - 1);
                break;
            }
        }
    }
    const uint16_t sb = (uint16_t)(b[24] & 0xffffu), zb = (uint16_t)(b[24] >> 16);
    unsigned long long k2 = ~0ull;
    if ((mask & ITQ3_CHECK_SCALE_NAN) && (sb & 0x7fff) > 0x7c00) k2 = 1;
    else if ((mask & ITQ3_CHECK_ZP) && !(zb == 0 || zb == 0x8000 || zb == 0x3C00 || zb == 0xBC00)) k2 = 2;
    else if ((mask & ITQ3_CHECK_ZP_FINITE) && (zb & 0x7c00) == 0x7c00) k2 = 4;
    if (k2 != ~0ull) {
        const unsigned long long kk = ((unsigned long long)blk << 16) | (k2 << 10);
        key = kk < key ? kk : key;
    }
    if (key != ~0ull) atomicMin(first_bad, key);
}

// ------------------------------------------------------------------------------------------
// K2 (generic): decode_block (codec.py:152-161) in binary64 with the reference's data flow.
// One warp per block; bit-exact for every block size and variant.
// ------------------------------------------------------------------------------------------
template <int N, typename TOut>
__global__ void __launch_bounds__(256) dequant_kernel(const uint8_t* __restrict__ payload, int64_t n_blocks, int ss,
                                                      int64_t numel, TOut* __restrict__ out) {
    constexpr int E = N / 32;
    const int lane = threadIdx.x & 31;
    const int64_t blk = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (blk >= n_blocks) return;
    const uint8_t* p = payload + blk * block_nbytes(N, ss);
    const uint16_t sb = *reinterpret_cast<const uint16_t*>(p + 3 * N / 8);
    const uint16_t zb = *reinterpret_cast<const uint16_t*>(p + 3 * N / 8 + 2);
    const double z = trunc(f16_bits_to_f64(zb));  // PackedBlock.zp = int(decode_f16(...))
    double scale = f16_bits_to_f64(sb);
    double v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int j = lane + 32 * e;
        const uint32_t p0 = *reinterpret_cast<const uint32_t*>(p + 4 * e);
        const uint32_t p1 = *reinterpret_cast<const uint32_t*>(p + N / 8 + 4 * e);
        const uint32_t p2 = *reinterpret_cast<const uint32_t*>(p + N / 4 + 4 * e);
        const int c = (int)((p0 >> lane) & 1u) + 2 * (int)((p1 >> lane) & 1u) + 4 * (int)((p2 >> lane) & 1u);
        if (ss) scale = f16_bits_to_f64(*reinterpret_cast<const uint16_t*>(p + 3 * N / 8 + 4 + 2 * (j / (N / 8))));
        v[e] = __dmul_rn(scale, __dsub_rn((double)(c - 1), z));
    }
    warp_butterfly<E>(v, lane);
    const double norm = __ddiv_rn(1.0, __dsqrt_rn((double)N));
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int64_t gi = blk * N + lane + 32 * e;
        if (gi < numel) out[gi] = (TOut)__dmul_rn(v[e], norm);
    }
}

// ------------------------------------------------------------------------------------------
// FWHT over contiguous vectors (fwht_forward / fwht_inverse, transform.py:61-96)
// ------------------------------------------------------------------------------------------
template <int N, typename T>
__global__ void __launch_bounds__(256) fwht_warp_kernel(const T* __restrict__ in, T* __restrict__ out,
                                                        int64_t n_vec, int normalize, T norm) {
    constexpr int E = N / 32;
    const int lane = threadIdx.x & 31;
    const int64_t vec = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (vec >= n_vec) return;
    T v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = in[vec * N + lane + 32 * e];
    warp_butterfly<E>(v, lane);
#pragma unroll
    for (int e = 0; e < E; ++e) out[vec * N + lane + 32 * e] = normalize ? mul_rn(v[e], norm) : v[e];
}

template <typename T>
__global__ void fwht_small_kernel(const T* __restrict__ in, T* __restrict__ out, int64_t n_vec, int n,
                                  int normalize, T norm) {
    const int64_t vec = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (vec >= n_vec) return;
    T v[16];
    for (int j = 0; j < n; ++j) v[j] = in[vec * n + j];
    for (int h = 1; h < n; h <<= 1)
        for (int j = 0; j < n; ++j)
            if ((j & h) == 0) {
                const T lo = v[j], hi = v[j + h];
                v[j] = add_rn(lo, hi);
                v[j + h] = sub_rn(lo, hi);
            }
    for (int j = 0; j < n; ++j) out[vec * n + j] = normalize ? mul_rn(v[j], norm) : v[j];
}

}  // namespace itq3

using namespace itq3;

// ==========================================================================================
// C ABI
// ==========================================================================================
template <typename TIn>
static int launch_encode(const TIn* w, int64_t numel, int n, int64_t nb, int ss, int policy, double coeff, int sym,
                         uint8_t* payload, cudaStream_t s) {
    const dim3 grid((unsigned)((nb + kEncWarps - 1) / kEncWarps)), block(32 * kEncWarps);
    switch (n) {
        case 32: encode_kernel<32, TIn><<<grid, block, 0, s>>>(w, numel, nb, ss, policy, coeff, sym, payload); break;
        case 64: encode_kernel<64, TIn><<<grid, block, 0, s>>>(w, numel, nb, ss, policy, coeff, sym, payload); break;
        case 128: encode_kernel<128, TIn><<<grid, block, 0, s>>>(w, numel, nb, ss, policy, coeff, sym, payload); break;
        case 256: encode_kernel<256, TIn><<<grid, block, 0, s>>>(w, numel, nb, ss, policy, coeff, sym, payload); break;
        case 512: encode_kernel<512, TIn><<<grid, block, 0, s>>>(w, numel, nb, ss, policy, coeff, sym, payload); break;
    }
    return check_launch("itq3_encode");
}

extern "C" int itq3_encode(const void* w, int w_dtype, int64_t numel, int block_n, int sub_scales, int policy,
                           double coeff, int symmetric, uint8_t* payload, void* stream) {
    if (!valid_block_n(block_n)) {
        set_error("itq3_encode: block_n must be one of (32, 64, 128, 256, 512), got %d", block_n);
        return ITQ3_E_DOMAIN;
    }
    if (numel <= 0) {
        set_error("itq3_encode: expected a non-empty tensor");
        return ITQ3_E_SHAPE;
    }
    if (policy < 0 || policy > 2 || !(coeff > 0.0)) {
        set_error("itq3_encode: bad scale policy %d / coefficient %g", policy, coeff);
        return ITQ3_E_DOMAIN;
    }
    const int64_t nb = (numel + block_n - 1) / block_n;
    cudaStream_t s = (cudaStream_t)stream;
    if (w_dtype == ITQ3_F32)
        return launch_encode((const float*)w, numel, block_n, nb, sub_scales, policy, coeff, symmetric, payload, s);
    if (w_dtype == ITQ3_F64)
        return launch_encode((const double*)w, numel, block_n, nb, sub_scales, policy, coeff, symmetric, payload, s);
    set_error("itq3_encode: weights must be float32 or float64");
    return ITQ3_E_DOMAIN;
}

extern "C" int itq3_validate(const uint8_t* payload, int64_t n_blocks, int block_n, int sub_scales,
                             uint32_t check_mask, unsigned long long* d_first_bad, void* stream) {
    if (!valid_block_n(block_n)) {
        set_error("itq3_validate: invalid block_n %d", block_n);
        return ITQ3_E_DOMAIN;
    }
    if (n_blocks <= 0) return ITQ3_OK;
    const int64_t threads = n_blocks * 32;
    if (block_n == 256 && !sub_scales) {
        validate256_kernel<<<(unsigned)((n_blocks + 255) / 256), 256, 0, (cudaStream_t)stream>>>(payload, n_blocks,
                                                                                               check_mask, d_first_bad);
        return check_launch("itq3_validate");
    }
    validate_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        payload, n_blocks, block_n, sub_scales, check_mask, d_first_bad);
    return check_launch("itq3_validate");
}

// The exact pass behind the tensor-core dequantiser (dequant.cu): a warp screens 32 blocks at a
// time (one lane each) and decodes, with the reference's float64 data flow, only the blocks that
// path leaves out (scale zero, negative, inf or NaN; zero-point other than +-0 / +-1) -- normally none.
template <typename TOut>
__global__ void __launch_bounds__(256) dequant_fixup_kernel(const uint8_t* __restrict__ payload, int64_t n_blocks,
                                                            int64_t numel, TOut* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t b0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; b0 < n_blocks; b0 += nwarps * 32) {
        const int64_t bl = b0 + lane;
        bool unsafe = false;
        if (bl < n_blocks) {
            const uint32_t w = *reinterpret_cast<const uint32_t*>(payload + bl * 100 + 96);
            const uint16_t sb = (uint16_t)(w & 0xffffu), zb = (uint16_t)(w >> 16);
            unsafe = !(sb != 0 && !(sb & 0x8000) && (sb & 0x7c00) != 0x7c00 &&
                       (zb == 0 || zb == 0x8000 || zb == 0x3C00 || zb == 0xBC00));
        }
        uint32_t m = __ballot_sync(FULL, unsafe);
        while (m) {
            const int64_t blk = b0 + __ffs(m) - 1;
            m &= m - 1;
            const uint8_t* p = payload + blk * 100;
            const uint16_t sb = *reinterpret_cast<const uint16_t*>(p + 96);
            const uint16_t zb = *reinterpret_cast<const uint16_t*>(p + 98);
            const double z = trunc(f16_bits_to_f64(zb));
            const double scale = f16_bits_to_f64(sb);
            double v[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const uint32_t p0 = *reinterpret_cast<const uint32_t*>(p + 4 * e);
                const uint32_t p1 = *reinterpret_cast<const uint32_t*>(p + 32 + 4 * e);
                const uint32_t p2 = *reinterpret_cast<const uint32_t*>(p + 64 + 4 * e);
                const int c = (int)((p0 >> lane) & 1u) + 2 * (int)((p1 >> lane) & 1u) + 4 * (int)((p2 >> lane) & 1u);
                v[e] = __dmul_rn(scale, __dsub_rn((double)(c - 1), z));
            }
            warp_butterfly<8>(v, lane);
            const double norm = __ddiv_rn(1.0, __dsqrt_rn(256.0));
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int64_t gi = blk * 256 + lane + 32 * e;
                if (gi < numel) out[gi] = (TOut)__dmul_rn(v[e], norm);
            }
        }
    }
}

template <typename TOut>
int itq3_dequant_tc(const uint8_t* payload, int64_t n_blocks, int64_t numel, TOut* out, cudaStream_t s);

template <typename TOut>
static int launch_dequant(const uint8_t* payload, int64_t nb, int n, int ss, int64_t numel, TOut* out,
                          cudaStream_t s) {
    const unsigned grid = (unsigned)((nb * 32 + 255) / 256);
    if (n == 256 && !ss) {  // tensor-core IFWHT (dequant.cu) + exact pass for the blocks it leaves out
        const int rc = itq3_dequant_tc<TOut>(payload, nb, numel, out, s);
        if (rc) return rc;
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
        const int64_t want = (nb + 255) / 256;
        const unsigned fgrid = (unsigned)(want < 8 * sms ? (want > 0 ? want : 1) : 8 * sms);
        dequant_fixup_kernel<TOut><<<fgrid, 256, 0, s>>>(payload, nb, numel, out);
        return check_launch("itq3_dequant (exact pass)");
    }
    switch (n) {
        case 32: dequant_kernel<32, TOut><<<grid, 256, 0, s>>>(payload, nb, ss, numel, out); break;
        case 64: dequant_kernel<64, TOut><<<grid, 256, 0, s>>>(payload, nb, ss, numel, out); break;
        case 128: dequant_kernel<128, TOut><<<grid, 256, 0, s>>>(payload, nb, ss, numel, out); break;
        case 256: dequant_kernel<256, TOut><<<grid, 256, 0, s>>>(payload, nb, ss, numel, out); break;
        case 512: dequant_kernel<512, TOut><<<grid, 256, 0, s>>>(payload, nb, ss, numel, out); break;
    }
    return check_launch("itq3_dequant");
}

extern "C" int itq3_dequant(const uint8_t* payload, int64_t n_blocks, int block_n, int sub_scales, int64_t numel,
                            void* out, int out_dtype, void* stream) {
    if (!valid_block_n(block_n)) {
        set_error("itq3_dequant: invalid block_n %d", block_n);
        return ITQ3_E_DOMAIN;
    }
    if (numel > n_blocks * block_n || numel <= (n_blocks - 1) * block_n) {
        set_error("itq3_dequant: numel %lld inconsistent with %lld blocks of %d", (long long)numel,
                  (long long)n_blocks, block_n);
        return ITQ3_E_SHAPE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (out_dtype == ITQ3_F64) return launch_dequant(payload, n_blocks, block_n, sub_scales, numel, (double*)out, s);
    if (out_dtype == ITQ3_F32) return launch_dequant(payload, n_blocks, block_n, sub_scales, numel, (float*)out, s);
    set_error("itq3_dequant: output dtype must be float32 or float64");
    return ITQ3_E_DOMAIN;
}

template <typename T>
static int launch_fwht(const T* in, T* out, int64_t n_vec, int n, int normalize, cudaStream_t s) {
    const T norm = (T)(1.0 / __builtin_sqrt((double)n));  // np.asarray(1.0 / math.sqrt(n), dtype)
    if (n < 32) {
        fwht_small_kernel<T><<<(unsigned)((n_vec + 127) / 128), 128, 0, s>>>(in, out, n_vec, n, normalize, norm);
        return check_launch("itq3_fwht");
    }
    const unsigned grid = (unsigned)((n_vec * 32 + 255) / 256);
    switch (n) {
        case 32: fwht_warp_kernel<32, T><<<grid, 256, 0, s>>>(in, out, n_vec, normalize, norm); break;
        case 64: fwht_warp_kernel<64, T><<<grid, 256, 0, s>>>(in, out, n_vec, normalize, norm); break;
        case 128: fwht_warp_kernel<128, T><<<grid, 256, 0, s>>>(in, out, n_vec, normalize, norm); break;
        case 256: fwht_warp_kernel<256, T><<<grid, 256, 0, s>>>(in, out, n_vec, normalize, norm); break;
        case 512: fwht_warp_kernel<512, T><<<grid, 256, 0, s>>>(in, out, n_vec, normalize, norm); break;
    }
    return check_launch("itq3_fwht");
}

extern "C" int itq3_fwht(const void* in, void* out, int dtype, int64_t n_vec, int n, int normalize, void* stream) {
    if (n < 2 || n > 512 || (n & (n - 1))) {
        set_error("fwht: block length must be a power of two in [2, 512], got %d", n);
        return ITQ3_E_LENGTH;
    }
    if (n_vec <= 0) return ITQ3_OK;
    cudaStream_t s = (cudaStream_t)stream;
    if (dtype == ITQ3_F64) return launch_fwht((const double*)in, (double*)out, n_vec, n, normalize, s);
    if (dtype == ITQ3_F32) return launch_fwht((const float*)in, (float*)out, n_vec, n, normalize, s);
    set_error("fwht: dtype must be float32 or float64");
    return ITQ3_E_DOMAIN;
}

// ------------------------------------------------------------------------------------------
// pack_ternary / unpack_ternary for batches of code rows (packing.py:43-84)
// ------------------------------------------------------------------------------------------
namespace itq3 {
__global__ void pack_codes_kernel(const int8_t* __restrict__ codes, int64_t n_rows, int n, uint8_t* __restrict__ out,
                                  unsigned long long* bad) {
    const int bytes_per_row = 3 * n / 8;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n_rows * bytes_per_row) return;
    const int64_t row = idx / bytes_per_row;
    const int bi = (int)(idx % bytes_per_row);
    const int plane = bi / (n / 8), k = bi % (n / 8);
    uint32_t byte = 0;
    for (int i = 0; i < 8; ++i) {
        const int q = codes[row * n + 8 * k + i];
        if (q < -1 || q > 1) atomicMin(bad, ((unsigned long long)row << 16) | (unsigned long long)(8 * k + i));
        byte |= (((uint32_t)(q + 1) >> plane) & 1u) << i;
    }
    out[idx] = (uint8_t)byte;
}

__global__ void unpack_codes_kernel(const uint8_t* __restrict__ planes, int64_t n_rows, int n,
                                    int8_t* __restrict__ codes, unsigned long long* bad) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n_rows * n) return;
    const int64_t row = idx / n;
    const int j = (int)(idx % n);
    const uint8_t* p = planes + row * (3 * n / 8);
    const int c = ((p[j >> 3] >> (j & 7)) & 1) + 2 * ((p[n / 8 + (j >> 3)] >> (j & 7)) & 1) +
                  4 * ((p[n / 4 + (j >> 3)] >> (j & 7)) & 1);
    if (c > 2) atomicMin(bad, ((unsigned long long)row << 16) | ((unsigned long long)c << 12) | (unsigned long long)j);
    codes[idx] = (int8_t)(c - 1);
}
}  // namespace itq3

extern "C" int itq3_pack_codes(const int8_t* codes, int64_t n_rows, int n, uint8_t* planes,
                               unsigned long long* d_bad, void* stream) {
    if (n <= 0 || n % 8 || n > 512) {
        set_error("pack_ternary: length must be a positive multiple of 8, at most 512, got %d", n);
        return ITQ3_E_LENGTH;
    }
    const int64_t total = n_rows * (3 * n / 8);
    if (total == 0) return ITQ3_OK;
    pack_codes_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(codes, n_rows, n, planes,
                                                                                        d_bad);
    return check_launch("itq3_pack_codes");
}

extern "C" int itq3_unpack_codes(const uint8_t* planes, int64_t n_rows, int n, int8_t* codes,
                                 unsigned long long* d_bad, void* stream) {
    if (n <= 0 || n % 8 || n > 512) {
        set_error("unpack_ternary: invalid block length %d", n);
        return ITQ3_E_LENGTH;
    }
    const int64_t total = n_rows * n;
    if (total == 0) return ITQ3_OK;
    unpack_codes_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(planes, n_rows, n, codes,
                                                                                          d_bad);
    return check_launch("itq3_unpack_codes");
}
