// Fused rotated-activation GEMV / small-M matmul on the tiled layout, plus the generic
// fp64 fused matmul for every other layout (sm_100a).
//
// Algebra: the reference reconstructs
//   w_hat_b = (1/16) H (d_b (c_b - 1 - z_b))           (codec.py:152-161, H = +-1 Sylvester)
// and accumulates w_hat . x (compute.py:115-124).  H is symmetric, so
//   <w_hat_b, x_b> = (d_b / 16) (<c_b, H x_b> - (1 + z_b) sum(H x_b)),
// i.e. the 256-point IFWHT moves to the activations (once per token per 256-block) and the
// weights stay 2-bit codes c in {0,1,2}.  x' = H x_b is held as a fixed-point integer with a
// per-(block, token) power-of-two scale, split into `limbs` signed bytes; every limb is one
// column of an m16n8k32 u8 x s8 integer MMA, so the per-block products are exact int32 and
// the only approximation is the fixed-point rounding of x' (bounded a priori, tested).
//
// Tiled layout (itq3_repack_tiled): tile = 16 rows x one 256-block.  Lane (g = lane/4,
// t = lane%4) of a warp owns two uint4 words (group G = 0, 1).  Word r (0..3), byte beta,
// bit pair i (0..3) holds c(row, k) with
//     row = 16*rt + g + 8*(r & 1),   k = 256*b + 128*G + 32*i + 16*(r >> 1) + 4*t + beta,
// which is exactly the mma A-fragment (a0..a3) of the MMA for chunk q = 4G + i when the
// word is masked with 0x03030303 << 2i: the bytes then hold c * 4^i (u8 <= 128).  One LOP3
// per 4 weights decodes the A operand; the 4^i class factor is removed per tile with shifts.
#include "common.cuh"

namespace itq3 {

constexpr int kTileBytes = 1024;      // 16 rows x 256 codes x 2 bits
constexpr int kTileScaleBytes = 32;   // 16 x f16, packed as (row g, row g+8) pairs
constexpr int kTileZpBytes = 16;      // 16 x int8 (asymmetric only)
constexpr int kActFragBytes = 2048;   // 8 chunks x 32 lanes x 8 B per (pass, block)
constexpr int kActMetaD = 8 * 2 * 8;  // 8 columns x (factor, correction) x double
constexpr int kActMetaF = 8 * 2 * 4;  // same in float

struct TiledPtrs {
    uint4* codes;
    uint32_t* scales;
    uint16_t* zps;
};

__host__ __device__ inline TiledPtrs tiled_ptrs(uint8_t* base, int64_t RT, int64_t NB) {
    TiledPtrs p;
    p.codes = reinterpret_cast<uint4*>(base);
    p.scales = reinterpret_cast<uint32_t*>(base + RT * NB * kTileBytes);
    p.zps = reinterpret_cast<uint16_t*>(base + RT * NB * (kTileBytes + kTileScaleBytes));
    return p;
}

// ------------------------------------------------------------------------------------------
// Repack: container payload (block_n 256, variant s, cols % 256 == 0) -> tiled layout.
// Plane 2 is dropped (validated zero beforehand, packing.py:80-83).  One warp per tile.
// ------------------------------------------------------------------------------------------
__global__ void repack_kernel(const uint8_t* __restrict__ payload, int64_t rows, int64_t NB, int64_t RT, int asym,
                              uint8_t* __restrict__ tiled) {
    const int lane = threadIdx.x & 31;
    const int64_t tile = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (tile >= RT * NB) return;
    const int64_t rt = tile / NB, b = tile % NB;
    const int g = lane >> 2, t = lane & 3;
    TiledPtrs P = tiled_ptrs(tiled, RT, NB);
#pragma unroll
    for (int G = 0; G < 2; ++G) {
        uint32_t word[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int64_t row = rt * 16 + g + 8 * (r & 1);
            uint32_t wv = 0;
            if (row < rows) {
                const uint8_t* blk = payload + (row * NB + b) * 100;
                const int pos = 16 * (r >> 1) + 4 * t;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint32_t p0 = *reinterpret_cast<const uint32_t*>(blk + 4 * (4 * G + i));
                    const uint32_t p1 = *reinterpret_cast<const uint32_t*>(blk + 32 + 4 * (4 * G + i));
#pragma unroll
                    for (int beta = 0; beta < 4; ++beta) {
                        const uint32_t c = ((p0 >> (pos + beta)) & 1u) | (((p1 >> (pos + beta)) & 1u) << 1);
                        wv |= c << (8 * beta + 2 * i);
                    }
                }
            }
            word[r] = wv;
        }
        P.codes[(tile * 2 + G) * 32 + lane] = make_uint4(word[0], word[1], word[2], word[3]);
    }
    if (t == 0) {
        const int64_t r0 = rt * 16 + g, r1 = r0 + 8;
        uint32_t s0 = 0, s1 = 0;
        int z0 = 0, z1 = 0;
        if (r0 < rows) {
            const uint8_t* blk = payload + (r0 * NB + b) * 100;
            s0 = *reinterpret_cast<const uint16_t*>(blk + 96);
            z0 = (int)f16_bits_to_f64(*reinterpret_cast<const uint16_t*>(blk + 98));
        }
        if (r1 < rows) {
            const uint8_t* blk = payload + (r1 * NB + b) * 100;
            s1 = *reinterpret_cast<const uint16_t*>(blk + 96);
            z1 = (int)f16_bits_to_f64(*reinterpret_cast<const uint16_t*>(blk + 98));
        }
        P.scales[tile * 8 + g] = s0 | (s1 << 16);
        if (asym) P.zps[tile * 8 + g] = (uint16_t)((uint8_t)(int8_t)z0 | ((uint16_t)(uint8_t)(int8_t)z1 << 8));
    }
}

// ------------------------------------------------------------------------------------------
// K3: activation rotation + fixed-point limb split, written in mma B-fragment order.
// CTA = (256-block b, pass); warp w = token pass*tpp + w.  Butterfly in binary64 (exact for
// fp32/bf16 inputs up to the final rounding of each stage, ~2^-50 relative).
// ------------------------------------------------------------------------------------------
template <typename TX>
__global__ void __launch_bounds__(256) rotate_act_kernel(const TX* __restrict__ x, int64_t NB, int64_t M,
                                                         int64_t stride_k, int64_t stride_m, int L, int tpp,
                                                         uint8_t* __restrict__ act, int64_t n_pass) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // let the GEMV launch (PDL)
    __shared__ __align__(16) uint8_t img[kActFragBytes];
    __shared__ double meta[8][2];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t b = blockIdx.x, pass = blockIdx.y;
    for (int i = threadIdx.x; i < kActFragBytes / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(img)[i] = 0u;
    if (threadIdx.x < 16) (&meta[0][0])[threadIdx.x] = 0.0;
    __syncthreads();
    const int64_t m = pass * tpp + w;
    if (w < tpp && m < M) {
        double v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = (double)x[(b * 256 + lane + 32 * e) * stride_k + m * stride_m];
        // unnormalised butterfly, same schedule as the codec (stride layout)
#pragma unroll
        for (int h = 1; h < 32; h <<= 1) {
            const bool high = (lane & h) != 0;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const double p = __shfl_xor_sync(FULL, v[e], h);
                v[e] = high ? __dsub_rn(p, v[e]) : __dadd_rn(v[e], p);
            }
        }
#pragma unroll
        for (int hh = 1; hh < 8; hh <<= 1)
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if ((e & hh) == 0) {
                    const double lo = v[e], hi = v[e + hh];
                    v[e] = __dadd_rn(lo, hi);
                    v[e + hh] = __dsub_rn(lo, hi);
                }
        double amax = 0.0;
#pragma unroll
        for (int e = 0; e < 8; ++e) amax = fmax(amax, fabs(v[e]));
#pragma unroll
        for (int o = 16; o; o >>= 1) amax = fmax(amax, __shfl_xor_sync(FULL, amax, o));
        // power-of-two scale 2^ex with |x'| / 2^ex < 2^(8L-2): limbs never overflow
        const int ex = amax > 0.0 ? ilogb(amax) + 3 - 8 * L : 0;
        long long Q = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            long long q = llrint(scalbn(v[e], -ex));
            Q += q;
            const int j = lane + 32 * e;
            const int chunk = j >> 5, kap = j & 31;
            const int tt = (kap & 15) >> 2, beta = kap & 3, half = kap >> 4;
            for (int l = 0; l < L; ++l) {
                const int lb = (int)(((q + 128) & 255)) - 128;
                q = (q - lb) >> 8;
                const int col = w * L + l;
                img[(chunk * 32 + 4 * col + tt) * 8 + half * 4 + beta] = (uint8_t)(int8_t)lb;
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) Q += __shfl_xor_sync(FULL, Q, o);
        if (lane < L) {
            const int col = w * L + lane;
            meta[col][0] = ldexp(1.0, 8 * lane + ex - 4);                  // 256^l * 2^ex / 16
            meta[col][1] = lane == 0 ? ldexp((double)Q, ex - 4) : 0.0;     // 2^ex * sum(q) / 16
        }
    }
    __syncthreads();
    uint8_t* frag = act + (pass * NB + b) * kActFragBytes;
    for (int i = threadIdx.x; i < kActFragBytes / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(frag)[i] = reinterpret_cast<const uint4*>(img)[i];
    double* md = reinterpret_cast<double*>(act + n_pass * NB * kActFragBytes) + (pass * NB + b) * 16;
    float* mf = reinterpret_cast<float*>(act + n_pass * NB * (kActFragBytes + kActMetaD)) + (pass * NB + b) * 16;
    if (threadIdx.x < 16) {
        md[threadIdx.x] = (&meta[0][0])[threadIdx.x];
        mf[threadIdx.x] = (float)(&meta[0][0])[threadIdx.x];
    }
}

// ------------------------------------------------------------------------------------------
// K4: fused GEMV.  CTA = one 16-row tile x one token pass; 8 warps split the 256-blocks of K
// (warp w takes blocks w, w+8, ...), then a fixed-order smem reduction (deterministic).
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void mma_u8s8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <typename ACC>
struct MetaT;
template <>
struct MetaT<float> {
    __device__ static const float* base(const uint8_t* act, int64_t n_pass, int64_t NB) {
        return reinterpret_cast<const float*>(act + n_pass * NB * (kActFragBytes + kActMetaD));
    }
};
template <>
struct MetaT<double> {
    __device__ static const double* base(const uint8_t* act, int64_t n_pass, int64_t NB) {
        return reinterpret_cast<const double*>(act + n_pass * NB * kActFragBytes);
    }
};

__device__ __forceinline__ float h2acc(uint16_t h, float) { return f16_bits_to_f32(h); }
__device__ __forceinline__ double h2acc(uint16_t h, double) { return f16_bits_to_f64(h); }

constexpr int kGemvWarps = 8;

template <typename ACC, typename TY>
__global__ void __launch_bounds__(32 * kGemvWarps) gemv_kernel(const uint8_t* __restrict__ tiled, int64_t rows,
                                                               int64_t NB, int64_t RT, int asym,
                                                               const uint8_t* __restrict__ act, int64_t M, int L,
                                                               int tpp, int64_t n_pass, TY* __restrict__ y,
                                                               int64_t stride_r, int64_t stride_m) {
    __shared__ ACC red[kGemvWarps][16][8];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int64_t rt = blockIdx.x, pass = blockIdx.y;
    TiledPtrs P = tiled_ptrs(const_cast<uint8_t*>(tiled), RT, NB);
    const uint2* frag = reinterpret_cast<const uint2*>(act);
    const ACC* meta = MetaT<ACC>::base(act, n_pass, NB);
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the rotation launched before this GEMV is done

    ACC acc[2][2] = {{ACC(0), ACC(0)}, {ACC(0), ACC(0)}};
    for (int64_t b = w; b < NB; b += kGemvWarps) {
        const int64_t tile = rt * NB + b;
        const uint4 wa0 = __ldg(&P.codes[(tile * 2 + 0) * 32 + lane]);
        const uint4 wa1 = __ldg(&P.codes[(tile * 2 + 1) * 32 + lane]);
        const uint32_t sc = __ldg(&P.scales[tile * 8 + g]);
        uint2 bf[8];
        const uint2* fb = frag + ((pass * NB + b) * 8) * 32 + lane;
#pragma unroll
        for (int q = 0; q < 8; ++q) bf[q] = __ldg(fb + q * 32);
        const ACC* mb = meta + (pass * NB + b) * 16 + 4 * t;  // columns 2t, 2t+1: (f, corr) pairs
        const ACC f0 = mb[0], c0 = mb[1], f1 = mb[2], c1 = mb[3];

        int C[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i) C[i][0] = C[i][1] = C[i][2] = C[i][3] = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t mk = 0x03030303u << (2 * i);
            mma_u8s8(C[i], wa0.x & mk, wa0.y & mk, wa0.z & mk, wa0.w & mk, bf[i].x, bf[i].y);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t mk = 0x03030303u << (2 * i);
            mma_u8s8(C[i], wa1.x & mk, wa1.y & mk, wa1.z & mk, wa1.w & mk, bf[4 + i].x, bf[4 + i].y);
        }
        int Cc[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) Cc[r] = C[0][r] + (C[1][r] >> 2) + (C[2][r] >> 4) + (C[3][r] >> 6);

        const ACC d0 = h2acc((uint16_t)(sc & 0xffffu), ACC(0)), d1 = h2acc((uint16_t)(sc >> 16), ACC(0));
        ACC zf0 = ACC(1), zf1 = ACC(1);
        if (asym) {
            const uint16_t zz = __ldg(&P.zps[tile * 8 + g]);
            zf0 = ACC(1 + (int)(int8_t)(zz & 0xff));
            zf1 = ACC(1 + (int)(int8_t)(zz >> 8));
        }
        acc[0][0] += d0 * (f0 * (ACC)Cc[0] - zf0 * c0);
        acc[0][1] += d0 * (f1 * (ACC)Cc[1] - zf0 * c1);
        acc[1][0] += d1 * (f0 * (ACC)Cc[2] - zf1 * c0);
        acc[1][1] += d1 * (f1 * (ACC)Cc[3] - zf1 * c1);
    }
    red[w][g][2 * t] = acc[0][0];
    red[w][g][2 * t + 1] = acc[0][1];
    red[w][g + 8][2 * t] = acc[1][0];
    red[w][g + 8][2 * t + 1] = acc[1][1];
    __syncthreads();
    const int tid = threadIdx.x;
    if (tid < 16 * tpp) {
        const int r = tid & 15, ml = tid >> 4;
        const int64_t m = pass * tpp + ml;
        const int64_t row = rt * 16 + r;
        if (m < M && row < rows) {
            ACC s = ACC(0);
            for (int ww = 0; ww < kGemvWarps; ++ww)
                for (int l = 0; l < L; ++l) s += red[ww][r][ml * L + l];
            y[row * stride_r + m * stride_m] = (TY)s;
        }
    }
}

// ------------------------------------------------------------------------------------------
// Generic fused matmul (fp64): one warp decodes one block exactly (same data flow as the
// codec) and writes per-row-segment partial dots; a second pass sums them per row in block
// order, so results are deterministic.  Handles every block size, variant and straddle.
// ------------------------------------------------------------------------------------------
template <int N>
__global__ void __launch_bounds__(256) generic_partial_kernel(const uint8_t* __restrict__ payload, int64_t nb,
                                                              int ss, int64_t rows, int64_t cols,
                                                              const double* __restrict__ X, int64_t k,
                                                              int64_t stride_c, int64_t stride_j, int maxseg,
                                                              double* __restrict__ ws) {
    constexpr int E = N / 32;
    const int lane = threadIdx.x & 31;
    const int64_t blk = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (blk >= nb) return;
    const uint8_t* p = payload + blk * block_nbytes(N, ss);
    const double z = trunc(f16_bits_to_f64(*reinterpret_cast<const uint16_t*>(p + 3 * N / 8 + 2)));
    double scale = f16_bits_to_f64(*reinterpret_cast<const uint16_t*>(p + 3 * N / 8));
    double v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int j = lane + 32 * e;
        const uint32_t p0 = *reinterpret_cast<const uint32_t*>(p + 4 * e);
        const uint32_t p1 = *reinterpret_cast<const uint32_t*>(p + N / 8 + 4 * e);
        const int c = (int)((p0 >> lane) & 1u) + 2 * (int)((p1 >> lane) & 1u);
        if (ss) scale = f16_bits_to_f64(*reinterpret_cast<const uint16_t*>(p + 3 * N / 8 + 4 + 2 * (j / (N / 8))));
        v[e] = __dmul_rn(scale, __dsub_rn((double)(c - 1), z));
    }
    // butterfly (stride layout) + normalisation, identical to decode_block
#pragma unroll
    for (int h = 1; h < 32; h <<= 1) {
        const bool high = (lane & h) != 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const double pp = __shfl_xor_sync(FULL, v[e], h);
            v[e] = high ? __dsub_rn(pp, v[e]) : __dadd_rn(v[e], pp);
        }
    }
#pragma unroll
    for (int hh = 1; hh < E; hh <<= 1)
#pragma unroll
        for (int e = 0; e < E; ++e)
            if ((e & hh) == 0) {
                const double lo = v[e], hi = v[e + hh];
                v[e] = __dadd_rn(lo, hi);
                v[e + hh] = __dsub_rn(lo, hi);
            }
    const double norm = __ddiv_rn(1.0, __dsqrt_rn((double)N));
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = __dmul_rn(v[e], norm);

    const int64_t p0 = blk * N, size = rows * cols;
    const int64_t pend = p0 + N < size ? p0 + N : size;
    const int64_t r_first = p0 / cols;
    for (int64_t r = r_first; r * cols < pend; ++r) {
        const int seg = (int)(r - r_first);
        const int64_t lo = (r * cols > p0 ? r * cols : p0) - p0;
        const int64_t hi = ((r + 1) * cols < pend ? (r + 1) * cols : pend) - p0;
        for (int64_t jj = 0; jj < k; ++jj) {
            double s = 0.0;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int j = lane + 32 * e;
                if (j >= lo && j < hi) s = __fma_rn(v[e], X[(p0 + j - r * cols) * stride_c + jj * stride_j], s);
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
            if (lane == 0) ws[(blk * maxseg + seg) * k + jj] = s;
        }
    }
}

__global__ void generic_reduce_kernel(const double* __restrict__ ws, int64_t rows, int64_t cols, int N, int64_t k,
                                      int maxseg, double* __restrict__ Y) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= rows * k) return;
    const int64_t r = idx / k, jj = idx % k;
    const int64_t b0 = (r * cols) / N, b1 = ((r + 1) * cols - 1) / N;
    double s = 0.0;
    for (int64_t b = b0; b <= b1; ++b) {
        const int seg = (int)(r - (b * N) / cols);
        s += ws[(b * maxseg + seg) * k + jj];
    }
    Y[r * k + jj] = s;
}

}  // namespace itq3

using namespace itq3;

// ==========================================================================================
// C ABI
// ==========================================================================================
extern "C" int64_t itq3_tiled_nbytes(int64_t rows, int64_t cols, int asymmetric) {
    const int64_t RT = (rows + 15) / 16, NB = cols / 256;
    return RT * NB * (kTileBytes + kTileScaleBytes + (asymmetric ? kTileZpBytes : 0));
}

extern "C" int itq3_repack_tiled(const uint8_t* payload, int64_t rows, int64_t cols, int asymmetric, uint8_t* tiled,
                                 void* stream) {
    if (rows <= 0 || cols <= 0 || cols % 256) {
        set_error("itq3_repack_tiled: tiled layout needs cols %% 256 == 0 (got %lld x %lld)", (long long)rows,
                  (long long)cols);
        return ITQ3_E_UNSUPPORTED;
    }
    const int64_t RT = (rows + 15) / 16, NB = cols / 256;
    const int64_t threads = RT * NB * 32;
    repack_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(payload, rows, NB, RT,
                                                                                       asymmetric, tiled);
    return check_launch("itq3_repack_tiled");
}

static inline int tokens_per_pass(int limbs) { return 8 / limbs; }

extern "C" int64_t itq3_act_nbytes(int64_t cols, int64_t m, int limbs) {
    if (limbs < 1 || limbs > 8) return -1;
    const int64_t NB = cols / 256, tpp = tokens_per_pass(limbs);
    const int64_t n_pass = (m + tpp - 1) / tpp;
    return n_pass * NB * (kActFragBytes + kActMetaD + kActMetaF);
}

extern "C" int itq3_rotate_act(const void* x, int x_dtype, int64_t cols, int64_t m, int64_t stride_k,
                               int64_t stride_m, int limbs, uint8_t* act, void* stream) {
    if (cols <= 0 || cols % 256 || m <= 0) {
        set_error("itq3_rotate_act: need cols %% 256 == 0 and m > 0 (got %lld, %lld)", (long long)cols,
                  (long long)m);
        return ITQ3_E_SHAPE;
    }
    if (limbs < 1 || limbs > 8) {
        set_error("itq3_rotate_act: limbs must be in [1, 8]");
        return ITQ3_E_DOMAIN;
    }
    const int64_t NB = cols / 256;
    const int tpp = tokens_per_pass(limbs);
    const int64_t n_pass = (m + tpp - 1) / tpp;
    const dim3 grid((unsigned)NB, (unsigned)n_pass), block(32 * tpp);
    cudaStream_t s = (cudaStream_t)stream;
    switch (x_dtype) {
        case ITQ3_F32:
            rotate_act_kernel<float><<<grid, block, 0, s>>>((const float*)x, NB, m, stride_k, stride_m, limbs, tpp,
                                                            act, n_pass);
            break;
        case ITQ3_F64:
            rotate_act_kernel<double><<<grid, block, 0, s>>>((const double*)x, NB, m, stride_k, stride_m, limbs,
                                                             tpp, act, n_pass);
            break;
        case ITQ3_BF16:
            rotate_act_kernel<__nv_bfloat16><<<grid, block, 0, s>>>((const __nv_bfloat16*)x, NB, m, stride_k,
                                                                    stride_m, limbs, tpp, act, n_pass);
            break;
        case ITQ3_F16:
            rotate_act_kernel<__half><<<grid, block, 0, s>>>((const __half*)x, NB, m, stride_k, stride_m, limbs, tpp,
                                                             act, n_pass);
            break;
        default:
            set_error("itq3_rotate_act: unsupported activation dtype %d", x_dtype);
            return ITQ3_E_DOMAIN;
    }
    return check_launch("itq3_rotate_act");
}

extern "C" int itq3_gemv(const uint8_t* tiled, int64_t rows, int64_t cols, int asymmetric, const uint8_t* act,
                         int64_t m, int limbs, void* y, int y_dtype, int64_t stride_r, int64_t stride_m,
                         void* stream) {
    if (rows <= 0 || cols <= 0 || cols % 256 || m <= 0) {
        set_error("itq3_gemv: bad shape %lld x %lld, m=%lld", (long long)rows, (long long)cols, (long long)m);
        return ITQ3_E_SHAPE;
    }
    if (limbs < 1 || limbs > 8) {
        set_error("itq3_gemv: limbs must be in [1, 8]");
        return ITQ3_E_DOMAIN;
    }
    const int64_t NB = cols / 256, RT = (rows + 15) / 16;
    const int tpp = tokens_per_pass(limbs);
    const int64_t n_pass = (m + tpp - 1) / tpp;
    const dim3 grid((unsigned)RT, (unsigned)n_pass), block(32 * kGemvWarps);
    cudaStream_t s = (cudaStream_t)stream;
    // programmatic dependent launch: the GEMV's launch and prologue overlap the preceding rotation
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (y_dtype == ITQ3_F32)
        cudaLaunchKernelEx(&cfg, gemv_kernel<float, float>, tiled, rows, NB, RT, asymmetric, act, m, limbs, tpp, n_pass,
                           (float*)y, stride_r, stride_m);
    else if (y_dtype == ITQ3_F64)
        cudaLaunchKernelEx(&cfg, gemv_kernel<double, double>, tiled, rows, NB, RT, asymmetric, act, m, limbs, tpp,
                           n_pass, (double*)y, stride_r, stride_m);
    else if (y_dtype == ITQ3_BF16)
        cudaLaunchKernelEx(&cfg, gemv_kernel<float, __nv_bfloat16>, tiled, rows, NB, RT, asymmetric, act, m, limbs,
                           tpp, n_pass, (__nv_bfloat16*)y, stride_r, stride_m);
    else {
        set_error("itq3_gemv: output dtype must be float32, float64 or bfloat16");
        return ITQ3_E_DOMAIN;
    }
    return check_launch("itq3_gemv");
}

static int generic_maxseg(int64_t cols, int block_n) { return (int)((block_n - 1) / cols + 2); }

extern "C" int64_t itq3_generic_ws_nbytes(int64_t rows, int64_t cols, int block_n, int64_t k) {
    const int64_t nb = (rows * cols + block_n - 1) / block_n;
    return nb * generic_maxseg(cols, block_n) * k * (int64_t)sizeof(double);
}

extern "C" int itq3_matmul_generic(const uint8_t* payload, int64_t rows, int64_t cols, int block_n, int sub_scales,
                                   const double* X, int64_t k, int64_t stride_c, int64_t stride_j, double* Y,
                                   void* workspace, void* stream) {
    if (!valid_block_n(block_n)) {
        set_error("itq3_matmul_generic: invalid block_n %d", block_n);
        return ITQ3_E_DOMAIN;
    }
    if (rows <= 0 || cols <= 0 || k <= 0) {
        set_error("itq3_matmul_generic: bad shape");
        return ITQ3_E_SHAPE;
    }
    const int64_t nb = (rows * cols + block_n - 1) / block_n;
    const int maxseg = generic_maxseg(cols, block_n);
    cudaStream_t s = (cudaStream_t)stream;
    double* ws = (double*)workspace;
    const unsigned grid = (unsigned)((nb * 32 + 255) / 256);
#define ITQ3_GEN(NN)                                                                                            \
    generic_partial_kernel<NN><<<grid, 256, 0, s>>>(payload, nb, sub_scales, rows, cols, X, k, stride_c, stride_j, \
                                                    maxseg, ws)
    switch (block_n) {
        case 32: ITQ3_GEN(32); break;
        case 64: ITQ3_GEN(64); break;
        case 128: ITQ3_GEN(128); break;
        case 256: ITQ3_GEN(256); break;
        case 512: ITQ3_GEN(512); break;
    }
#undef ITQ3_GEN
    int rc = check_launch("itq3_matmul_generic/partial");
    if (rc) return rc;
    const int64_t n = rows * k;
    generic_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(ws, rows, cols, block_n, k, maxseg, Y);
    return check_launch("itq3_matmul_generic/reduce");
}
