// Probe: cycles per chain-kernel rotation (itq3::chain_rotate_to_smem) on one SM, with 1 / 4 / 16
// concurrent warps, and knock-out variants, to split its cost into latency and shared-pipe throughput.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/probes/rot_probe tools/probes/rot_probe.cu build/runtime.o
#include "../../paper_2603_27914_b200/csrc/chain.cu"
#include <cstdio>
#include <vector>

using namespace itq3;

namespace itq3 {
template <int R>
__device__ __forceinline__ void swap_butterfly(int (&v)[8], int M, bool hi) {
#pragma unroll
    for (int e0 = 0; e0 < 8; ++e0)
        if (!(e0 & R)) {
            const int e1 = e0 | R;
            const int keep = hi ? v[e1] : v[e0];
            const int p = __shfl_xor_sync(FULL, hi ? v[e0] : v[e1], M);
            const int a = hi ? p : keep, b = hi ? keep : p;
            v[e0] = a + b;
            v[e1] = a - b;
        }
}

// Fragment image word of (32-k chunk q, limb column l, t-group tt, k-half h): the 32 words of a chunk
// are XOR-swizzled by sigma(q) so that the writer (one store per (l, h): lanes = (q, tt)) and the reader
// (one 8-byte load per q: lanes = (l, tt)) are both free of bank conflicts.
__host__ __device__ constexpr int swap_sigma(int q) { return (q & 1) | (((q >> 1) & 3) << 3); }

__device__ __forceinline__ void swap_rotate_to_smem(const float (&fin)[8], int L, uint8_t* img, int lane) {
    float f[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) f[e] = fin[e];
    // warp max of |f| as an integer max of the (non-negative) float bit patterns: one REDUX
    unsigned fbits = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) fbits = max(fbits, __float_as_uint(fabsf(f[e])));
    fbits = __reduce_max_sync(FULL, fbits);
    const float fmaxa = __uint_as_float(fbits);
    const int e_in = fmaxa > 0.f ? ilogbf(fmaxa) - 21 : 0;
    const float sc_in = pow2f(-e_in);
    int v[8];  // lane L, register e: element k = L + 32 e (lane bits k0..k4, register bits k5..k7)
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = __float2int_rn(f[e] * sc_in);
    // exact int32 FWHT: the register bits k5..k7 in registers ...
#pragma unroll
    for (int hh = 1; hh < 8; hh <<= 1)
#pragma unroll
        for (int e = 0; e < 8; ++e)
            if ((e & hh) == 0) {
                const int lo = v[e], hi = v[e + hh];
                v[e] = lo + hi;
                v[e + hh] = lo - hi;
            }
    // ... and the lane bits k0..k4 as swap butterflies, which also move (k0, k1, k4) into the register
    // index, where the fragment words need them: register bits (1, 2, 4) end as (k0, k1, k4) and the
    // lane bits (0..4) as (k5, k6, k7, k2, k3), i.e. chunk q = k >> 5 = lane & 7 (class i = lane & 3),
    // t-group tt = (k >> 2) & 3 = lane >> 3, byte beta = e & 3, k-half h = e >> 2.
    swap_butterfly<1>(v, 1, lane & 1);    // k0 <-> k5
    swap_butterfly<2>(v, 2, lane & 2);    // k1 <-> k6
    swap_butterfly<4>(v, 4, lane & 4);    // k2 <-> k7
    swap_butterfly<4>(v, 8, lane & 8);    // k3 <-> k2
    swap_butterfly<4>(v, 16, lane & 16);  // k4 <-> k3
    unsigned amax = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) amax = max(amax, (unsigned)abs(v[e]));
    amax = __reduce_max_sync(FULL, amax);
    // shift k so that |q| <= 2^(8L-2) (limbs never overflow): bitlen(amax) - k <= 8L - 2
    const int bl = 32 - __clz(amax);
    // (limbs = 4 gives no more than 22 bits: q 4^3 and the class differences must fit the four
    // balanced record limbs of an int32)
    const int k = max(0, bl - min(8 * L - 2, 22));
    const int ex = e_in + k;
    // Class folding: chunk q = 4G + i pairs with the A operand c * 4^i (bit pair i of the code
    // bytes), so its activations are stored pre-scaled by 4^(3-i); every IMMA of a tile then
    // accumulates 64 * sum(c x') into ONE integer accumulator (no per-tile class recombination).
    // |q| <= 2^22 -> |q 4^(3-i)| <= 2^28: four balanced base-256 limbs = the bytes of
    // (qs + 0x80808080) ^ 0x80808080, all four record columns used.
    // Cumulative masks: with P_i = codes & (4^(i+1) - 1 per byte) (P_3 = the raw word, no mask),
    // sum_i (c_i 4^i) A_i = sum_i P_i (A_i - A_{i+1}) (A_4 = 0, exact in int32), so chunk q stores
    // the difference of its pre-scaled activation and the next class's (the lane above: class i + 1,
    // same G, tt and register): the tile needs 3 LOP3 per A register group instead of 4 and produces
    // the same integer accumulators.
    const int cls = lane & 3;
    int Q = 0;
    uint32_t limbs[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int q = k ? ((v[e] + (1 << (k - 1))) >> k) : v[e];
        Q += q;
        const int qs = q << (2 * (3 - cls));
        const int up = __shfl_down_sync(FULL, qs, 1);
        const int dq = cls < 3 ? qs - up : qs;  // |dq| < 2^29
        limbs[e] = (uint32_t)(dq + (int)0x80808080u) ^ 0x80808080u;
    }
    // 4x4 byte transposes: word (l, h) = byte l of the limbs of beta = 0..3 (registers 4h .. 4h + 3)
    uint32_t* w32 = reinterpret_cast<uint32_t*>(img);
    const int q = lane & 7, tt = lane >> 3;
    uint32_t* wq = w32 + q * 32;
    const int sw = (tt * 2) ^ swap_sigma(q);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint32_t t0 = __byte_perm(limbs[4 * h], limbs[4 * h + 1], 0x5140);
        const uint32_t t1 = __byte_perm(limbs[4 * h], limbs[4 * h + 1], 0x7362);
        const uint32_t t2 = __byte_perm(limbs[4 * h + 2], limbs[4 * h + 3], 0x5140);
        const uint32_t t3 = __byte_perm(limbs[4 * h + 2], limbs[4 * h + 3], 0x7362);
        wq[sw ^ (0 * 8 + h)] = __byte_perm(t0, t2, 0x5410);
        wq[sw ^ (1 * 8 + h)] = __byte_perm(t0, t2, 0x7632);
        wq[sw ^ (2 * 8 + h)] = __byte_perm(t1, t3, 0x5410);
        wq[sw ^ (3 * 8 + h)] = __byte_perm(t1, t3, 0x7632);
    }
    Q = __reduce_add_sync(FULL, Q);
    float* meta = reinterpret_cast<float*>(img + 8 * 16 * 8);  // f[0..7], corr[0..7]
    if (lane < 8) {
        meta[lane] = lane < 4 ? pow2f(8 * lane + ex - 10) : 0.0f;  // 256^l 2^ex / 16 / 64
        meta[8 + lane] = lane == 0 ? (float)Q * pow2f(ex - 4) : 0.0f;
    }
}

// B fragments of lane (g, t) from a rotation image: chunk q's words (limb g, t-group t, h = 0 / 1), two
// conflict-free 4-byte loads (the swizzle may swap the pair); columns g >= 4 are zero.
__device__ __forceinline__ void swap_load_frags(const uint8_t* img, int g, int t, uint2 (&bf)[8]) {
    const uint32_t* w32 = reinterpret_cast<const uint32_t*>(img);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        if (g < 4) {
            bf[q].x = w32[q * 32 + ((g * 8 + t * 2) ^ swap_sigma(q))];
            bf[q].y = w32[q * 32 + ((g * 8 + t * 2 + 1) ^ swap_sigma(q))];
        } else {
            bf[q] = make_uint2(0u, 0u);
        }
    }
}

}  // namespace itq3


// lean rotation candidate: bit-built scale (no pow2f branches), IMAD butterflies (p + s v), exact
// correction from element 0 (no Q reduction)
__device__ __forceinline__ void lean_rotate_to_smem(const float (&f)[8], int L, uint8_t* img, int lane) {
    unsigned fbits = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) fbits = max(fbits, __float_as_uint(f[e]) & 0x7fffffffu);
    fbits = __reduce_max_sync(FULL, fbits);
    const int bexp = (int)(fbits >> 23);  // biased exponent of max|f| (0: zero or subnormal)
    int e_in;
    float sc_in;
    if (bexp >= 21) {  // max|f| >= 2^-106: 2^-e_in is a normal float
        e_in = bexp - 148;
        sc_in = __int_as_float((127 - e_in) << 23);
    } else {
        const float fmaxa = __uint_as_float(fbits);
        e_in = fmaxa > 0.f ? ilogbf(fmaxa) - 21 : 0;
        sc_in = pow2f(-e_in);
    }
    int v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = __float_as_int(fmaf(f[e], sc_in, 12582912.0f)) - 0x4B400000;
    const int v0 = v[0];  // lane 0: element 0; sum_k (H v)_k = 256 v_0
#pragma unroll
    for (int h = 1; h < 32; h <<= 1) {
        const int sg = (lane & h) ? -1 : 1;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int p = __shfl_xor_sync(FULL, v[e], h);
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
    unsigned amax = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) amax = max(amax, (unsigned)abs(v[e]));
    amax = __reduce_max_sync(FULL, amax);
    const int bl = 32 - __clz(amax);
    const int k = max(0, bl - min(8 * L - 2, 22));
    const int ex = e_in + k;
    const int rnd = (1 << k) >> 1;
    const int tt = (lane & 15) >> 2, beta = lane & 3, half = lane >> 4;
    int qs[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) qs[e] = ((v[e] + rnd) >> k) << (2 * (3 - (e & 3)));
    uint8_t* dst0 = img + tt * 8 + half * 4 + beta;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int dq = (e & 3) < 3 ? qs[e] - qs[e + 1] : qs[e];
        const uint32_t limbs = (uint32_t)(dq + (int)0x80808080u) ^ 0x80808080u;
        uint8_t* dst = dst0 + e * 128;
#pragma unroll
        for (int l = 0; l < 4; ++l) dst[l * 32] = (uint8_t)(limbs >> (8 * l));
    }
    float* meta = reinterpret_cast<float*>(img + 8 * 16 * 8);  // f[0..7], corr[0..7]
    if (lane < 8) {
        meta[lane] = lane < 4 ? __int_as_float((8 * lane + ex - 10 + 127) << 23) : 0.0f;  // 256^l 2^ex / 16 / 64
        meta[8 + lane] = lane == 0 ? (float)v0 * pow2f(e_in + 4) : 0.0f;
    }
}


// lane L holds elements k = sig(L) + 32 e: lane bits (0,1) <-> k bits (2,3) swapped, so that one
// stmatrix.m16n8.trans.b8 per 4 chunks writes the fragment image (see chain.cu)
__device__ __forceinline__ int sig_lane(int L) { return ((L & 3) << 2) | ((L >> 2) & 3) | (L & 16); }

__device__ __forceinline__ void stsm_rotate_to_smem(const float (&f)[8], int L, uint8_t* img, int lane) {
    unsigned fbits = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) fbits = max(fbits, __float_as_uint(f[e]) & 0x7fffffffu);
    fbits = __reduce_max_sync(FULL, fbits);
    const int bexp = (int)(fbits >> 23);
    int e_in;
    float sc_in;
    if (bexp >= 21) {
        e_in = bexp - 148;
        sc_in = __int_as_float((127 - e_in) << 23);
    } else {
        const float fmaxa = __uint_as_float(fbits);
        e_in = fmaxa > 0.f ? ilogbf(fmaxa) - 21 : 0;
        sc_in = pow2f(-e_in);
    }
    int v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = __float_as_int(fmaf(f[e], sc_in, 12582912.0f)) - 0x4B400000;
    const int v0 = v[0];
#pragma unroll
    for (int h = 1; h < 32; h <<= 1) {
        const int sg = (lane & h) ? -1 : 1;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int p = __shfl_xor_sync(FULL, v[e], h);
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
    unsigned amax = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) amax = max(amax, (unsigned)abs(v[e]));
    amax = __reduce_max_sync(FULL, amax);
    const int bl = 32 - __clz(amax);
    const int k = max(0, bl - min(8 * L - 2, 22));
    const int ex = e_in + k;
    const int rnd = (1 << k) >> 1;
    int qs[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) qs[e] = ((v[e] + rnd) >> k) << (2 * (3 - (e & 3)));
    uint32_t lw[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int dq = (e & 3) < 3 ? qs[e] - qs[e + 1] : qs[e];
        lw[e] = (uint32_t)(dq + (int)0x80808080u) ^ 0x80808080u;
    }
    const uint32_t a = smem_u32(img) + (lane >> 3) * 128 + (lane & 7) * 16;
    asm volatile("stmatrix.sync.aligned.m16n8.x4.trans.shared.b8 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(lw[0]),
                 "r"(lw[1]), "r"(lw[2]), "r"(lw[3]) : "memory");
    asm volatile("stmatrix.sync.aligned.m16n8.x4.trans.shared.b8 [%0], {%1, %2, %3, %4};" ::"r"(a + 512), "r"(lw[4]),
                 "r"(lw[5]), "r"(lw[6]), "r"(lw[7]) : "memory");
    float* meta = reinterpret_cast<float*>(img + 8 * 16 * 8);
    if (lane < 8) {
        meta[lane] = lane < 4 ? __int_as_float((8 * lane + ex - 10 + 127) << 23) : 0.0f;
        meta[8 + lane] = lane == 0 ? (float)v0 * pow2f(e_in + 4) : 0.0f;
    }
}
// fragments of lane (g, t) from the stmatrix image
__device__ __forceinline__ void stsm_load_frags(const uint8_t* img, int g, int t, uint2 (&bf)[8]) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
        bf[q] = g < 4 ? *reinterpret_cast<const uint2*>(img + q * 128 + (2 * t + (g & 1)) * 16 + 8 * (g >> 1))
                      : make_uint2(0u, 0u);
}

template <int VAR>
__device__ __forceinline__ void rot_variant(float (&f)[8], uint8_t* img, int lane) {
    if (VAR == 0) {  // the kernel's rotation
        chain_rotate_to_smem(f, 3, img, lane);
        return;
    }
    if (VAR == 7) {
        stsm_rotate_to_smem(f, 3, img, lane);
        return;
    }
    if (VAR == 6) {
        lean_rotate_to_smem(f, 3, img, lane);
        return;
    }
    if (VAR == 5) {  // swap-butterfly variant (round 2 experiment): 28 SHFL + 8 STS.32 instead of 40 + 32 STS.U8
        swap_rotate_to_smem(f, 3, img, lane);
        return;
    }
    // VAR 1: FWHT only (fixed scale, no maxima, no limbs, no stores)
    // VAR 2: + the two REDUX maxima;  VAR 3: + limbs and class differences;  VAR 4: + byte stores
    unsigned fbits = 0;
    float sc_in = 1024.f;
    int e_in = -10;
    if (VAR >= 2) {
#pragma unroll
        for (int e = 0; e < 8; ++e) fbits = max(fbits, __float_as_uint(fabsf(f[e])));
        fbits = __reduce_max_sync(FULL, fbits);
        const float fmaxa = __uint_as_float(fbits);
        e_in = fmaxa > 0.f ? ilogbf(fmaxa) - 21 : 0;
        sc_in = pow2f(-e_in);
    }
    int v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = __float_as_int(fmaf(f[e], sc_in, 12582912.0f)) - 0x4B400000;
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
    int k = 2;
    if (VAR >= 2) {
        unsigned amax = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) amax = max(amax, (unsigned)abs(v[e]));
        amax = __reduce_max_sync(FULL, amax);
        k = max(0, 32 - __clz(amax) - 22);
    }
    if (VAR == 1 || VAR == 2) {
        int acc = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) acc ^= v[e] >> k;
        f[0] += (float)(acc & 1);
        return;
    }
    const int tt = (lane & 15) >> 2, beta = lane & 3, half = lane >> 4;
    int qs[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int q = k ? ((v[e] + (1 << (k - 1))) >> k) : v[e];
        qs[e] = q << (2 * (3 - (e & 3)));
    }
    uint32_t x = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int dq = (e & 3) < 3 ? qs[e] - qs[e + 1] : qs[e];
        const uint32_t limbs = (uint32_t)(dq + (int)0x80808080u) ^ 0x80808080u;
        if (VAR == 3) {
            x ^= limbs;
        } else {
            uint8_t* dst = img + (e * 16 + tt) * 8 + half * 4 + beta;
#pragma unroll
            for (int l = 0; l < 4; ++l) dst[l * 32] = (uint8_t)(limbs >> (8 * l));
        }
    }
    f[0] += (float)(x & 1);
}

template <int VAR>
__global__ void __launch_bounds__(576, 1) rot_probe(const float* x, int nwarps, int iters, long long* out) {
    __shared__ __align__(16) uint8_t img[16][kActSmemBlock];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp >= nwarps) return;
    float f[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) f[e] = x[warp * 256 + lane + 32 * e];
    __syncwarp();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        rot_variant<VAR>(f, img[warp], lane);
        __syncwarp();
        // dependency on the image (as the kernel's fragment loads): one word back into f
        f[1] += (float)(reinterpret_cast<const uint32_t*>(img[warp])[lane] & 1u) * 1e-30f;
    }
    const long long t1 = clock64();
    if (lane == 0) out[blockIdx.x * 32 + warp] = (t1 - t0) / iters;
    if (f[0] == 12345.f) out[0] = 0;  // keep f live
}


// correctness: the kernel's rotation (chain_rotate_to_smem + chain_load_frags) must give the same fragments
// and factors as the probe's stmatrix reference (stsm_rotate_to_smem + stsm_load_frags)
__global__ void check(const float* x, long long* out) {
    __shared__ __align__(16) uint8_t i0[kActSmemBlock], i1[kActSmemBlock];
    const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
    long long bad = 0, badm = 0;
    for (int b = 0; b < 16; ++b) {
        float f0[8], f1[8];
        for (int e = 0; e < 8; ++e) {
            f0[e] = x[b * 256 + rot_lane_element(lane) + 32 * e] * (b + 1);
            f1[e] = x[b * 256 + sig_lane(lane) + 32 * e] * (b + 1);
        }
        chain_rotate_to_smem(f0, 3, i0, lane);
        stsm_rotate_to_smem(f1, 3, i1, lane);
        __syncwarp();
        uint2 b0[8], b1[8];
        chain_load_frags(i0, g, t, b0);
        stsm_load_frags(i1, g, t, b1);
        for (int q = 0; q < 8; ++q) bad += (b0[q].x != b1[q].x) + (b0[q].y != b1[q].y);
        if (lane < 8) badm += reinterpret_cast<const float*>(i0 + 1024)[lane] != reinterpret_cast<const float*>(i1 + 1024)[lane];
        __syncwarp();
    }
    for (int o = 16; o; o >>= 1) { bad += __shfl_xor_sync(FULL, bad, o); badm += __shfl_xor_sync(FULL, badm, o); }
    if (lane == 0) { out[0] = bad; out[1] = badm; }
}

template <int VAR>
void run(const float* dx, long long* dout, const char* name) {
    for (int nw : {1, 4, 8, 16}) {
        rot_probe<VAR><<<148, 576>>>(dx, nw, 200, dout);
        cudaDeviceSynchronize();
        std::vector<long long> h(148 * 32);
        cudaMemcpy(h.data(), dout, h.size() * 8, cudaMemcpyDeviceToHost);
        double s = 0;
        for (int w = 0; w < nw; ++w) s += h[w];
        printf("%-28s warps %2d: %6.0f cycles per rotation\n", name, nw, s / nw);
    }
}

int main() {
    float* dx;
    long long* dout;
    cudaMalloc(&dx, 16 * 256 * 4);
    cudaMalloc(&dout, 148 * 32 * 8);
    std::vector<float> hx(16 * 256);
    for (size_t i = 0; i < hx.size(); ++i) hx[i] = sinf(0.37f * i) * (1 + i % 7);
    cudaMemcpy(dx, hx.data(), hx.size() * 4, cudaMemcpyHostToDevice);
    run<0>(dx, dout, "kernel rotation");
    run<1>(dx, dout, "FWHT only");
    run<2>(dx, dout, "+ 2 REDUX maxima");
    run<3>(dx, dout, "+ limbs/class diffs");
    run<4>(dx, dout, "+ 32 byte stores");
    run<5>(dx, dout, "swap-butterfly rotation");
    run<6>(dx, dout, "lean rotation");
    run<7>(dx, dout, "lean + stmatrix rotation");
    check<<<1, 32>>>(dx, dout);
    cudaDeviceSynchronize();
    long long hc[2];
    cudaMemcpy(hc, dout, 16, cudaMemcpyDeviceToHost);
    printf("fragment check (kernel rotation vs the probe's stmatrix reference, 16 blocks): %lld mismatching words, %lld meta f diffs\n", hc[0], hc[1]);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
