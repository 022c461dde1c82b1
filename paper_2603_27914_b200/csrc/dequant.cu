// K2t: dequantize_tensor / decode_block (codec.py:152-202) on the 5th-gen tensor cores.
//
// For a 256-block with stored scale d, zero-point z and codes c: w_hat = (d / 16) * H t with
// t = c - 1 - z in {-2..2} (decode_block: y = d (c - z'), then the unnormalised inverse FWHT and the
// exact 1/16).  H is symmetric, so 128 consecutive blocks (one per TMEM lane) form ONE GEMM
//     D[128 blocks x 256] = T[128 x 256] * (H / 16)[256 x 256]
// with A = T in f16 (small integers, exact), B = H/16 in f16 (+-2^-4, exact), fp32 accumulation:
// every partial sum is a multiple of 1/16 below 2^5 in magnitude, so D = I / 16 exactly, and the
// epilogue's d * D (11-bit x 10-bit significands) is exact in fp32 -- the reference's float64 value,
// bit for bit, for every block with a finite positive scale.  Blocks whose scale is zero, negative,
// infinite or NaN (signed zeros / NaN propagation follow the butterfly's order there) are left to
// the exact per-block kernel (codec.cu dequant_kernel, `unsafe_only` pass launched right after).
//
// The IFWHT therefore costs tensor-core time instead of 8 dependent shuffle stages per weight
// (the warp-per-block kernel is SHFL-bound at ~0.4 Gweights/ms); this kernel is bound by the HBM
// write of the decoded weights.
//
// Per CTA (persistent, one per SM): H/16 resident in shared memory (128 KB, SWIZZLE_128B K-major,
// built once); 10 warps: warp 1 allocates TMEM (A ring 2 x 128 columns, D ring 2 x 128 columns)
// and issues the MMAs (M = 128, N = 128 per half tile, K = 16); warps 2-5 expand codes into TMEM
// (one block per thread); warps 6-9 drain D, scale by d and store the rows.
#include "common.cuh"

namespace itq3dq {

using itq3::FULL;

constexpr int kThreads = 32 * 14;  // warp 1 MMA, 2-5 expanders, 6-9 / 10-13 epilogue of half 0 / 1

__device__ __forceinline__ uint32_t saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t* b, unsigned n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "W_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W_%=;\n}\n" ::"r"(saddr(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void commit(uint64_t* b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(b))
                 : "memory");
}
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n selp.b32 %0, 1, 0, P;\n}\n" : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ uint64_t desc_sw128(uint32_t a) {
    return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint32_t sw128_off(int r, int j) {
    return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((j ^ (r & 7)) << 4));
}

// blocks the tensor-core path reproduces exactly: scale finite and > 0, zero-point one of +-0, +-1
__device__ __forceinline__ bool block_safe(uint32_t szw) {
    const uint16_t sb = (uint16_t)(szw & 0xffffu), zb = (uint16_t)(szw >> 16);
    return sb != 0 && !(sb & 0x8000) && (sb & 0x7c00) != 0x7c00 &&
           (zb == 0 || zb == 0x8000 || zb == 0x3C00 || zb == 0xBC00);
}

// optional per-CTA cycle accounting (tools/codec_bench.py --trace), 16 counters per CTA, null = off
__device__ unsigned long long* g_dq_trace = nullptr;
#define DQ_T(acc, stmt)                       \
    {                                         \
        const long long _t0 = clock64();      \
        stmt;                                 \
        acc += clock64() - _t0;               \
    }

constexpr int kStageRow = 528;  // staged output bytes per block: 512 + 16 pad (conflict-free 16-B stores)
// B = H_128 / 16 only: H_256[n][k] = H_128[n mod 128][k mod 128] * (-1)^(bit 7 of n and k), so
//   D_half0 = (T_lo + T_hi) H_128 / 16,  D_half1 = (T_lo - T_hi) H_128 / 16
// with T_hi negated through the instruction descriptor (a_negate) for half 1.
struct Smem {
    uint8_t H[2][128 * 128];  // [64-k chunk][128 rows n][128 B], SW128: 32 KB
    uint8_t stage[2][128][kStageRow];  // per epilogue group: one 512-byte output run per block
    uint32_t runmask[2][4];            // per group and warp: blocks whose run is stored (ballot)
    uint64_t aready[2], aempty[2], dfull[2], dempty[2];
    uint32_t tmem_base;
};

template <typename TOut>
__global__ void __launch_bounds__(kThreads, 1)
    dequant_tc_kernel(const uint8_t* __restrict__ payload, int64_t n_blocks, int64_t numel, TOut* __restrict__ out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Smem& sm = *reinterpret_cast<Smem*>(base);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t ntiles = (n_blocks + 127) / 128;

    // H_128/16 in f16: element (n, k) = +-0.0625 by the parity of popc(n & k) (Sylvester order)
    for (int i = threadIdx.x; i < 2 * 128 * 8; i += kThreads) {
        const int kc = i >> 10, n = (i >> 3) & 127, j = i & 7;
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int k0 = 64 * kc + 8 * j + 2 * e;
            const uint32_t lo = (__popc(n & k0) & 1) ? 0xAC00u : 0x2C00u;
            const uint32_t hi = (__popc(n & (k0 + 1)) & 1) ? 0xAC00u : 0x2C00u;
            w[e] = lo | (hi << 16);
        }
        *reinterpret_cast<uint4*>(sm.H[kc] + sw128_off(n, j)) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor-core reads
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s) {
            bar_init(&sm.aready[s], 4);
            bar_init(&sm.aempty[s], 1);
            bar_init(&sm.dfull[s], 1);
            bar_init(&sm.dempty[s], 4);  // the 4 warps of epilogue group s
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(saddr(&sm.tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = sm.tmem_base;
    constexpr uint32_t kColA = 256;

    if (warp == 1) {
        // MMA issuer: per tile two N = 128 halves into D slots 0/1; A slot = tile parity
        const uint32_t idesc = (1u << 4) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        uint32_t i = 0;
        long long c_ar = 0, c_de = 0;
        const long long c0 = clock64();
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
            const uint32_t a = i & 1u;
            DQ_T(c_ar, bar_wait(&sm.aready[a], (i >> 1) & 1u));
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                DQ_T(c_de, bar_wait(&sm.dempty[h], (i & 1u) ^ 1u));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if (elect_one()) {
#pragma unroll
                    for (int s = 0; s < 16; ++s) {  // k = 16 s .. 16 s + 15
                        const uint64_t bd = desc_sw128(saddr(sm.H[(s >> 2) & 1]) + 32 * (s & 3));
                        const uint32_t acc = s > 0;
                        const uint32_t id = (h == 1 && s >= 8) ? (idesc | (1u << 13)) : idesc;  // -T_hi
                        asm volatile(
                            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                            " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem + 128u * h),
                            "r"(tmem + kColA + 128u * a + 8u * s), "l"(bd), "r"(id), "r"(acc));
                    }
                    commit(&sm.dfull[h]);
                    if (h == 1) commit(&sm.aempty[a]);
                }
                __syncwarp();
            }
        }
        if (g_dq_trace && lane == 0) {
            g_dq_trace[blockIdx.x * 16 + 3] = c_ar;
            g_dq_trace[blockIdx.x * 16 + 4] = c_de;
            g_dq_trace[blockIdx.x * 16 + 5] = clock64() - c0;
            g_dq_trace[blockIdx.x * 16 + 9] = i;
        }
    } else if (warp >= 2 && warp < 6) {
        // expanders: thread = TMEM lane = block; t = c - 1 - z as f16 pairs, 128 columns per block
        const int q = warp & 3, r = 32 * q + lane;
        const uint32_t ta_row = tmem + ((uint32_t)(32 * q) << 16) + kColA;
        uint32_t i = 0;
        long long c_ae = 0, c_ld = 0;
        const long long c0 = clock64();
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
            const uint32_t a = i & 1u;
            const int64_t g = t * 128 + r;
            uint32_t p0[8], p1[8], sz = 0;
            const long long cl = clock64();
            if (g < n_blocks) {
                const uint32_t* p = reinterpret_cast<const uint32_t*>(payload + g * 100);
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    p0[e] = __ldg(p + e);
                    p1[e] = __ldg(p + 8 + e);
                }
                sz = __ldg(p + 24);
            } else {
#pragma unroll
                for (int e = 0; e < 8; ++e) p0[e] = p1[e] = 0;
            }
            const uint16_t zb = (uint16_t)(sz >> 16);
            c_ld += clock64() - cl;
            const int z = zb == 0x3C00 ? 1 : (zb == 0xBC00 ? -1 : 0);  // int(decode_f16(zp)) for valid blocks
            const uint32_t off2 = (uint32_t)__half_as_ushort(__int2half_rn(1025 + z)) * 0x10001u;
            DQ_T(c_ae, bar_wait(&sm.aempty[a], ((i >> 1) & 1u) ^ 1u));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
            for (int st = 0; st < 4; ++st) {  // 32 columns = k 64 st .. 64 st + 63
                uint32_t v[32];
#pragma unroll
                for (int ww = 0; ww < 4; ++ww) {
                    const int w = 4 * st + ww;  // 16-k group: k = 16 w .. 16 w + 15
                    const uint32_t x = (p0[w >> 1] >> (16 * (w & 1))) & 0xFFFFu;
                    const uint32_t y = (p1[w >> 1] >> (16 * (w & 1))) & 0xFFFFu;
                    // bits 2m / 2m+1 = (plane 0, plane 1) of k = 16 w + 2 m; bits 16 + 2m .. of k + 1
                    const uint32_t W = (x & 0x5555u) | ((y & 0x5555u) << 1) | ((x & 0xAAAAu) << 15) | ((y & 0xAAAAu) << 16);
#pragma unroll
                    for (int m = 0; m < 8; ++m) {
                        const uint32_t cv = ((W >> (2 * m)) & 0x00030003u) | 0x64006400u;  // f16x2 1024 + c
                        const __half2 tv = __hsub2(*reinterpret_cast<const __half2*>(&cv),
                                                   *reinterpret_cast<const __half2*>(&off2));  // c - 1 - z, exact
                        v[8 * ww + m] = *reinterpret_cast<const uint32_t*>(&tv);
                    }
                }
                asm volatile(
                    "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
                    "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(
                        ta_row + 128u * a + 32u * st),
                    "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                    "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
                    "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
                    "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
                    : "memory");
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) bar_arrive(&sm.aready[a]);
        }
        if (g_dq_trace && warp == 2 && lane == 0) {
            g_dq_trace[blockIdx.x * 16 + 0] = c_ae;
            g_dq_trace[blockIdx.x * 16 + 1] = clock64() - c0;
            g_dq_trace[blockIdx.x * 16 + 2] = c_ld;
        }
    } else if (warp >= 6) {
        // epilogue group h (4 warps, D half h): thread = block; d * D is staged in shared memory as
        // 512-byte runs (128 fp32, or 64 fp64 per pass), then the group writes the runs back with
        // coalesced 16-byte stores, one warp instruction per run (cp.async.bulk per thread would
        // serialise 128 small requests on the SM's TMA unit)
        const int q = warp & 3, r = 32 * q + lane, h = (warp - 6) >> 2;
        const uint32_t td_row = tmem + ((uint32_t)(32 * q) << 16);
        const uint32_t srow = saddr(sm.stage[h][r]);
        constexpr int kPer = 512 / (int)sizeof(TOut);  // outputs per staged run
        constexpr int kPasses = 128 / kPer;            // 1 (fp32) or 2 (fp64) runs per half
        uint32_t i = 0;
        long long c_df = 0, c_wg = 0;
        const long long c0 = clock64();
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
            const int64_t g = t * 128 + r;
            uint32_t szw = 0;
            if (g < n_blocks) szw = __ldg(reinterpret_cast<const uint32_t*>(payload + g * 100 + 96));
            const float d = __half2float(__ushort_as_half((uint16_t)(szw & 0xffffu)));
            const bool full = (g + 1) * 256 <= numel;
            const bool write = g < n_blocks && block_safe(szw);
            DQ_T(c_df, bar_wait(&sm.dfull[h], i & 1u));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
            for (int ps = 0; ps < kPasses; ++ps) {
#pragma unroll
                for (int cc = 0; cc < kPer / 32; ++cc) {
                    const int c = ps * (kPer / 32) + cc;  // 32-column chunk of the half
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
                    if (c == 3) {  // D half drained: the MMAs of the next tile may overwrite it
                        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                        __syncwarp();
                        if (lane == 0) bar_arrive(&sm.dempty[h]);
                    }
                    if (write && !full) {  // the ragged last block: plain stores by its owner
                        const int64_t o = g * 256 + 128 * h + 32 * c;
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (o + j < numel) out[o + j] = (TOut)(d * __uint_as_float(v[j]));
                    }
                    const uint32_t sa = srow + (uint32_t)sizeof(TOut) * 32u * cc;
                    if constexpr (sizeof(TOut) == 4) {
#pragma unroll
                        for (int j = 0; j < 32; j += 4)
                            asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(sa + 4u * j),
                                         "f"(d * __uint_as_float(v[j])), "f"(d * __uint_as_float(v[j + 1])),
                                         "f"(d * __uint_as_float(v[j + 2])), "f"(d * __uint_as_float(v[j + 3]))
                                         : "memory");
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; j += 2)
                            asm volatile("st.shared.v2.f64 [%0], {%1,%2};" ::"r"(sa + 8u * j),
                                         "d"((double)(d * __uint_as_float(v[j]))),
                                         "d"((double)(d * __uint_as_float(v[j + 1])))
                                         : "memory");
                    }
                }
                // run flags: bit 0 = store this block's run (safe, in range and not the ragged tail)
                const uint32_t mine = (write && full) ? 1u : 0u;
                const uint32_t wmask = __ballot_sync(FULL, mine);
                if (lane == 0) sm.runmask[h][q] = wmask;
                DQ_T(c_wg, asm volatile("bar.sync %0, 128;" ::"r"(1 + h) : "memory"));
                // the warp of lane quarter q writes the runs of the tile's blocks 32 q .. 32 q + 31
                const uint32_t rm = sm.runmask[h][q];
#pragma unroll 1
                for (int jj = 0; jj < 32; ++jj) {
                    const int j = 32 * q + jj;
                    if (!((rm >> jj) & 1u)) continue;
                    const int64_t gj = t * 128 + j;
                    const uint4 val = *reinterpret_cast<const uint4*>(sm.stage[h][j] + 16 * lane);
                    *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(out + gj * 256 + 128 * h + ps * kPer) +
                                              16 * lane) = val;
                }
                asm volatile("bar.sync %0, 128;" ::"r"(1 + h) : "memory");  // staging free for the next pass
            }
        }
        if (g_dq_trace && warp == 6 && lane == 0) {
            g_dq_trace[blockIdx.x * 16 + 6] = c_df;
            g_dq_trace[blockIdx.x * 16 + 7] = clock64() - c0;
            g_dq_trace[blockIdx.x * 16 + 8] = c_wg;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

}  // namespace itq3dq

// Host side (called from codec.cu's itq3_dequant for block_n 256, variant s).
template <typename TOut>
int itq3_dequant_tc(const uint8_t* payload, int64_t n_blocks, int64_t numel, TOut* out, cudaStream_t s) {
    using namespace itq3dq;
    const int smem = (int)sizeof(Smem) + 1024;
    static std::atomic<unsigned long long> attr{0};
    if (int rc = itq3::ensure_smem_attr(dequant_tc_kernel<TOut>, smem, attr, "itq3_dequant: smem attribute")) return rc;
    const int sms = itq3::device_sms();
    const int64_t ntiles = (n_blocks + 127) / 128;
    const unsigned grid = (unsigned)(ntiles < sms ? ntiles : sms);
    dequant_tc_kernel<TOut><<<grid, kThreads, smem, s>>>(payload, n_blocks, numel, out);
    return itq3::check_launch("itq3_dequant (tensor cores)");
}

extern "C" int itq3_dequant_set_trace(void* buf) {
    unsigned long long* p = (unsigned long long*)buf;
    return cudaMemcpyToSymbol(itq3dq::g_dq_trace, &p, sizeof(p)) == cudaSuccess ? 0
                                                                              : itq3::check_launch("itq3_dequant_set_trace");
}

template int itq3_dequant_tc<float>(const uint8_t*, int64_t, int64_t, float*, cudaStream_t);
template int itq3_dequant_tc<double>(const uint8_t*, int64_t, int64_t, double*, cudaStream_t);
