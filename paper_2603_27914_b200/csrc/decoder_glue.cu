// Decoder-stack glue (decoder.py): the non-ITQ3 operations of a
// Llama-style decode step fused into three small kernels so that a layer is 4 GEMV launches + 4
// glue launches.  Not on the ITQ3_S hot path; fp32 throughout.
#include "common.cuh"

namespace itq3 {

constexpr int kGlueThreads = 1024;

__device__ __forceinline__ float block_sum(float v, float* red) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    v = l < (int)(blockDim.x >> 5) ? red[l] : 0.f;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

// x += r (if r), then out = x * rsqrt(mean(x^2) + eps) * gain (if gain; else out = x).  One CTA;
// each thread keeps its (up to 8) elements in registers across the reduction.
__global__ void __launch_bounds__(kGlueThreads) glue_residual_rmsnorm(float* __restrict__ x,
                                                                     const float* __restrict__ r,
                                                                     const float* __restrict__ gain,
                                                                     float* __restrict__ out, int n, float eps) {
    __shared__ float red[32];
    constexpr int kPer = 8;  // n <= 8 * 1024
    float v[kPer];
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const int i = threadIdx.x + j * kGlueThreads;
        v[j] = 0.f;
        if (i < n) {
            v[j] = x[i] + (r ? r[i] : 0.f);
            if (r) x[i] = v[j];
            ss += v[j] * v[j];
        }
    }
    float s = 1.f;
    if (gain) s = rsqrtf(block_sum(ss, red) / (float)n + eps);
    if (!out) return;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const int i = threadIdx.x + j * kGlueThreads;
        if (i < n) out[i] = gain ? v[j] * s * gain[i] : v[j];
    }
}

// One CTA (1024 threads) per query head: RoPE (rotate-half) of its query and of its kv head's key at
// position pos, append k / v at pos (the group's first head writes the cache), then softmax
// attention over positions 0..pos -- the current position from shared memory, earlier ones from
// the cache.  Scores: one warp per position; P V: 8 position classes x 128 dims, reduced in smem.
// qkv = [q (nh*hd) | k (nkv*hd) | v (nkv*hd)]; caches [nkv][ctx][hd]; out [nh*hd].
__global__ void __launch_bounds__(1024) glue_rope_attention(const float* __restrict__ qkv, const float* __restrict__ cosb,
                                                           const float* __restrict__ sinb,
                                                           const int64_t* __restrict__ pos_p, float* __restrict__ kc,
                                                           float* __restrict__ vc, float* __restrict__ out, int nh,
                                                           int nkv, int ctx) {
    constexpr int HD = 128;
    __shared__ float qs[HD], kcur[HD], vcur[HD];
    __shared__ float ps[1024];
    __shared__ float red[32];
    __shared__ float part[8][HD];
    const int h = blockIdx.x, t = threadIdx.x, w = t >> 5, l = t & 31, kvh = h / (nh / nkv);
    const int pos = (int)*pos_p;
    float* kch = kc + (int64_t)kvh * ctx * HD;
    float* vch = vc + (int64_t)kvh * ctx * HD;
    if (t < HD) {
        const int i = t & (HD / 2 - 1);
        const float c = cosb[(int64_t)pos * (HD / 2) + i], s = sinb[(int64_t)pos * (HD / 2) + i];
        auto rope = [&](const float* v) {
            const float a = v[i], b = v[i + HD / 2];
            return t < HD / 2 ? a * c - b * s : a * s + b * c;
        };
        const float kv = rope(qkv + (int64_t)nh * HD + kvh * HD);
        const float vv = qkv[(int64_t)(nh + nkv) * HD + kvh * HD + t];
        qs[t] = rope(qkv + (int64_t)h * HD) * rsqrtf((float)HD);
        kcur[t] = kv;
        vcur[t] = vv;
        if (h % (nh / nkv) == 0) {
            kch[(int64_t)pos * HD + t] = kv;
            vch[(int64_t)pos * HD + t] = vv;
        }
    }
    __syncthreads();
    float mx = -INFINITY;
    const float q0 = qs[l], q1 = qs[l + 32], q2 = qs[l + 64], q3 = qs[l + 96];
    for (int p0 = w; p0 <= pos; p0 += 32 * 4) {  // four positions per warp in flight
        float d[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int p = p0 + 32 * u;
            const float* kp = p == pos ? kcur : kch + (int64_t)min(p, pos) * HD;
            d[u] = p <= pos ? q0 * kp[l] + q1 * kp[l + 32] + q2 * kp[l + 64] + q3 * kp[l + 96] : -INFINITY;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            for (int o = 16; o; o >>= 1) d[u] += __shfl_xor_sync(FULL, d[u], o);
            const int p = p0 + 32 * u;
            if (p <= pos) {
                if (l == 0) ps[p] = d[u];
                mx = fmaxf(mx, d[u]);
            }
        }
    }
    if (l == 0) red[w] = mx;
    __syncthreads();
    mx = red[l];
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, o));
    __syncthreads();
    float se = 0.f;
    for (int p = t; p <= pos; p += blockDim.x) {
        const float e = __expf(ps[p] - mx);
        ps[p] = e;
        se += e;
    }
    for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(FULL, se, o);
    if (l == 0) red[w] = se;
    __syncthreads();
    se = red[l];
    for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(FULL, se, o);
    const int g = t >> 7, dcol = t & (HD - 1);
    float a8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // eight independent loads in flight
    int p = g;
    for (; p + 56 < pos; p += 64)
#pragma unroll
        for (int u = 0; u < 8; ++u) a8[u] += ps[p + 8 * u] * vch[(int64_t)(p + 8 * u) * HD + dcol];
    for (; p < pos; p += 8) a8[0] += ps[p] * vch[(int64_t)p * HD + dcol];
    float acc = ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
    if ((pos & 7) == g) acc += ps[pos] * vcur[dcol];
    part[g][dcol] = acc;
    __syncthreads();
    if (t < HD) {
        float o = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) o += part[j][t];
        out[(int64_t)h * HD + t] = o / se;
    }
}

__global__ void glue_silu_mul(const float* __restrict__ gu, float* __restrict__ out, int inter) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= inter) return;
    const float g = gu[i];
    out[i] = g / (1.f + __expf(-g)) * gu[inter + i];
}

}  // namespace itq3

using namespace itq3;

extern "C" int itq3_glue_residual_rmsnorm(float* x, const float* r, const float* gain, float* out, int n, float eps,
                                          void* stream) {
    if (n <= 0 || n > 8 * kGlueThreads) {
        set_error("itq3_glue_residual_rmsnorm: 0 < n <= %d", 8 * kGlueThreads);
        return ITQ3_E_SHAPE;
    }
    glue_residual_rmsnorm<<<1, kGlueThreads, 0, (cudaStream_t)stream>>>(x, r, gain, out, n, eps);
    return check_launch("itq3_glue_residual_rmsnorm");
}

extern "C" int itq3_glue_rope_attention(const float* qkv, const float* cos_tab, const float* sin_tab,
                                        const int64_t* pos, float* k_cache, float* v_cache, float* out, int n_heads,
                                        int n_kv, int head_dim, int ctx, void* stream) {
    if (head_dim != 128 || ctx > 1024 || n_kv <= 0 || n_heads % n_kv) {
        set_error("itq3_glue_rope_attention: head_dim 128, ctx <= 1024, n_heads a multiple of n_kv");
        return ITQ3_E_UNSUPPORTED;
    }
    glue_rope_attention<<<n_heads, 1024, 0, (cudaStream_t)stream>>>(qkv, cos_tab, sin_tab, pos, k_cache, v_cache, out,
                                                                   n_heads, n_kv, ctx);
    return check_launch("itq3_glue_rope_attention");
}

extern "C" int itq3_glue_silu_mul(const float* gu, float* out, int inter, void* stream) {
    glue_silu_mul<<<(inter + 255) / 256, 256, 0, (cudaStream_t)stream>>>(gu, out, inter);
    return check_launch("itq3_glue_silu_mul");
}
