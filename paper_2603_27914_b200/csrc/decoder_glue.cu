// Decoder-stack glue (decoder.py): the one non-ITQ3 operation of a
// Llama-style decode step that does not fold into the chain launches -- RoPE + KV-cache append +
// grouped-query decode attention.  (RMSNorm, SiLU gating and the residual adds live in the chain
// kernel's decoder flags.)  Not on the ITQ3_S hot path; fp32 throughout.
#include "common.cuh"

namespace itq3 {

// Flash-decoding attention: CTA (h, sp) of a (query head, position split) grid handles positions
// [lo, hi) of 0..pos.  Every CTA applies RoPE (rotate-half) to its query and to its kv head's key at
// pos; the (group-leader head, split 0) CTA appends k / v to the cache.  A CTA writes its partial
// (max, sum of exp, exp-weighted V) to `ws`; the last split of a head to arrive (per-head counter,
// reset for the next launch) combines them.  Scores: one warp per position, four in flight;
// P V: 8 position classes x 128 dims, reduced in smem.
// qkv = [q (nh*hd) | k (nkv*hd) | v (nkv*hd)]; caches [nkv][ctx][hd]; out [nh*hd].
constexpr int kAttnSplits = 4;
__global__ void __launch_bounds__(1024) glue_rope_attention(const float* __restrict__ qkv, const float* __restrict__ cosb,
                                                           const float* __restrict__ sinb,
                                                           const int64_t* __restrict__ pos_p, float* __restrict__ kc,
                                                           float* __restrict__ vc, float* __restrict__ out, int nh,
                                                           int nkv, int ctx, float* __restrict__ ws,
                                                           unsigned* __restrict__ counters) {
    constexpr int HD = 128;
    __shared__ float qs[HD], kcur[HD], vcur[HD];
    __shared__ float ps[1024];
    __shared__ float red[32];
    __shared__ float part[8][HD];
    __shared__ bool last;
    const int h = blockIdx.x, sp = blockIdx.y, t = threadIdx.x, w = t >> 5, l = t & 31, kvh = h / (nh / nkv);
    const int64_t pos64 = *pos_p;
    if (pos64 < 0 || pos64 >= ctx) {  // beyond the KV cache: no cache write, zero output, error word set
        if (t < HD && sp == 0) out[(int64_t)h * HD + t] = 0.f;
        if (t == 0 && h == 0 && sp == 0) atomicOr(counters + nh, 1u);
        return;
    }
    const int pos = (int)pos64;
    const int chunk = (pos + kAttnSplits) / kAttnSplits;  // ceil((pos + 1) / splits)
    const int lo = sp * chunk, hi = min(pos + 1, lo + chunk);
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
        if (sp == 0 && h % (nh / nkv) == 0) {
            kch[(int64_t)pos * HD + t] = kv;
            vch[(int64_t)pos * HD + t] = vv;
        }
    }
    __syncthreads();
    float mx = -INFINITY;
    const float q0 = qs[l], q1 = qs[l + 32], q2 = qs[l + 64], q3 = qs[l + 96];
    for (int p0 = lo + w; p0 < hi; p0 += 32 * 4) {  // four positions per warp in flight
        float d[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int p = p0 + 32 * u;
            const float* kp = p == pos ? kcur : kch + (int64_t)min(p, pos) * HD;
            d[u] = p < hi ? q0 * kp[l] + q1 * kp[l + 32] + q2 * kp[l + 64] + q3 * kp[l + 96] : -INFINITY;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            for (int o = 16; o; o >>= 1) d[u] += __shfl_xor_sync(FULL, d[u], o);
            const int p = p0 + 32 * u;
            if (p < hi) {
                if (l == 0) ps[p - lo] = d[u];
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
    for (int p = lo + t; p < hi; p += blockDim.x) {
        const float e = __expf(ps[p - lo] - mx);
        ps[p - lo] = e;
        se += e;
    }
    for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(FULL, se, o);
    if (l == 0) red[w] = se;
    __syncthreads();
    se = red[l];
    for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(FULL, se, o);
    const int g = t >> 7, dcol = t & (HD - 1);
    const int vend = min(hi, pos);  // positions read from the cache; pos itself from smem
    float a8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // eight independent loads in flight
    int p = lo + g;
    for (; p + 56 < vend; p += 64)
#pragma unroll
        for (int u = 0; u < 8; ++u) a8[u] += ps[p + 8 * u - lo] * vch[(int64_t)(p + 8 * u) * HD + dcol];
    for (; p < vend; p += 8) a8[0] += ps[p - lo] * vch[(int64_t)p * HD + dcol];
    float acc = ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
    if (hi == pos + 1 && lo <= pos && ((pos - lo) & 7) == g) acc += ps[pos - lo] * vcur[dcol];
    part[g][dcol] = acc;
    __syncthreads();
    float* mine = ws + ((int64_t)h * kAttnSplits + sp) * (HD + 2);
    if (t < HD) {
        float o = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) o += part[j][t];
        mine[2 + t] = o;
    }
    if (t == 0) {
        mine[0] = mx;
        mine[1] = se;
    }
    __threadfence();
    __syncthreads();
    if (t == 0) {
        last = atomicAdd(counters + h, 1u) == kAttnSplits - 1;
        if (last) counters[h] = 0;  // ready for the next launch (graph replays)
    }
    __syncthreads();
    if (!last || t >= HD) return;
    __threadfence();
    const float* hw = ws + (int64_t)h * kAttnSplits * (HD + 2);
    float m = -INFINITY;
#pragma unroll
    for (int j = 0; j < kAttnSplits; ++j) m = fmaxf(m, __ldcg(hw + j * (HD + 2)));
    float num = 0.f, den = 0.f;
#pragma unroll
    for (int j = 0; j < kAttnSplits; ++j) {
        const float mj = __ldcg(hw + j * (HD + 2));
        const float f = mj == -INFINITY ? 0.f : __expf(mj - m);
        den += f * __ldcg(hw + j * (HD + 2) + 1);
        num += f * __ldcg(hw + j * (HD + 2) + 2 + t);
    }
    out[(int64_t)h * HD + t] = num / den;
}


// Grouped-query variant (n_heads / n_kv = G <= 4): CTA (kv head, split) of a (n_kv, 16) grid serves
// the G query heads that share the kv head, so every cached K / V row is read ONCE per launch (the
// per-head kernel above reads it G times).  128 G threads: RoPE of the G queries and of k; scores with
// a warp per position (lane = 4 dims, G dot products); per-head softmax over the split's positions;
// P V with thread (position class c, dim d) accumulating all G heads from one read of v[p][d].
// Partials (max, sum, G x 128 weighted V) go to ws; the last split of a kv head (counter) combines.
constexpr int kGqaSplits = 16;
template <int G>
__global__ void __launch_bounds__(128 * G) glue_gqa_attention(const float* __restrict__ qkv, const float* __restrict__ cosb,
                                                              const float* __restrict__ sinb,
                                                              const int64_t* __restrict__ pos_p, float* __restrict__ kc,
                                                              float* __restrict__ vc, float* __restrict__ out, int nh,
                                                              int nkv, int ctx, float* __restrict__ ws,
                                                              unsigned* __restrict__ counters) {
    constexpr int HD = 128, NT = 128 * G, NW = NT / 32, PCH = (1024 + kGqaSplits - 1) / kGqaSplits;
    __shared__ float qs[G][HD], kcur[HD], vcur[HD];
    __shared__ float ps[G][PCH];
    __shared__ float stat[G][2];
    __shared__ float part[G][G][HD];  // [position class][head][dim]
    __shared__ bool last;
    const int kvh = blockIdx.x, sp = blockIdx.y, t = threadIdx.x, w = t >> 5, l = t & 31;
    const int64_t pos64 = *pos_p;
    if (pos64 < 0 || pos64 >= ctx) {  // beyond the KV cache: no cache write, zero output, error word set
        if (sp == 0) out[(int64_t)kvh * G * HD + t] = 0.f;
        if (t == 0 && kvh == 0 && sp == 0) atomicOr(counters + nh, 1u);
        return;
    }
    const int pos = (int)pos64;
    const int chunk = (pos + kGqaSplits) / kGqaSplits;  // ceil((pos + 1) / splits) <= PCH
    const int lo = sp * chunk, hi = min(pos + 1, lo + chunk), n = max(0, hi - lo);
    float* kch = kc + (int64_t)kvh * ctx * HD;
    float* vch = vc + (int64_t)kvh * ctx * HD;
    {  // RoPE (rotate-half) of the G queries, k and v at pos
        const int g = t >> 7, i = t & (HD - 1), ih = i & (HD / 2 - 1);
        const float c = cosb[(int64_t)pos * (HD / 2) + ih], sn = sinb[(int64_t)pos * (HD / 2) + ih];
        auto rope = [&](const float* v) {
            const float a = v[ih], b = v[ih + HD / 2];
            return i < HD / 2 ? a * c - b * sn : a * sn + b * c;
        };
        qs[g][i] = rope(qkv + (int64_t)(kvh * G + g) * HD) * rsqrtf((float)HD);
        if (g == 0) {
            const float kv = rope(qkv + (int64_t)nh * HD + kvh * HD);
            const float vv = qkv[(int64_t)(nh + nkv) * HD + kvh * HD + i];
            kcur[i] = kv;
            vcur[i] = vv;
            if (sp == 0) {
                kch[(int64_t)pos * HD + i] = kv;
                vch[(int64_t)pos * HD + i] = vv;
            }
        }
    }
    __syncthreads();
    float qr[G][4];
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
        for (int j = 0; j < 4; ++j) qr[g][j] = qs[g][l + 32 * j];
    for (int p = lo + w; p < hi; p += NW) {
        const float* kp = p == pos ? kcur : kch + (int64_t)p * HD;
        const float k0 = kp[l], k1 = kp[l + 32], k2 = kp[l + 64], k3 = kp[l + 96];
        float d[G];
#pragma unroll
        for (int g = 0; g < G; ++g) d[g] = qr[g][0] * k0 + qr[g][1] * k1 + qr[g][2] * k2 + qr[g][3] * k3;
#pragma unroll
        for (int o = 16; o; o >>= 1)
#pragma unroll
            for (int g = 0; g < G; ++g) d[g] += __shfl_xor_sync(FULL, d[g], o);
        if (l == 0)
#pragma unroll
            for (int g = 0; g < G; ++g) ps[g][p - lo] = d[g];
    }
    __syncthreads();
    if (w < G) {  // softmax statistics of head w over this split's positions
        float m = -INFINITY;
        for (int i = l; i < n; i += 32) m = fmaxf(m, ps[w][i]);
        for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(FULL, m, o));
        float se = 0.f;
        for (int i = l; i < n; i += 32) {
            const float e = __expf(ps[w][i] - m);
            ps[w][i] = e;
            se += e;
        }
        for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(FULL, se, o);
        if (l == 0) {
            stat[w][0] = m;
            stat[w][1] = se;
        }
    }
    __syncthreads();
    {  // P V: thread (class c, dim d) takes positions lo + c, lo + c + G, ... for all G heads
        const int c = t >> 7, dcol = t & (HD - 1);
        float acc[G];
#pragma unroll
        for (int g = 0; g < G; ++g) acc[g] = 0.f;
        for (int i = c; i < n; i += G) {
            const int p = lo + i;
            const float v = p == pos ? vcur[dcol] : vch[(int64_t)p * HD + dcol];
#pragma unroll
            for (int g = 0; g < G; ++g) acc[g] += ps[g][i] * v;
        }
#pragma unroll
        for (int g = 0; g < G; ++g) part[c][g][dcol] = acc[g];
    }
    __syncthreads();
    float* mine = ws + (((int64_t)kvh * kGqaSplits + sp) * G) * (HD + 2);
    {
        const int g = t >> 7, dcol = t & (HD - 1);
        float o = 0.f;
#pragma unroll
        for (int c = 0; c < G; ++c) o += part[c][g][dcol];
        mine[g * (HD + 2) + 2 + dcol] = o;
        if (dcol == 0) {
            mine[g * (HD + 2)] = stat[g][0];
            mine[g * (HD + 2) + 1] = stat[g][1];
        }
    }
    __threadfence();
    __syncthreads();
    if (t == 0) {
        last = atomicAdd(counters + kvh, 1u) == kGqaSplits - 1;
        if (last) counters[kvh] = 0;  // ready for the next launch (graph replays)
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    const int g = t >> 7, dcol = t & (HD - 1);
    const float* hw = ws + (int64_t)kvh * kGqaSplits * G * (HD + 2) + g * (HD + 2);
    float m = -INFINITY;
#pragma unroll
    for (int j = 0; j < kGqaSplits; ++j) m = fmaxf(m, __ldcg(hw + j * G * (HD + 2)));
    float num = 0.f, den = 0.f;
#pragma unroll
    for (int j = 0; j < kGqaSplits; ++j) {
        const float mj = __ldcg(hw + j * G * (HD + 2));
        const float f = mj == -INFINITY ? 0.f : __expf(mj - m);
        den += f * __ldcg(hw + j * G * (HD + 2) + 1);
        num += f * __ldcg(hw + j * G * (HD + 2) + 2 + dcol);
    }
    out[(int64_t)(kvh * G + g) * HD + dcol] = num / den;
}

}  // namespace itq3

using namespace itq3;

extern "C" int64_t itq3_glue_attention_ws_nbytes(int n_heads) {
    // partials for the larger of the two launch shapes (per-head x 4 splits, grouped x 16 splits),
    // then n_heads u32 counters, then the out-of-cache error word
    const int splits = kGqaSplits > kAttnSplits ? kGqaSplits : kAttnSplits;
    return (int64_t)n_heads * (splits * (128 + 2) * 4 + 4) + 4;
}

extern "C" int itq3_glue_rope_attention(const float* qkv, const float* cos_tab, const float* sin_tab,
                                        const int64_t* pos, float* k_cache, float* v_cache, float* out, int n_heads,
                                        int n_kv, int head_dim, int ctx, void* ws, void* stream) {
    if (head_dim != 128 || ctx > 1024 || n_kv <= 0 || n_heads % n_kv) {
        set_error("itq3_glue_rope_attention: head_dim 128, ctx <= 1024, n_heads a multiple of n_kv");
        return ITQ3_E_UNSUPPORTED;
    }
    // ws: [n_heads][splits][2 + 128] fp32 partials, then n_heads u32 counters (zero before first use),
    // then one u32 error word (bit 0: a launch saw a position outside [0, ctx))
    float* part = (float*)ws;
    const int splits = kGqaSplits > kAttnSplits ? kGqaSplits : kAttnSplits;
    unsigned* cnt = (unsigned*)(part + (int64_t)n_heads * splits * (128 + 2));
    const int G = n_heads / n_kv;
    if (G == 4 || G == 2 || G == 1) {  // grouped-query kernel: one read of every cached K / V row
        cudaStream_t s = (cudaStream_t)stream;
        const dim3 grid((unsigned)n_kv, kGqaSplits);
        if (G == 4)
            glue_gqa_attention<4><<<grid, 512, 0, s>>>(qkv, cos_tab, sin_tab, pos, k_cache, v_cache, out, n_heads, n_kv,
                                                       ctx, part, cnt);
        else if (G == 2)
            glue_gqa_attention<2><<<grid, 256, 0, s>>>(qkv, cos_tab, sin_tab, pos, k_cache, v_cache, out, n_heads, n_kv,
                                                       ctx, part, cnt);
        else
            glue_gqa_attention<1><<<grid, 128, 0, s>>>(qkv, cos_tab, sin_tab, pos, k_cache, v_cache, out, n_heads, n_kv,
                                                       ctx, part, cnt);
        return check_launch("itq3_glue_rope_attention (grouped)");
    }
    glue_rope_attention<<<dim3(n_heads, kAttnSplits), 1024, 0, (cudaStream_t)stream>>>(
        qkv, cos_tab, sin_tab, pos, k_cache, v_cache, out, n_heads, n_kv, ctx, part, cnt);
    return check_launch("itq3_glue_rope_attention");
}
