// Block-level utilities of the reference API (pkg/src/itq3/quantizer.py:78-197): block statistics,
// ternary quantise / dequantise and the uniform b-bit baseline, on the device with the reference's
// float64 data flow (numpy's pairwise summation order, correctly rounded division and square root,
// round half away from zero).  These are the per-block building blocks the K1 encoder fuses; here
// they serve the drop-in API for single blocks and arbitrary arrays.
#include "common.cuh"

namespace itq3 {

// numpy's pairwise sum (umath loops_utils: blocks of 8 partial sums up to 128 elements, halves
// rounded down to a multiple of 8 above) of f(i), i in [0, n), float64, as an explicit-stack walk.
template <typename F>
__device__ double np_pairwise_sum(F f, int64_t n) {
    struct Frame {
        int64_t off, len;
        int state;  // 0: not started, 1: left half done
        double left;
    };
    Frame st[64];
    int sp = 0;
    st[0] = {0, n, 0, 0.0};
    double ret = 0.0;
    while (sp >= 0) {
        Frame& fr = st[sp];
        if (fr.len <= 128) {
            double res;
            if (fr.len < 8) {
                res = 0.0;
                for (int64_t i = 0; i < fr.len; ++i) res = __dadd_rn(res, f(fr.off + i));
            } else {
                double r[8];
                for (int j = 0; j < 8; ++j) r[j] = f(fr.off + j);
                int64_t i = 8;
                for (; i < fr.len - (fr.len % 8); i += 8)
                    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], f(fr.off + i + j));
                res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                                __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
                for (; i < fr.len; ++i) res = __dadd_rn(res, f(fr.off + i));
            }
            ret = res;
            --sp;
        } else {
            int64_t n2 = fr.len / 2;
            n2 -= n2 % 8;
            if (fr.state == 0) {
                fr.state = 1;
                st[sp + 1] = {fr.off, n2, 0, 0.0};
                ++sp;
                continue;
            }
            if (fr.state == 1) {
                fr.state = 2;
                fr.left = ret;
                st[sp + 1] = {fr.off + n2, fr.len - n2, 0, 0.0};
                ++sp;
                continue;
            }
            ret = __dadd_rn(fr.left, ret);
            --sp;
        }
        // a finished child hands `ret` to its parent, which resumes at its saved state
    }
    return ret;
}

// x^4 as the correctly rounded value of the exact fourth power in almost every case (the
// reference's numpy ** 4 is libm pow): x^2 = h + l exactly, then (h + l)^2 ~ h^2 + 2 h l.
__device__ __forceinline__ double pow4(double x) {
    const double h = __dmul_rn(x, x);
    const double l = __fma_rn(x, x, -h);
    const double hh = __dmul_rn(h, h);
    const double e = __fma_rn(h, h, -hh);
    return __dadd_rn(hh, __fma_rn(2.0 * h, l, e));
}

// out = {n, mean, sigma, l1, linf, excess_kurtosis} (quantizer.py:78-99)
__global__ void block_stats_kernel(const double* __restrict__ v, int64_t n, double* __restrict__ out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const double mean = __ddiv_rn(np_pairwise_sum([&](int64_t i) { return v[i]; }, n), (double)n);
    const double var = __ddiv_rn(np_pairwise_sum([&](int64_t i) {
                                     const double d = __dsub_rn(v[i], mean);
                                     return __dmul_rn(d, d);
                                 }, n),
                                 (double)n);
    const double sigma = __dsqrt_rn(var);
    double kurt = 0.0;
    if (sigma > 0.0) {
        const double m4 = __ddiv_rn(np_pairwise_sum([&](int64_t i) { return pow4(__dsub_rn(v[i], mean)); }, n),
                                    (double)n);
        kurt = __dsub_rn(__ddiv_rn(m4, __dmul_rn(var, var)), 3.0);
    }
    const double l1 = np_pairwise_sum([&](int64_t i) { return fabs(v[i]); }, n);
    double linf = 0.0;
    for (int64_t i = 0; i < n; ++i) linf = fmax(linf, fabs(v[i]));
    out[0] = (double)n;
    out[1] = mean;
    out[2] = sigma;
    out[3] = l1;
    out[4] = linf;
    out[5] = kurt;
}

// codes = clip(copysign(floor(|x / d| + 0.5), x / d) + z, -1, 1) (quantizer.py:152-168)
__global__ void ternary_quantize_kernel(const double* __restrict__ x, int64_t n, double d, int z,
                                        int8_t* __restrict__ codes) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double q = __ddiv_rn(x[i], d);
    const double r = copysign(floor(__dadd_rn(fabs(q), 0.5)), q);
    codes[i] = (int8_t)fmin(fmax(__dadd_rn(r, (double)z), -1.0), 1.0);
}

// d * (code - z) (quantizer.py:171-181)
__global__ void ternary_dequantize_kernel(const int8_t* __restrict__ codes, int64_t n, double d, int z,
                                          double* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = __dmul_rn(d, (double)((int)codes[i] - z));
}

// clip(delta * floor(x / delta + 0.5), wmin, wmax) (quantizer.py:184-197)
__global__ void uniform_quantize_kernel(const double* __restrict__ x, int64_t n, double delta, double wmin,
                                        double wmax, double* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double y = __dmul_rn(delta, floor(__dadd_rn(__ddiv_rn(x[i], delta), 0.5)));
    out[i] = fmin(fmax(y, wmin), wmax);
}

}  // namespace itq3

using namespace itq3;

extern "C" int itq3_block_stats(const double* v, int64_t n, double* out, void* stream) {
    if (n <= 0) {
        set_error("block_stats: expects a non-empty 1-D block");
        return ITQ3_E_DOMAIN;
    }
    block_stats_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(v, n, out);
    return check_launch("itq3_block_stats");
}

extern "C" int itq3_ternary_quantize(const double* x, int64_t n, double d, int z, int8_t* codes, void* stream) {
    if (n <= 0) return ITQ3_OK;
    ternary_quantize_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(x, n, d, z, codes);
    return check_launch("itq3_ternary_quantize");
}

extern "C" int itq3_ternary_dequantize(const int8_t* codes, int64_t n, double d, int z, double* out, void* stream) {
    if (n <= 0) return ITQ3_OK;
    ternary_dequantize_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(codes, n, d, z, out);
    return check_launch("itq3_ternary_dequantize");
}

extern "C" int itq3_uniform_quantize(const double* x, int64_t n, double delta, double wmin, double wmax, double* out,
                                     void* stream) {
    if (n <= 0) return ITQ3_OK;
    uniform_quantize_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(x, n, delta, wmin, wmax,
                                                                                          out);
    return check_launch("itq3_uniform_quantize");
}
