// K8: the evaluation harness -- eval_error / eval_container / rotation_benefit
// (compute.py:136-356) -- on the device, bit-exact with the reference.
//
// One warp per block computes, in registers, everything the reference derives from that block:
// the rotated grid reconstruction (or, for eval_container, the stored codes/scales), the
// unrotated ternary baseline, the uniform 3-bit baseline, the clamp mask, the zero count and
// the grid bound.  It writes the per-element squared errors of the three codecs (flat, in the
// reference's row-major order) and per-block statistics.  The reductions then replay numpy's
// add.reduce tree (pairwise summation, loops_utils.h.src) exactly, so mse / linf / the
// baselines equal the reference's floats; only frobenius_rel depends on BLAS ddot's order in the
// reference and is reproduced to rounding.
//
// Semantics follow the reference's *vectorised* encoder (compute.py:146-201): scales are cast
// with astype(float16) (overflow -> inf), not encode_f16's saturation.
#include "common.cuh"

namespace itq3 {

// float64 -> float16 -> float64 exactly as ndarray.astype(np.float16) does (RNE, overflow -> inf).
__device__ __forceinline__ double f16_cast(double x) {
    if (fabs(x) >= 65520.0) return copysign(__longlong_as_double(0x7ff0000000000000ll), x);
    return f16_bits_to_f64(f64_to_f16_bits(x));
}

constexpr int kEvalWarps = 4;

// Grid quantisation of one (n,) row held in stride layout: compute.py:169-201 (_ternary_blocks).
// v: values (rotated coefficients or raw weights); sm: per-warp scratch of N doubles.
// Outputs the reconstruction d16*(code - z), the integer code, the clamp flag and the grid bound.
template <int N>
__device__ __forceinline__ void grid_quant(const double (&v)[N / 32], int lane, double* sm, int ss, int policy,
                                           double coeff, int symmetric, double (&rec)[N / 32], int (&code)[N / 32],
                                           bool (&clamp)[N / 32], double& budget) {
    constexpr int E = N / 32;
    constexpr int M = N / kSubBlocks;
#pragma unroll
    for (int e = 0; e < E; ++e) sm[lane + 32 * e] = v[e];
    __syncwarp();
    const double mu = __ddiv_rn(warp_pairwise_sum(sm, N, lane), (double)N);
    double d16_e[E], deff_e[E];
    double z = 0.0;
    auto zp = [&](double d_eff) {  // compute.py:162-166
        if (symmetric) return 0.0;
        const double r = __ddiv_rn(mu, d_eff);
        return clip1(-copysign(floor(__dadd_rn(fabs(r), 0.5)), r));
    };
    if (!ss) {
        __syncwarp();
        double d;
        if (policy == ITQ3_POLICY_MEAN_ABS) {
#pragma unroll
            for (int e = 0; e < E; ++e) sm[lane + 32 * e] = fabs(v[e]);
            __syncwarp();
            d = __dmul_rn(2.0 / 3.0, __ddiv_rn(warp_pairwise_sum(sm, N, lane), (double)N));
        } else {
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const double c = __dsub_rn(v[e], mu);
                sm[lane + 32 * e] = __dmul_rn(c, c);
            }
            __syncwarp();
            d = __dmul_rn(coeff, __dsqrt_rn(__ddiv_rn(warp_pairwise_sum(sm, N, lane), (double)N)));
        }
        const double d_raw = d > 0.0 ? d : 1e-8;  // EPSILON_D
        const double d16 = f16_cast(d_raw);
        const double d_eff = d16 > 0.0 ? d16 : d_raw;
        z = zp(d_eff);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            d16_e[e] = d16;
            deff_e[e] = d_eff;
        }
        budget = __ddiv_rn(__dmul_rn((double)N, __dmul_rn(d16, d16)), 4.0);
    } else {
        // lane s < 8 owns sub-block s (stats over the M-element sub-row, pairwise)
        double mean_s = 0.0, d_raw_s = 0.0;
        if (lane < kSubBlocks) mean_s = __ddiv_rn(serial_pairwise_sum(sm + lane * M, M), (double)M);
        __syncwarp();
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int j = lane + 32 * e;
            if (policy == ITQ3_POLICY_MEAN_ABS) {
                sm[j] = fabs(v[e]);
            } else {
                const double c = __dsub_rn(v[e], __shfl_sync(FULL, mean_s, j / M));
                sm[j] = __dmul_rn(c, c);
            }
        }
        __syncwarp();
        if (lane < kSubBlocks) {
            const double s = __ddiv_rn(serial_pairwise_sum(sm + lane * M, M), (double)M);
            const double d = policy == ITQ3_POLICY_MEAN_ABS ? __dmul_rn(2.0 / 3.0, s) : __dmul_rn(coeff, __dsqrt_rn(s));
            d_raw_s = d > 0.0 ? d : 1e-8;
        }
        const double d16_s = f16_cast(d_raw_s);
        const double deff_s = d16_s > 0.0 ? d16_s : d_raw_s;
        double r8[8], q8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            r8[k] = __shfl_sync(FULL, d_raw_s, k);
            const double dk = __shfl_sync(FULL, d16_s, k);
            q8[k] = __dmul_rn(dk, dk);
        }
        const double mean_raw = __ddiv_rn(serial_pairwise_sum(r8, 8), 8.0);
        double db = f16_cast(mean_raw);
        db = db > 0.0 ? db : mean_raw;
        z = zp(db);
        budget = __ddiv_rn(__dmul_rn((double)M, serial_pairwise_sum(q8, 8)), 4.0);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int s = (lane + 32 * e) / M;
            d16_e[e] = __shfl_sync(FULL, d16_s, s);
            deff_e[e] = __shfl_sync(FULL, deff_s, s);
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const double pre = __dadd_rn(round_half_away(__ddiv_rn(v[e], deff_e[e])), z);
        const double c = clip1(pre);
        code[e] = (int)c;
        clamp[e] = fabs(pre) > 1.0;
        rec[e] = __dmul_rn(d16_e[e], __dsub_rn(c, z));
    }
    __syncwarp();
}

// Per-warp pairwise sum of E-per-lane values through the scratch row.
template <int N>
__device__ __forceinline__ double row_sum(const double (&x)[N / 32], int lane, double* sm) {
    __syncwarp();
#pragma unroll
    for (int e = 0; e < N / 32; ++e) sm[lane + 32 * e] = x[e];
    __syncwarp();
    const double s = warp_pairwise_sum(sm, N, lane);
    __syncwarp();
    return s;
}

struct EvalPtrs {
    double *e_rot, *e_noro, *e_uni;                           // [nb*N] squared errors
    double *in_max, *rot_max, *a2, *err2, *noro2, *uni2, *slack;  // [nb]
    int *clamp_cnt, *zero_cnt;                                // [nb]
    int* nonfinite;  // set when a rotated grid value is inf/NaN (fwht_inverse raises, transform.py:36-42)
};

template <int N, typename TIn>
__global__ void __launch_bounds__(32 * kEvalWarps) eval_kernel(const TIn* __restrict__ w, int64_t numel, int64_t nb,
                                                               const uint8_t* __restrict__ payload, int ss, int policy,
                                                               double coeff, int symmetric, EvalPtrs o) {
    constexpr int E = N / 32;
    __shared__ double sm_all[kEvalWarps][N];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t blk = (int64_t)blockIdx.x * kEvalWarps + wid;
    if (blk >= nb) return;
    double* sm = sm_all[wid];
    const double norm = __ddiv_rn(1.0, __dsqrt_rn((double)N));

    double a[E], y[E], t[E], rec[E];
    int code[E];
    bool clamp[E];
    double in_max = 0.0, rot_max = 0.0, lo = INFINITY, hi = -INFINITY;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int64_t gi = blk * N + lane + 32 * e;
        a[e] = gi < numel ? (double)w[gi] : 0.0;  // zero tail pad (compute.py:136-143)
        y[e] = a[e];
        in_max = fmax(in_max, fabs(a[e]));
        lo = fmin(lo, a[e]);
        hi = fmax(hi, a[e]);
    }
    warp_butterfly<E>(y, lane);
#pragma unroll
    for (int e = 0; e < E; ++e) {
        y[e] = __dmul_rn(y[e], norm);
        rot_max = fmax(rot_max, fabs(y[e]));
    }
#pragma unroll
    for (int o2 = 16; o2; o2 >>= 1) {
        in_max = fmax(in_max, __shfl_xor_sync(FULL, in_max, o2));
        rot_max = fmax(rot_max, __shfl_xor_sync(FULL, rot_max, o2));
        lo = fmin(lo, __shfl_xor_sync(FULL, lo, o2));
        hi = fmax(hi, __shfl_xor_sync(FULL, hi, o2));
    }

    // ---- rotated codec: recon of the grid values (eval_error) or of the stored block (eval_container)
    double budget;
    if (payload == nullptr) {
        grid_quant<N>(y, lane, sm, ss, policy, coeff, symmetric, t, code, clamp, budget);
    } else {  // compute.py:294-308
        const uint8_t* p = payload + blk * block_nbytes(N, ss);
        const double z = trunc(f16_bits_to_f64(*reinterpret_cast<const uint16_t*>(p + 3 * N / 8 + 2)));
        double q8[8];
        if (ss) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const double dk = f16_bits_to_f64(*reinterpret_cast<const uint16_t*>(p + 3 * N / 8 + 4 + 2 * k));
                q8[k] = __dmul_rn(dk, dk);
            }
            budget = __ddiv_rn(__dmul_rn((double)(N / kSubBlocks), serial_pairwise_sum(q8, 8)), 4.0);
        } else {
            const double d = f16_bits_to_f64(*reinterpret_cast<const uint16_t*>(p + 3 * N / 8));
            budget = __ddiv_rn(__dmul_rn((double)N, __dmul_rn(d, d)), 4.0);
        }
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int j = lane + 32 * e;
            const uint32_t p0 = *reinterpret_cast<const uint32_t*>(p + 4 * e);
            const uint32_t p1 = *reinterpret_cast<const uint32_t*>(p + N / 8 + 4 * e);
            const int c = (int)((p0 >> lane) & 1u) + 2 * (int)((p1 >> lane) & 1u) - 1;  // plane 2 validated zero
            const uint16_t sb = ss ? *reinterpret_cast<const uint16_t*>(p + 3 * N / 8 + 4 + 2 * (j / (N / kSubBlocks)))
                                   : *reinterpret_cast<const uint16_t*>(p + 3 * N / 8);
            const double sc = f16_bits_to_f64(sb);
            const double cf = (double)c;
            const double pre = sc > 0.0 ? __dadd_rn(round_half_away(__ddiv_rn(y[e], sc)), z) : __dmul_rn(2.0, cf);
            code[e] = c;
            clamp[e] = fabs(pre) > 1.0;
            t[e] = __dmul_rn(sc, __dsub_rn(cf, z));
        }
    }
    bool bad = false;
#pragma unroll
    for (int e = 0; e < E; ++e) bad |= !isfinite(t[e]);
    if (__any_sync(FULL, bad) && lane == 0) *o.nonfinite = 1;
    warp_butterfly<E>(t, lane);  // fwht_inverse of the grid values
    int nclamp = 0, nzero = 0;
    double sq[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const double d = __dsub_rn(__dmul_rn(t[e], norm), a[e]);
        sq[e] = __dmul_rn(d, d);
        nclamp += clamp[e];
        nzero += code[e] == 0;
        o.e_rot[blk * N + lane + 32 * e] = sq[e];
    }
    const double err2 = row_sum<N>(sq, lane, sm);

    // ---- unrotated ternary baseline (compute.py:258 / :327)
    {
        double bdummy;
        grid_quant<N>(a, lane, sm, ss, policy, coeff, symmetric, rec, code, clamp, bdummy);
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const double d = __dsub_rn(rec[e], a[e]);
        sq[e] = __dmul_rn(d, d);
        o.e_noro[blk * N + lane + 32 * e] = sq[e];
    }
    const double noro2 = row_sum<N>(sq, lane, sm);

    // ---- uniform 3-bit baseline (compute.py:204-211)
    const bool ok = hi > lo;
    const double step = ok ? __ddiv_rn(__dsub_rn(hi, lo), 7.0) : 1.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        double r = a[e];
        if (ok) r = fmin(fmax(__dmul_rn(step, floor(__dadd_rn(__ddiv_rn(a[e], step), 0.5))), lo), hi);
        const double d = __dsub_rn(r, a[e]);
        sq[e] = __dmul_rn(d, d);
        o.e_uni[blk * N + lane + 32 * e] = sq[e];
    }
    const double uni2 = row_sum<N>(sq, lane, sm);
#pragma unroll
    for (int e = 0; e < E; ++e) sq[e] = __dmul_rn(a[e], a[e]);
    const double a2 = row_sum<N>(sq, lane, sm);

    nclamp = __reduce_add_sync(FULL, nclamp);
    nzero = __reduce_add_sync(FULL, nzero);
    if (lane == 0) {
        o.in_max[blk] = in_max;
        o.rot_max[blk] = rot_max;
        o.a2[blk] = a2;
        o.err2[blk] = err2;
        o.noro2[blk] = noro2;
        o.uni2[blk] = uni2;
        o.slack[blk] = nclamp ? INFINITY : __dsub_rn(budget, err2);
        o.clamp_cnt[blk] = nclamp;
        o.zero_cnt[blk] = nzero;
    }
}

// ------------------------------------------------------------------------------------------
// numpy add.reduce over a contiguous float64 vector, replayed exactly.
// The tree: n <= 128 is a leaf (n < 8 sequential, else 8 strided accumulators + tree + tail);
// larger n splits at n2 = n/2 rounded down to a multiple of 8.  Every node above depth D with
// n > 144*2^(D-1) is > 128 long and therefore splits, so the depth-D nodes can be summed
// independently (one thread each) and the top of the tree combined level by level.
// ------------------------------------------------------------------------------------------
constexpr int kPwMaxDepth = 14;
constexpr int kPwJobs = 6;

__device__ double pw_leaf(const double* v, int64_t n) {
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, v[i]);
        return r;
    }
    double r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = v[k];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], v[i + k]);
    }
    double s = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) s = __dadd_rn(s, v[i]);
    return s;
}

// The recursion with an explicit stack (depth <= 40 for any int64 length).
__device__ double pw_tree(const double* v, int64_t n) {
    int64_t fs[40], fm[40];
    double fl[40];
    int8_t st[40];
    int top = 0;
    fs[0] = 0;
    fm[0] = n;
    st[0] = 0;
    double val = 0.0;
    for (;;) {
        const int64_t s = fs[top], m = fm[top];
        if (st[top] == 0) {
            if (m <= 128) {
                val = pw_leaf(v + s, m);
            } else {
                const int64_t m2 = (m / 2) - (m / 2) % 8;
                st[top] = 1;
                ++top;
                fs[top] = s;
                fm[top] = m2;
                st[top] = 0;
                continue;
            }
        } else if (st[top] == 1) {
            const int64_t m2 = (m / 2) - (m / 2) % 8;
            fl[top] = val;
            st[top] = 2;
            ++top;
            fs[top] = s + m2;
            fm[top] = m - m2;
            st[top] = 0;
            continue;
        } else {
            val = __dadd_rn(fl[top], val);
        }
        if (top == 0) return val;
        --top;
    }
}

struct PwJobs {
    const double* v[kPwJobs];
    int64_t n[kPwJobs];
    int depth[kPwJobs];
    double* nodes;  // [kPwJobs][1 << kPwMaxDepth]
};

__host__ __device__ inline int pw_depth(int64_t n) {
    int d = 0;
    while (d < kPwMaxDepth && n > (int64_t)144 << d) ++d;  // all nodes above depth d+1 split
    return d;
}

__global__ void pw_nodes_kernel(PwJobs jobs) {
    const int j = blockIdx.y;
    const int D = jobs.depth[j];
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= ((int64_t)1 << D)) return;
    int64_t s = 0, m = jobs.n[j];
    for (int l = 0; l < D; ++l) {
        const int64_t m2 = (m / 2) - (m / 2) % 8;
        if ((k >> (D - 1 - l)) & 1) {
            s += m2;
            m -= m2;
        } else {
            m = m2;
        }
    }
    jobs.nodes[(int64_t)j * (1 << kPwMaxDepth) + k] = pw_tree(jobs.v[j] + s, m);
}

// Combine the depth-D node sums (left + right, bottom-up) and finish the report.
// report: mse, frobenius_rel, linf_in, linf_rot, bound_slack, clamp_fraction, zero_fraction,
//         mse_uniform3, mse_ternary_noro, n_blocks, unclamped_blocks (compute.py:256-269),
//         nonfinite flag (the reference raises DomainError from fwht_inverse).
constexpr int kFinThreads = 1024;

__global__ void __launch_bounds__(kFinThreads) eval_finish_kernel(PwJobs jobs, int64_t numel, int64_t nb, int N,
                                                                  const double* slack, const int* clamp_cnt,
                                                                  const int* zero_cnt, const int* nonfinite,
                                                                  double* report) {
    extern __shared__ double tree[];
    __shared__ double total[kPwJobs];
    __shared__ double red_min[kFinThreads / 32];
    __shared__ long long red_c[kFinThreads / 32], red_z[kFinThreads / 32], red_u[kFinThreads / 32];
    const int tid = threadIdx.x;
    for (int j = 0; j < kPwJobs; ++j) {
        const int D = jobs.depth[j];
        const double* nodes = jobs.nodes + (int64_t)j * (1 << kPwMaxDepth);
        for (int i = tid; i < (1 << D); i += kFinThreads) tree[i] = nodes[i];
        __syncthreads();
        for (int l = D; l > 0; --l) {
            const int cnt = 1 << (l - 1);
            double tmp[(1 << kPwMaxDepth) / 2 / kFinThreads];
#pragma unroll
            for (int r = 0; r < (1 << kPwMaxDepth) / 2 / kFinThreads; ++r) {
                const int i = tid + r * kFinThreads;
                if (i < cnt) tmp[r] = __dadd_rn(tree[2 * i], tree[2 * i + 1]);
            }
            __syncthreads();
#pragma unroll
            for (int r = 0; r < (1 << kPwMaxDepth) / 2 / kFinThreads; ++r) {
                const int i = tid + r * kFinThreads;
                if (i < cnt) tree[i] = tmp[r];
            }
            __syncthreads();
        }
        if (tid == 0) total[j] = __dadd_rn(0.0, tree[0]);  // add.reduce starts from the identity
        __syncthreads();
    }
    double mn = INFINITY;
    long long nc = 0, nz = 0, nu = 0;
    for (int64_t b = tid; b < nb; b += kFinThreads) {
        const int c = clamp_cnt[b];
        nc += c;
        nz += zero_cnt[b];
        if (c == 0) {
            ++nu;
            mn = fmin(mn, slack[b]);
        }
    }
    for (int o = 16; o; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(FULL, mn, o));
        nc += __shfl_xor_sync(FULL, nc, o);
        nz += __shfl_xor_sync(FULL, nz, o);
        nu += __shfl_xor_sync(FULL, nu, o);
    }
    if ((tid & 31) == 0) {
        red_min[tid >> 5] = mn;
        red_c[tid >> 5] = nc;
        red_z[tid >> 5] = nz;
        red_u[tid >> 5] = nu;
    }
    __syncthreads();
    if (tid == 0) {
        for (int i = 1; i < kFinThreads / 32; ++i) {
            mn = fmin(mn, red_min[i]);
            nc += red_c[i];
            nz += red_z[i];
            nu += red_u[i];
        }
        const double size = (double)numel, total_elems = (double)(nb * N);
        const double s_rot = total[0], s_a2 = total[5];
        report[0] = __ddiv_rn(s_rot, size);
        report[1] = s_a2 > 0.0 ? __ddiv_rn(__dsqrt_rn(s_rot), __dsqrt_rn(s_a2)) : 0.0;
        report[2] = __ddiv_rn(total[3], (double)nb);
        report[3] = __ddiv_rn(total[4], (double)nb);
        report[4] = nu ? mn : 0.0;
        report[5] = __ddiv_rn((double)nc, total_elems);
        report[6] = __ddiv_rn((double)nz, total_elems);
        report[7] = __ddiv_rn(total[2], size);
        report[8] = __ddiv_rn(total[1], size);
        report[9] = (double)nb;
        report[10] = (double)nu;
        report[11] = (double)*nonfinite;
    }
}

// ---- workspace layout ----------------------------------------------------------------------
struct EvalLayout {
    size_t off[ITQ3_EVAL_NFIELDS];
    size_t total;
};

static EvalLayout eval_layout(int64_t nb, int n) {
    EvalLayout L;
    size_t o = 0;
    auto take = [&](int f, size_t bytes) {
        L.off[f] = o;
        o += (bytes + 255) & ~(size_t)255;
    };
    const size_t flat = (size_t)nb * n * sizeof(double), per = (size_t)nb * sizeof(double);
    take(ITQ3_EVAL_E_ROT, flat);
    take(ITQ3_EVAL_E_NORO, flat);
    take(ITQ3_EVAL_E_UNI, flat);
    take(ITQ3_EVAL_IN_MAX, per);
    take(ITQ3_EVAL_ROT_MAX, per);
    take(ITQ3_EVAL_A2, per);
    take(ITQ3_EVAL_ERR2, per);
    take(ITQ3_EVAL_NORO2, per);
    take(ITQ3_EVAL_UNI2, per);
    take(ITQ3_EVAL_SLACK, per);
    take(ITQ3_EVAL_CLAMP, (size_t)nb * sizeof(int));
    take(ITQ3_EVAL_ZERO, (size_t)nb * sizeof(int));
    take(ITQ3_EVAL_FLAG, sizeof(int));
    take(ITQ3_EVAL_NODES, (size_t)kPwJobs * (1 << kPwMaxDepth) * sizeof(double));
    L.total = o;
    return L;
}

}  // namespace itq3

using namespace itq3;

extern "C" size_t itq3_eval_ws_nbytes(int64_t n_blocks, int block_n) {
    return eval_layout(n_blocks, block_n).total;
}

extern "C" int64_t itq3_eval_ws_offset(int64_t n_blocks, int block_n, int field) {
    if (field < 0 || field >= ITQ3_EVAL_NFIELDS) return -1;
    return (int64_t)eval_layout(n_blocks, block_n).off[field];
}

template <typename TIn>
static void launch_eval(const TIn* w, int64_t numel, int n, int64_t nb, const uint8_t* payload, int ss, int policy,
                        double coeff, int sym, const EvalPtrs& o, cudaStream_t s) {
    const dim3 grid((unsigned)((nb + kEvalWarps - 1) / kEvalWarps)), block(32 * kEvalWarps);
#define ITQ3_EVAL_CASE(NN) \
    case NN: eval_kernel<NN, TIn><<<grid, block, 0, s>>>(w, numel, nb, payload, ss, policy, coeff, sym, o); break;
    switch (n) {
        ITQ3_EVAL_CASE(32)
        ITQ3_EVAL_CASE(64)
        ITQ3_EVAL_CASE(128)
        ITQ3_EVAL_CASE(256)
        ITQ3_EVAL_CASE(512)
    }
#undef ITQ3_EVAL_CASE
}

extern "C" int itq3_eval(const void* w, int w_dtype, int64_t numel, int block_n, int sub_scales, int policy,
                         double coeff, int symmetric, const uint8_t* payload, void* workspace, double* d_report,
                         void* stream) {
    if (!valid_block_n(block_n)) {
        set_error("eval_error: block_n must be one of (32, 64, 128, 256, 512), got %d", block_n);
        return ITQ3_E_DOMAIN;
    }
    if (numel <= 0) {
        set_error("eval_error: expected a non-empty 2-D matrix");
        return ITQ3_E_SHAPE;
    }
    if (policy < 0 || policy > 2 || !(coeff > 0.0)) {
        set_error("eval_error: bad scale policy %d / coefficient %g", policy, coeff);
        return ITQ3_E_DOMAIN;
    }
    if (w_dtype != ITQ3_F32 && w_dtype != ITQ3_F64) {
        set_error("eval_error: weights must be float32 or float64");
        return ITQ3_E_DOMAIN;
    }
    const int64_t nb = (numel + block_n - 1) / block_n;
    const EvalLayout L = eval_layout(nb, block_n);
    char* ws = (char*)workspace;
    auto dp = [&](int f) { return (double*)(ws + L.off[f]); };
    EvalPtrs o{dp(ITQ3_EVAL_E_ROT), dp(ITQ3_EVAL_E_NORO), dp(ITQ3_EVAL_E_UNI), dp(ITQ3_EVAL_IN_MAX),
               dp(ITQ3_EVAL_ROT_MAX), dp(ITQ3_EVAL_A2), dp(ITQ3_EVAL_ERR2), dp(ITQ3_EVAL_NORO2),
               dp(ITQ3_EVAL_UNI2), dp(ITQ3_EVAL_SLACK), (int*)(ws + L.off[ITQ3_EVAL_CLAMP]),
               (int*)(ws + L.off[ITQ3_EVAL_ZERO]), (int*)(ws + L.off[ITQ3_EVAL_FLAG])};
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMemsetAsync(o.nonfinite, 0, sizeof(int), s) != cudaSuccess) return check_launch("itq3_eval(memset)");
    if (w_dtype == ITQ3_F32)
        launch_eval((const float*)w, numel, block_n, nb, payload, sub_scales, policy, coeff, symmetric, o, s);
    else
        launch_eval((const double*)w, numel, block_n, nb, payload, sub_scales, policy, coeff, symmetric, o, s);
    int rc = check_launch("itq3_eval");
    if (rc) return rc;
    // reductions: e_rot, e_noro, e_uni over the unpadded size; in_max, rot_max, a2 over blocks
    PwJobs jobs;
    const double* srcs[kPwJobs] = {o.e_rot, o.e_noro, o.e_uni, o.in_max, o.rot_max, o.a2};
    const int64_t lens[kPwJobs] = {numel, numel, numel, nb, nb, nb};
    int maxd = 0;
    for (int j = 0; j < kPwJobs; ++j) {
        jobs.v[j] = srcs[j];
        jobs.n[j] = lens[j];
        jobs.depth[j] = pw_depth(lens[j]);
        maxd = jobs.depth[j] > maxd ? jobs.depth[j] : maxd;
    }
    jobs.nodes = dp(ITQ3_EVAL_NODES);
    const int nodes = 1 << maxd;
    pw_nodes_kernel<<<dim3((unsigned)((nodes + 127) / 128), kPwJobs), 128, 0, s>>>(jobs);
    rc = check_launch("itq3_eval(pairwise)");
    if (rc) return rc;
    const size_t smem = (size_t)(1 << kPwMaxDepth) * sizeof(double);
    static std::atomic<unsigned long long> attr{0};
    if (int rc2 = ensure_smem_attr(eval_finish_kernel, (int)smem, attr, "itq3_eval: smem attribute")) return rc2;
    eval_finish_kernel<<<1, kFinThreads, smem, s>>>(jobs, numel, nb, block_n, o.slack, o.clamp_cnt, o.zero_cnt,
                                                    o.nonfinite, d_report);
    return check_launch("itq3_eval(finish)");
}
