/*
 * libitq3 -- C ABI of the B200-native ITQ3_S hot path.
 *
 * Plain pointers and sizes only (no torch / numpy types).  Every entry point
 *   * takes a cudaStream_t (passed as void*; NULL = legacy default stream),
 *   * is stream-ordered, does NO hidden host synchronisation and never frees
 *     or allocates caller memory (the caller owns every buffer),
 *   * returns ITQ3_OK or an ITQ3_E_* code whose classes mirror the reference's
 *     exception taxonomy (reference: pkg/src/itq3/errors.py:16-59); the detail
 *     string is available from itq3_last_error() on the calling thread.
 * Device-side data errors (corrupt planes, NaN scales) are reported through a
 * caller-owned device word written by itq3_validate, read back when the caller
 * synchronises -- the library itself never blocks.
 *
 * Payload = the container's block array exactly as write_container emits it
 * (codec.py:222-235): n_blocks x block_nbytes(block_n, ss) bytes, each block =
 * 3 bit planes (3n/8 B) | scale f16 LE | zero-point f16 LE [| 8 x sub-scale f16 LE].
 * "Tiled" = the device-resident GEMV/MMQ layout produced by itq3_repack_tiled
 * (2-bit codes in mma-fragment order, 66 B per 256 weights).
 */
#ifndef ITQ3_H
#define ITQ3_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum itq3_status {
    ITQ3_OK = 0,
    ITQ3_E_LENGTH = 1,      /* LengthError    errors.py:16-19 */
    ITQ3_E_DOMAIN = 2,      /* DomainError    errors.py:22-25 */
    ITQ3_E_SHAPE = 3,       /* ShapeError     errors.py:28-31 */
    ITQ3_E_CORRUPT = 4,     /* CorruptionError errors.py:34-37 */
    ITQ3_E_UNSUPPORTED = 8, /* layout has no kernel here (caller routes elsewhere) */
    ITQ3_E_CUDA = 16        /* launch / runtime failure */
};

enum itq3_dtype { ITQ3_F32 = 0, ITQ3_F64 = 1, ITQ3_BF16 = 2, ITQ3_F16 = 3 };

/* ScalePolicy.kind (quantizer.py:33-49) */
enum itq3_policy { ITQ3_POLICY_CONSTANT = 0, ITQ3_POLICY_ARGMIN = 1, ITQ3_POLICY_MEAN_ABS = 2 };

/* itq3_validate check mask bits and the error kinds packed in the first-bad key */
enum itq3_check {
    ITQ3_CHECK_PLANES = 1,    /* stored code > 2 (packing.py:80-83)            kind 0 */
    ITQ3_CHECK_SCALE_NAN = 2, /* scale is NaN (packing.py:185-186)             kind 1 */
    ITQ3_CHECK_ZP = 4,        /* zero-point not in {-1,0,1} (packing.py:187-189) kind 2 */
    ITQ3_CHECK_SUB_NAN = 8,   /* sub-scale NaN (packing.py:193-195)            kind 3 */
    ITQ3_CHECK_ZP_FINITE = 16 /* zero-point non-finite: int() would raise       kind 4 */
};

const char* itq3_version(void);
const char* itq3_last_error(void);
int itq3_sm_count(void);
/* fp32 copy (n % 4 == 0, 16-byte aligned pointers) by one small kernel; `src` / `dst` may be pinned host
 * memory (UVA-mapped): the e2e step's input copy inside its CUDA graph (no DMA memcpy node) */
int itq3_copy_f32(float* dst, const float* src, int64_t n, void* stream);

/* ---- K1 encoder: replaces quantize_tensor / encode_block (codec.py:113-189) ----
 * w: numel values (f32 or f64, row-major flattened); the tail of the last block
 * is zero-padded as codec.py:173-179 does.  Writes n_blocks*block_nbytes bytes.
 * Bit-exact with the reference (fp64, numpy pairwise summation order). */
int itq3_encode(const void* w, int w_dtype, int64_t numel, int block_n, int sub_scales, int policy,
                double coeff, int symmetric, uint8_t* payload, void* stream);

/* ---- K7 validation: replaces the per-block checks of deserialize_block /
 * unpack_ternary (packing.py:67-84,171-197).  *d_first_bad (device u64) must be
 * preset to UINT64_MAX; receives min over offenders of
 * (block << 16) | (kind << 10) | index. */
int itq3_validate(const uint8_t* payload, int64_t n_blocks, int block_n, int sub_scales, uint32_t check_mask,
                  unsigned long long* d_first_bad, void* stream);

/* ---- K2 dequantiser: replaces dequantize_tensor / decode_block (codec.py:152-202).
 * out: numel values (F64 = bit-exact with the reference, F32 = exact value cast). */
int itq3_dequant(const uint8_t* payload, int64_t n_blocks, int block_n, int sub_scales, int64_t numel, void* out,
                 int out_dtype, void* stream);
/* diagnostics: device buffer of 16 u64 counters per CTA (cycle accounting of the tensor-core
 * dequantiser used for block_n 256 / variant s; tools/dequant_trace.py), or NULL to switch it off. */
int itq3_dequant_set_trace(void* buf);

/* ---- block utilities of the reference API (quantizer.py:78-197), float64 device data flow:
 * block_stats writes {n, mean, sigma, l1, linf, excess_kurtosis} (numpy pairwise sums; the
 * kurtosis' fourth powers are rounded once, numpy uses libm pow); ternary_quantize
 * clip(round_half_away(x / d) + z, -1, 1) -> int8; ternary_dequantize d * (code - z);
 * uniform_quantize clip(delta * floor(x / delta + 0.5), wmin, wmax). */
int itq3_block_stats(const double* v, int64_t n, double* out6, void* stream);
int itq3_ternary_quantize(const double* x, int64_t n, double d, int z, int8_t* codes, void* stream);
int itq3_ternary_dequantize(const int8_t* codes, int64_t n, double d, int z, double* out, void* stream);
int itq3_uniform_quantize(const double* x, int64_t n, double delta, double wmin, double wmax, double* out,
                          void* stream);

/* ---- decoder-stack glue (decoder.py; not on the ITQ3_S path): RoPE + KV append + grouped-query
 * split decode attention (head_dim 128, ctx <= 1024, position read from *pos); ws from
 * itq3_glue_attention_ws_nbytes, zero-initialised once. */
int64_t itq3_glue_attention_ws_nbytes(int n_heads);
int itq3_glue_rope_attention(const float* qkv, const float* cos_tab, const float* sin_tab, const int64_t* pos,
                             float* k_cache, float* v_cache, float* out, int n_heads, int n_kv, int head_dim, int ctx,
                             void* ws, void* stream);

/* ---- transform: fwht_forward / fwht_inverse (transform.py:61-96) on n_vec
 * contiguous vectors of length n (2..512, power of two), dtype F32 or F64,
 * bit-identical to numpy's butterfly order.  normalize=0 skips the 1/sqrt(n). */
int itq3_fwht(const void* in, void* out, int dtype, int64_t n_vec, int n, int normalize, void* stream);

/* ---- fast layout (block_n = 256, variant s, cols % 256 == 0) ---- */
int64_t itq3_tiled_nbytes(int64_t rows, int64_t cols, int asymmetric);
int itq3_repack_tiled(const uint8_t* payload, int64_t rows, int64_t cols, int asymmetric, uint8_t* tiled,
                      void* stream);

/* ---- K3 activation rotation: x'_b = H_256 x_b per 256-block of K, quantised to
 * `limbs` signed-byte limbs (fixed point, per (block, token) power-of-two scale)
 * in mma-fragment order.  x element (k, m) at x[k*stride_k + m*stride_m]. */
int64_t itq3_act_nbytes(int64_t cols, int64_t m, int limbs);
int itq3_rotate_act(const void* x, int x_dtype, int64_t cols, int64_t m, int64_t stride_k, int64_t stride_m,
                    int limbs, uint8_t* act, void* stream);

/* ---- K4 fused GEMV / small-M matmul (replaces fused_matvec / fused_matmul,
 * compute.py:98-133) on the tiled layout:  y[r, m] = sum_k w_hat[r, k] x[k, m].
 * y element (r, m) at y[r*stride_r + m*stride_m]; y_dtype F32 (fp32 accumulate)
 * or F64 (fp64 accumulate, parity mode). */
int itq3_gemv(const uint8_t* tiled, int64_t rows, int64_t cols, int asymmetric, const uint8_t* act, int64_t m,
              int limbs, void* y, int y_dtype, int64_t stride_r, int64_t stride_m, void* stream);

/* ---- K5 batched MMQ on tcgen05 tensor cores (csrc/mmq.cu): Y = w_hat @ X for M >= 16 tokens.
 * Weights: itq3_repack_mmq layout (2-bit codes, 66 B per 256 weights + padding to 128 rows);
 * activations: itq3_rotate_act_f16 (x'' = H x / 16 as f16, pre-swizzled token tiles of
 * itq3_mmq_block_n(m) tokens).  A = d*t is exact in f16; fp32 accumulation in TMEM.
 * flags (nbytes / repack / mmq): ITQ3_MMQ_ASYM (asymmetric zero-points) | ITQ3_MMQ_PER32 (records with a
 * scale and zero-point per 32-k group: variant ss -- t scaled by the stored per-32 sub-scale,
 * codec.py:134-161 -- or block_n != 256).  itq3_repack_mmq covers block_n 256 (ITQ3_MMQ_PER32 there
 * means variant ss); itq3_repack_mmq_n any block_n in {32..512} with cols % block_n == 0 (variant ss
 * needs block_n >= 256) and always writes PER32 records.  The matching activations come from
 * itq3_rotate_act_f16_n with the same block_n (x'' = H_n x / sqrt(n)). */
#define ITQ3_MMQ_ASYM 1
#define ITQ3_MMQ_PER32 2
int64_t itq3_mmq_nbytes(int64_t rows, int64_t cols, int flags);
int itq3_repack_mmq(const uint8_t* payload, int64_t rows, int64_t cols, int flags, uint8_t* out, void* stream);
int itq3_repack_mmq_n(const uint8_t* payload, int64_t rows, int64_t cols, int block_n, int variant_ss, int asymmetric,
                      uint8_t* out, void* stream);
int itq3_rotate_act_f16_n(const void* x, int x_dtype, int64_t cols, int64_t m, int64_t stride_k, int64_t stride_m,
                          int block_n, uint8_t* out, unsigned* nonfinite, void* stream);
int itq3_mmq_block_n(int64_t m);
int64_t itq3_mmq_act_nbytes(int64_t cols, int64_t m);
/* nonfinite (nullable device u32): OR-ed with 1 if any input element is not finite -- fused_matmul's
 * DomainError check without a separate pass over X; the caller zeroes it before and reads it after. */
int itq3_rotate_act_f16(const void* x, int x_dtype, int64_t cols, int64_t m, int64_t stride_k, int64_t stride_m,
                        uint8_t* out, unsigned* nonfinite, void* stream);
/* workspace: itq3_mmq_ws_nbytes(rows, cols, m) bytes (may be 0 -> pass NULL); with a workspace,
 * small problems are split along K across CTAs and reduced in fixed order (deterministic). */
int64_t itq3_mmq_ws_nbytes(int64_t rows, int64_t cols, int64_t m);
/* diagnostics: device buffer of 16 u64 counters per CTA (cycle accounting per warp role of the next
 * itq3_mmq launches; tools/mmq_trace.py), or NULL to switch the accounting off. */
int itq3_mmq_set_trace(void* buf);
int itq3_mmq(const uint8_t* mmq, int64_t rows, int64_t cols, int flags, const uint8_t* act, int64_t m, void* y,
             int y_dtype, int64_t stride_r, int64_t stride_m, void* workspace, void* stream);
/* Row-sharded MMQ with the output all-gather fused into the epilogue: this
 * rank's `rows` weight rows are output rows [row0, row0 + rows) of a stage whose full Y lives on every
 * rank; each finished row-half is written to all npeer copies (d_ypeers: device array of npeer
 * pointers, e.g. torch symmetric-memory peer addresses over NVLink, each a full rows_total x m
 * output with strides stride_r / stride_m) by one bulk copy per peer from the epilogue's staging row,
 * or by the split reduce kernels when the workspace (itq3_mmq_ws_nbytes, may be NULL) splits K.
 * The caller orders the peers' reads after every rank's launch (a symmetric-memory barrier). */
int itq3_mmq_peers(const uint8_t* mmq, int64_t rows, int64_t cols, int flags, const uint8_t* act, int64_t m,
                   const void* d_ypeers, int npeer, int64_t row0, int y_dtype, int64_t stride_r, int64_t stride_m,
                   void* workspace, void* stream);

/* ---- generic fused matmul for every other layout (any block_n, variant ss,
 * row-straddling blocks): fp64 exact decode + fp64 dot, deterministic block order.
 * X (cols x k) fp64 at X[c*stride_c + j*stride_j]; Y (rows x k) fp64 row-major.
 * workspace: itq3_generic_ws_nbytes(...) bytes. */
int64_t itq3_generic_ws_nbytes(int64_t rows, int64_t cols, int block_n, int64_t k);
int itq3_matmul_generic(const uint8_t* payload, int64_t rows, int64_t cols, int block_n, int sub_scales,
                        const double* X, int64_t k, int64_t stride_c, int64_t stride_j, double* Y, void* workspace,
                        void* stream);

/* ---- packing utilities: pack_ternary / unpack_ternary (packing.py:43-84) on n_rows rows
 * of n codes (n % 8 == 0, n <= 512).  *d_bad (device u64, preset UINT64_MAX) receives
 * (row << 16) | index of the first out-of-range code (pack) or
 * (row << 16) | (code << 12) | index of the first stored code > 2 (unpack). */
int itq3_pack_codes(const int8_t* codes, int64_t n_rows, int n, uint8_t* planes, unsigned long long* d_bad,
                    void* stream);
int itq3_unpack_codes(const uint8_t* planes, int64_t n_rows, int n, int8_t* codes, unsigned long long* d_bad,
                      void* stream);

/* ---- K5b small-batch MMQ on tcgen05.mma kind::i8 (0 < m <= 64 tokens): raw 2-bit codes as the
 * TMEM A operand, activations as two s8 limbs of a 16-bit fixed point per (token, block)
 * (itq3_rotate_act_i8), one s32 accumulator per block folded with the f16 scale in the epilogue.
 * Weights: itq3_repack_mmq8 (itq3_mmq8_nbytes bytes).  Workspace: itq3_mmq8_ws_nbytes (split-K). */
int itq3_mmq8_block_n(int64_t m);
int64_t itq3_mmq8_nbytes(int64_t rows, int64_t cols);
int itq3_repack_mmq8(const uint8_t* payload, int64_t rows, int64_t cols, int asymmetric, uint8_t* out, void* stream);
int64_t itq3_mmq8_act_nbytes(int64_t cols, int64_t m);
int itq3_rotate_act_i8(const void* x, int x_dtype, int64_t cols, int64_t m, int64_t stride_k, int64_t stride_m,
                       uint8_t* out, unsigned* nonfinite, void* stream);
int64_t itq3_mmq8_ws_nbytes(int64_t rows, int64_t cols, int64_t m);
int itq3_mmq8(const uint8_t* w, int64_t rows, int64_t cols, const uint8_t* act, int64_t m, void* y, int y_dtype,
              int64_t stride_r, int64_t stride_m, void* workspace, void* stream);

/* ---- persistent chain kernel: a dependent chain of fused GEMVs (decode step) in ONE
 * cooperative launch (csrc/chain.cu).  Stage i multiplies its tiled weights by the first
 * cols_i entries of stage i-1's output (stage 0: x0).  A stage with K > 16 blocks is split in
 * nch = ceil(cols/4096) K-chunks computed by different CTAs; its y buffer holds nch partial
 * rows-vectors of 64-bit tagged words ([nch][rows] u64: low = fp32 bits, high = step epoch,
 * zero-initialised once) that the consumer sums in fixed order.  The caller fills a host
 * descriptor array with itq3_chain_write_desc (itq3_chain_desc_nbytes() bytes/stage), copies
 * it to device memory and passes two device u32 words (zero-initialised once): the step epoch
 * and a check-in counter; the kernel advances the epoch itself at the end of each launch.  `out` receives the last stage's outputs.
 * A stage whose descriptor has a non-NULL `xin` reads that fp32 vector instead of the previous
 * stage's output (independent stages: pure weight streaming, used to measure the roofline).  d_trace (optional):
 * n_ctas*n_stages*4 u64 globaltimer stamps for profiling. */
int64_t itq3_chain_desc_nbytes(void);
int itq3_chain_act_block_bytes(int limbs);
int itq3_chain_smem_bytes(void);
int itq3_chain_write_desc(void* host_desc, int index, const uint8_t* tiled, void* y, const float* xin, int64_t rows,
                          int64_t cols, int asymmetric, int reserved);
/* Host-balanced work split of stage `index` (optional): d_work = device int32[grid], CTA c computes K-chunk
 * d_work[c] / Gc and the row tiles d_work[c] % Gc + j Gc (Gc = grid / ceil(cols / 4096)), -1 = idle; every
 * (chunk, first row tile) pair exactly once.  Outputs do not depend on the assignment. */
int itq3_chain_set_work(void* host_desc, int index, const int32_t* d_work);
/* Tensor-parallel stage (no single reference counterpart: the reference's TP path is the per-stage
 * matvec + all-gather of SURVEY.md C5).  This rank computes output rows [row0, row0 + rows) of a
 * yrows-row stage from its row shard `tiled`, and the reducer stores every tagged output word into
 * all npeer ranks' copies of y (d_peers: device array of npeer pointers, e.g. symmetric-memory peer
 * addresses over NVLink; peer p's copy sits at the same layout as `y`).  y holds
 * 2 x nch x yrows u64 words (epoch-parity double buffer), nch = ceil(cols / 4096).  All ranks launch
 * itq3_chain_run the same number of times; consumers and the final fold read the full yrows rows.
 * `asymmetric` (both write_desc calls) is a flag word: bit 0 = asymmetric zero-points, bit 1 = gated
 * input -- the stage reads SiLU(prev[i]) * prev[cols + i] from the previous stage's output (a
 * gate | up projection feeding a down projection); bit 2 = RMSNorm input (stage 0, cols <= 4096:
 * x0 * rsqrt(mean(x0^2) + 1e-5) * xin, `xin` carrying the gain); bit 3 = the final fold adds into
 * `out` (residual stream) instead of overwriting it.  Bits 1-3 need itq3_chain_run_gated. */
int itq3_chain_write_desc_tp(void* host_desc, int index, const uint8_t* tiled, void* y, int64_t rows, int64_t cols,
                             int asymmetric, int64_t row0, int64_t yrows, const void* d_peers, int npeer);
/* Decoder flags (itq3_chain_run_gated): bit 4 = an RMSNorm stage's input is x0 + the previous stage's
 * output; bit 5 (with bit 3) = the final fold adds stage 0's output first; bit 6 = the RMSNorm input
 * is (x0 + stage 0's output) + the previous stage's output; bit 7 = that stage also writes the input
 * it formed (the new residual stream) to the buffer set here. */
int itq3_chain_set_xout(void* host_desc, int index, void* xout);
/* decoder, single GPU: the tagged residual buffer (u64 words) a flag-4 / flag-8 stage reads instead of
 * the launch input x0; flag-64 / flag-32 stages name the o stage whose output they add in flag bits 16-31 */
int itq3_chain_set_xres(void* host_desc, int index, const void* xres);
/* decoder attention as chain stages (GATED launches): kind 256 = per (kv head, split) partials of RoPE +
 * KV append + grouped-query attention over the previous (qkv) stage's outputs, kind 512 = per-head
 * combine into the next stage's input; params = device struct of itq3_chain_attn_params_nbytes() bytes:
 * {float* k_cache; float* v_cache; const float* cos; const float* sin; const int64_t* pos;
 *  int n_heads, n_kv, ctx, splits} (head_dim 128, 4 query heads per kv head, ceil(ctx / splits) <= 64) */
int itq3_chain_write_desc_attn(void* host_desc, int index, int kind, const void* params, void* y, int64_t yrows);
int itq3_chain_attn_params_nbytes(void);
int itq3_chain_run(const void* d_desc, int n_stages, const float* x0, int limbs, unsigned* d_epoch, float* out,
                   int grid, void* d_trace, void* stream);
/* the same, for chains with gated stages (descriptor flag bit 1) */
int itq3_chain_run_gated(const void* d_desc, int n_stages, const float* x0, int limbs, unsigned* d_epoch, float* out,
                         int grid, void* d_trace, void* stream);
/* flags: bit 0 = gated chain (itq3_chain_run_gated), bit 1 = every weight stage symmetric (no zero-point tile
 * loop), bit 2 = single GPU (no tensor-parallel stage: no peer-store paths); the specialised instantiations
 * are faster, and a stage needing what was left out traps the launch.  Plain chains with bits 1 and 2 (flags 6)
 * pass H_16 y between stages: every stage but the last stores H_16 (fp32) of each full 16-row tile of its
 * tagged outputs (a partial last tile plain) and reads its input in that form (stage 0 transforms x0 itself);
 * `out` and the last stage's outputs are plain.  Flags 2 = the same kernel family with plain stage outputs. */
int itq3_chain_run_ex(const void* d_desc, int n_stages, const float* x0, int limbs, unsigned* d_epoch, float* out,
                      int grid, void* d_trace, void* stream, int flags);

/* ---- K8 evaluation harness: replaces eval_error / eval_container / rotation_benefit
 * (compute.py:221-356).  One call quantises (payload == NULL: eval_error with the given
 * policy) or reads the stored blocks (payload != NULL: eval_container; the payload must
 * have passed itq3_validate), computes both baselines (unrotated ternary, uniform 3-bit),
 * and writes the 11 ErrorReport fields as doubles to d_report, in the order
 * mse, frobenius_rel, linf_in, linf_rot, bound_slack, clamp_fraction, zero_fraction,
 * mse_uniform3, mse_ternary_noro, n_blocks, unclamped_blocks, plus a 12th word that is 1.0
 * when a rotated grid value was inf/NaN (binary16 scale overflow: the reference's fwht_inverse
 * raises DomainError, transform.py:36-42, and so must the caller).  Every field but
 * frobenius_rel (BLAS ddot order in the reference) is bit-exact.  workspace:
 * itq3_eval_ws_nbytes(n_blocks, block_n) bytes; its per-block fields stay readable after the
 * call at itq3_eval_ws_offset(...) (rotation_benefit takes the medians of ERR2/NORO2/UNI2). */
enum itq3_eval_field {
    ITQ3_EVAL_E_ROT = 0,   /* [nb*n] f64 squared error, rotated codec       */
    ITQ3_EVAL_E_NORO = 1,  /* [nb*n] f64 squared error, unrotated ternary   */
    ITQ3_EVAL_E_UNI = 2,   /* [nb*n] f64 squared error, uniform 3-bit       */
    ITQ3_EVAL_IN_MAX = 3,  /* [nb] f64 max |w| per block                    */
    ITQ3_EVAL_ROT_MAX = 4, /* [nb] f64 max |Hw| per block                   */
    ITQ3_EVAL_A2 = 5,      /* [nb] f64 sum w^2 per block                    */
    ITQ3_EVAL_ERR2 = 6,    /* [nb] f64 pairwise sum of E_ROT per block      */
    ITQ3_EVAL_NORO2 = 7,   /* [nb] f64 pairwise sum of E_NORO per block     */
    ITQ3_EVAL_UNI2 = 8,    /* [nb] f64 pairwise sum of E_UNI per block      */
    ITQ3_EVAL_SLACK = 9,   /* [nb] f64 budget - err2 (unclamped) or +inf    */
    ITQ3_EVAL_CLAMP = 10,  /* [nb] i32 clamped codes per block              */
    ITQ3_EVAL_ZERO = 11,   /* [nb] i32 zero codes per block                 */
    ITQ3_EVAL_NODES = 12,  /* reduction scratch                             */
    ITQ3_EVAL_FLAG = 13,   /* i32 non-finite rotated grid value seen        */
    ITQ3_EVAL_NFIELDS = 14
};
size_t itq3_eval_ws_nbytes(int64_t n_blocks, int block_n);
int64_t itq3_eval_ws_offset(int64_t n_blocks, int block_n, int field);
int itq3_eval(const void* w, int w_dtype, int64_t numel, int block_n, int sub_scales, int policy, double coeff,
              int symmetric, const uint8_t* payload, void* workspace, double* d_report, void* stream);

/* ---- scalar binary16 codec (host): encode_f16 / decode_f16 (packing.py:87-109) */
uint16_t itq3_f16_encode(double x);
double itq3_f16_decode(uint16_t bits);

#ifdef __cplusplus
}
#endif

#endif /* ITQ3_H */
