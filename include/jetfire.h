/*
 * jetfire.h — C ABI of libjetfire.so, the B200 (sm_100a) INT8 data-flow hot path.
 *
 * Each entry point replaces one function of the reference's Python module
 * `int8flow` (arXiv 2403.12422 CPU reference, /root/reference/pkg/src/int8flow);
 * the reference interface it stands in for is cited beside it.
 *
 * Conventions (all entry points):
 *   - every pointer is a DEVICE pointer to row-major, contiguous memory
 *     (unless a leading dimension argument says otherwise);
 *   - a BlockQuantTensor [n x c] is two buffers: int8 codes q[n*c] in
 *     [-127,127] and float32 scales s[(n/32)*(c/32)], every scale on the
 *     binary16 grid (qtensor.py:73-105).  The block size is fixed at 32;
 *   - `stream` is a cudaStream_t; every kernel is enqueued on it, nothing
 *     synchronizes, nothing allocates device memory;
 *   - the return value is a host-side status: 0 = enqueued, nonzero = shape /
 *     argument / launch error (message via jf_last_error());
 *   - data-dependent errors (non-finite input, binary16 scale overflow) are
 *     reported asynchronously by OR-ing JF_EFLAG_* bits into *err (a device
 *     int32 the caller zeroes); the host checks it when it synchronizes and
 *     raises the reference's ValueError texts (qtensor.py:189,210).
 *   - dimension arguments are int64; all of n, c, d, k must be multiples of 32.
 */
#ifndef JETFIRE_H_
#define JETFIRE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *jf_stream_t; /* == cudaStream_t */

#define JF_OK 0
#define JF_ERR_ARG 1
#define JF_ERR_LAUNCH 2
#define JF_ERR_UNSUPPORTED 3

#define JF_EFLAG_NONFINITE 1 /* "input contains non-finite values" */
#define JF_EFLAG_OVERFLOW 2  /* "scale overflows the binary16 range" */

/* GEMM promotion modes (qgemm.py:183-229). */
#define JF_MODE_EXACT 0 /* acc = fl(acc + fl(fl(P*sa)*sb)): bit-exact with the reference */
#define JF_MODE_FAST 1  /* acc = fma(P, sa*sb, acc) (sa*sb exact): one rounding per chunk instead of three */

/* GEMM output kinds (qgemm.py:266-279). */
#define JF_OUT_INT8 0     /* requantized codes + scales (quantize=True) */
#define JF_OUT_F32 1      /* raw FP32 accumulator (+bias) (quantize=False) */
#define JF_OUT_INT8_DEQ 2 /* codes + scales AND their dequantized FP32 (QuantLinear dW path) */

int jf_version(void);
const char *jf_last_error(void);
int jf_sm_count(void);

/* K1 — quantize_per_block(x, 32)  [qtensor.py:219-246]
 * x: [n x c] float32 (or bfloat16 bits) with row stride ldx elements. */
int jf_quantize_f32(const float *x, int64_t n, int64_t c, int64_t ldx, int8_t *q, float *s,
                    int32_t *err, jf_stream_t stream);
int jf_quantize_bf16(const uint16_t *x, int64_t n, int64_t c, int64_t ldx, int8_t *q, float *s,
                     int32_t *err, jf_stream_t stream);

/* K2 — dequantize(xq)  [qtensor.py:249-255]; exact.  y: [n x c] float32 / bfloat16 bits. */
int jf_dequantize_f32(const int8_t *q, const float *s, int64_t n, int64_t c, float *y,
                      jf_stream_t stream);
int jf_dequantize_bf16(const int8_t *q, const float *s, int64_t n, int64_t c, uint16_t *y,
                       jf_stream_t stream);

/* Fused INT8-boundary attention (AttentionCore, qlayers.py:187-236, with the block's
 * dequantize/quantize crossings qlayers.py:350-351 and :406-408 done inside the kernels).
 * Causal, softmax scale 1/sqrt(head_dim); tcgen05 MMAs on bf16 operands (codes
 * dequantized exactly, then rounded to bf16), FP32 accumulation; tolerance class.
 * jf_attn_supported: 1 when seq % 256 == 0 and head_dim is 64 or 128.
 * jf_attn_fwd_q: QKV codes/scales [n x 3c] (n = batch*seq, c = heads*head_dim) ->
 *   O codes/scales [n x c]; also o_bf (bf16 O [n x c], for the backward's D_i) and
 *   lse [batch, heads, seq] (log2 domain).
 * jf_attn_bwd_q: + dO codes/scales [n x c] -> dQ|dK|dV codes/scales [n x 3c];
 *   dsum [batch, heads, seq] is scratch (D_i = rowsum(dO * O)).  Two kernels, no
 *   atomics: deterministic. */
int jf_attn_supported(int64_t seq, int64_t head_dim);
int jf_attn_fwd_q(const int8_t *qkv, const float *qkv_s, int64_t batch, int64_t seq, int64_t heads,
                  int64_t head_dim, int8_t *o, float *o_s, uint16_t *o_bf, float *lse, int32_t *err,
                  jf_stream_t stream);
int jf_attn_bwd_q(const int8_t *qkv, const float *qkv_s, const int8_t *dout, const float *dout_s,
                  const uint16_t *o_bf, const float *lse, float *dsum, int64_t batch, int64_t seq,
                  int64_t heads, int64_t head_dim, int8_t *dqkv, float *dqkv_s, int32_t *err,
                  jf_stream_t stream);
/* diagnostics: MN-major UMMA descriptor strides (lbo, sbo) and a device buffer for CTA-0
 * event clocks (long long[16*64]) of the attention kernels (null = off). */
int jf_attn_set_mn_desc(uint32_t lbo, uint32_t sbo);
int jf_attn_set_trace(long long *buf);

/* The attention boundary (qlayers.py:350-351 forward, :406-408 backward).
 * jf_dequantize_qkv_heads: QKV codes [n x 3c] (n = batch*seq, c = heads*head_dim) -> q, k, v
 *   bf16, each contiguous [batch, heads, seq, head_dim] (head_dim % 16 == 0).
 * jf_quantize_heads_bf16: bf16 x[batch, seq, heads, head_dim] with element strides
 *   (sb, ss, sh, 1) -> codes/scales of an [n x c] block tensor written into a column slice:
 *   q (row stride ldq bytes) and s (row stride lds floats) point at the slice. */
int jf_dequantize_qkv_heads(const int8_t *q, const float *s, int64_t batch, int64_t seq, int64_t heads,
                            int64_t head_dim, uint16_t *yq, uint16_t *yk, uint16_t *yv, jf_stream_t stream);
int jf_quantize_heads_bf16(const uint16_t *x, int64_t batch, int64_t seq, int64_t heads, int64_t head_dim,
                           int64_t sb, int64_t ss, int64_t sh, int8_t *q, int64_t ldq, float *s, int64_t lds,
                           int32_t *err, jf_stream_t stream);

/* BlockQuantTensor.transposed()  [qtensor.py:130-136]: qt [c x n], st [c/32 x n/32]. */
int jf_transpose(const int8_t *q, const float *s, int64_t n, int64_t c, int8_t *qt, float *st,
                 jf_stream_t stream);

/* K3 — block_mm_forward  [qgemm.py:282-309]:  Y[n x d] = X[n x c] . W[d x c]^T (+ bias[d]). */
int jf_gemm_fwd(const int8_t *x, const float *xs, const int8_t *w, const float *ws,
                const float *bias, int64_t n, int64_t c, int64_t d, int32_t mode,
                int32_t out_kind, int8_t *yq, float *ys, float *yf, int32_t *err,
                jf_stream_t stream);

/* K4 — block_mm_grad_input  [qgemm.py:312-333]:  dX[n x c] = dY[n x d] . W[d x c].
 * wt/wts: optional W^T codes [c x d] and scales [c/32 x d/32] (NULL: W is transposed
 * internally into `scratch`, which must then hold c*d bytes, and W's grid is read strided). */
int jf_gemm_dgrad(const int8_t *dy, const float *dys, const int8_t *w, const float *ws,
                  const int8_t *wt, const float *wts, int64_t n, int64_t d, int64_t c,
                  int32_t mode, int32_t out_kind, int8_t *dxq, float *dxs, float *dxf,
                  void *scratch, int32_t *err, jf_stream_t stream);

/* K5 — block_mm_grad_weight  [qgemm.py:336-357]:  dW[d x c] = dY[n x d]^T . X[n x c].
 * dyt/dyts, xt/xts: optional transposed tensors dY^T [d x n] and X^T [c x n] (codes + scale
 * grids; NULL: codes transposed internally into `scratch` (n*d + n*c bytes), grids read strided). */
int jf_gemm_wgrad(const int8_t *dy, const float *dys, const int8_t *x, const float *xs,
                  const int8_t *dyt, const float *dyts, const int8_t *xt, const float *xts,
                  int64_t n, int64_t d, int64_t c, int32_t mode, int32_t out_kind, int8_t *dwq,
                  float *dws, float *dwf, void *scratch, int32_t *err, jf_stream_t stream);

/* f16-widened operand path (same products as K3-K5, bit-identical; B200 design choice,
 * no reference counterpart).  The int8 codes widened to f16 (exact) let the tcgen05
 * kind::f16 MMA accumulate the per-chunk integer partials in f32 directly, so the
 * promotion skips the int32->fp32 conversion that bounds the int8 kernels.
 * jf_widen_codes: y = f16(x) [rows x cols], or f16(x)^T [cols x rows] when transpose != 0
 * (rows, cols multiples of 64).  Used for the weights (cached per update) and activations. */
int jf_widen_codes(const int8_t *x, int64_t rows, int64_t cols, uint16_t *y, int32_t transpose,
                   jf_stream_t stream);

/* Y[m x n] = A[m x k] . B[n x k]^T, A and B f16-widened codes, both K-major; sa / sb the
 * per-32x32 scale grids of A [m/32 x k/32] and B [n/32 x k/32] with element strides
 * (s0, s1) (contiguous along one axis).  m, n, k multiples of 128.  Output kinds,
 * promotion and requantization as jf_gemm_fwd. */
int jf_gemm_f16(const uint16_t *a, const float *sa, int64_t sa_s0, int64_t sa_s1, const uint16_t *b,
                const float *sb, int64_t sb_s0, int64_t sb_s1, const float *bias, int64_t m, int64_t n,
                int64_t k, int32_t mode, int32_t out_kind, int8_t *yq, float *ys, float *yf,
                int32_t *err, jf_stream_t stream);

/* Scratch bytes jf_gemm_dgrad / jf_gemm_wgrad need for the given shape. */
size_t jf_gemm_scratch_bytes(int32_t which /*1=dgrad,2=wgrad*/, int64_t n, int64_t d, int64_t c);

/* Debug: exact int32 partial sums of K chunk `kblk`: P = A[:, 32k:32k+32] . B[32k:32k+32, :]
 * for A [m x k] codes and B given as Bt [n x k] codes (both K-major).  Computed by the same
 * tcgen05 kind::i8 MMA as the GEMMs (micro_mm_16, qgemm.py:168-180). */
int jf_gemm_partials(const int8_t *a, const int8_t *bt, int64_t m, int64_t n, int64_t k,
                     int64_t kblk, int32_t *p, jf_stream_t stream);

/* Diagnostics: GEMM launch options for A/B experiments ("cols" 32|64 columns per promotion
 * warp; "pipe" 0|1 software-pipelined TMEM loads; "tma_scales" 0 forces the generic kernel).
 * Defaults are the measured best; results are bit-identical across options. */
int jf_gemm_set_option(const char *key, int value);

/* K6 — add_forward(x1q, x2q, width)  [qnonlinear.py:246-267] + RowStats [:103-144].
 * b/bs may be NULL: the second operand is zeros_like(a) (qtensor.py:258-264).
 * mean/sumsq: [n x c/width] float32. */
int jf_add_stats(const int8_t *a, const float *as, const int8_t *b, const float *bs, int64_t n,
                 int64_t c, int64_t width, int8_t *yq, float *ys, float *mean, float *sumsq,
                 int32_t *err, jf_stream_t stream);

/* K7 — layernorm_forward  [qnonlinear.py:300-330]; writes mu/inv_std [n] (LayerNormContext). */
int jf_ln_fwd(const int8_t *x, const float *xs, const float *mean, const float *sumsq,
              int64_t n, int64_t c, int64_t width, const float *gamma, const float *beta,
              float eps, int8_t *yq, float *ys, float *mu, float *inv_std, int32_t *err,
              jf_stream_t stream);

/* K8 — layernorm_backward  [qnonlinear.py:333-355]; dgamma/dbeta [c] float32.
 * workspace: >= jf_ln_bwd_workspace_bytes(n, c) bytes. */
int jf_ln_bwd(const int8_t *x, const float *xs, const float *mu, const float *inv_std,
              const int8_t *dy, const float *dys, const float *gamma, int64_t n, int64_t c,
              int8_t *dxq, float *dxs, float *dgamma, float *dbeta, void *workspace,
              int32_t *err, jf_stream_t stream);
size_t jf_ln_bwd_workspace_bytes(int64_t n, int64_t c);

/* K9 / K10 — gelu_forward / gelu_backward  [qnonlinear.py:150-175].
 * tables: optional (NULL: per-tile tables) lookup tables built once by
 * jf_gelu_build_tables into a caller buffer of jf_gelu_tables_bytes() bytes:
 * f(code * s) for every positive binary16 scale s and code in [-127, 127]. */
size_t jf_gelu_tables_bytes(void);
int jf_gelu_build_tables(float *tables, jf_stream_t stream);
int jf_gelu_fwd(const int8_t *x, const float *xs, int64_t n, int64_t c, int8_t *yq, float *ys,
                const float *tables, int32_t *err, jf_stream_t stream);
int jf_gelu_bwd(const int8_t *x, const float *xs, const int8_t *dy, const float *dys, int64_t n,
                int64_t c, int8_t *dxq, float *dxs, const float *tables, int32_t *err,
                jf_stream_t stream);

/* K11 — dbias = dequantize(dY).sum(axis=0)  [qlayers.py:180]; out [c] float32.
 * workspace: >= jf_colsum_workspace_bytes(n, c) bytes. */
int jf_colsum(const int8_t *q, const float *s, int64_t n, int64_t c, float *out,
              void *workspace, jf_stream_t stream);
size_t jf_colsum_workspace_bytes(int64_t n, int64_t c);

/* Loss head (model step, trainer.py:387-406): softmax cross-entropy of bf16 logits [n x ld]
 * (columns v..ld are padding and get zero gradient; padded logits should be -inf).
 * row_loss[r] = -mask_r * log_softmax(logits)[r, y_r] / n_live; dlogits (bf16 [n x ld]) =
 * (softmax - onehot(y)) * mask_r / n_live.  mask may be NULL; n_live is a device scalar. */
int jf_cross_entropy_bf16(const uint16_t *logits, int64_t n, int64_t v, int64_t ld, const int64_t *y,
                          const float *mask, const float *n_live, float *row_loss, uint16_t *dlogits,
                          jf_stream_t stream);

/* AdamW step (trainer.py:247-262) in the reference's float32 operation order; lr, eps, wd,
 * bc1 = 1 - b1^t, bc2 = 1 - b2^t are the float32 roundings of the Python floats, b1 and b2 the
 * doubles themselves (the reference forms 1 - b1 in float64) (wd = 0: no decay).
 * jf_adamw: flat update of count elements of p, m, v (in place).
 * jf_adamw_quantize: same for a [n x c] matrix, then quantize_per_block(p) -> q, s
 *   (the INT8 weight copy, qlayers.py:139-143) in the same pass. */
int jf_adamw(float *p, const float *g, float *m, float *v, int64_t count, float lr, double b1, double b2,
             float eps, float wd, float bc1, float bc2, jf_stream_t stream);
int jf_adamw_quantize(float *p, const float *g, float *m, float *v, int64_t n, int64_t c, float lr, double b1,
                      double b2, float eps, float wd, float bc1, float bc2, int8_t *q, float *s, int32_t *err,
                      jf_stream_t stream);

/* AdamW over many small FP32 tensors in one launch (same per-element arithmetic as
 * jf_adamw).  `tensors`: device array of {float *p; const float *g; float *m; float *v;
 * int64 count; float wd; int32 pad} (48 bytes each); chunk c covers elements
 * [chunk_start[c], chunk_start[c] + chunk_len) of tensor chunk_tensor[c]. */
/* jf_adamw_quantize_multi: jf_adamw_quantize over several [n x c] matrices in one launch.
 * `tensors`: device array of {float *p; const float *g; float *m; float *v; int8_t *q;
 * float *s; int64 n, c; float wd; int32 pad; int64 tile_start} (80 bytes each), tile_start =
 * the matrix's first 32x256 tile in a running count (ascending); total_tiles = the sum. */
int jf_adamw_quantize_multi(const void *tensors, int32_t ntensors, int64_t total_tiles, float lr, double b1,
                            double b2, float eps, float bc1, float bc2, int32_t *err, jf_stream_t stream);
int jf_adamw_multi(const void *tensors, const int32_t *chunk_tensor, const int64_t *chunk_start,
                   int32_t nchunks, int64_t chunk_len, float lr, double b1, double b2, float eps,
                   float bc1, float bc2, jf_stream_t stream);

/* Dropout by scale folding  [qnonlinear.py:207-240]: codes zeroed where keep[i]==0,
 * scales snapped f16(s * keep_factor).  keep: [n x c] uint8 (the materialized mask). */
/* DropoutState.generate's keep mask  [qnonlinear.py:190-200]: keep[i] = (numpy
 * Generator(Philox(key=(key0, key1))).random() of element i) >= p, bit-identical to numpy
 * (Philox4x64-10, 53-bit doubles); total = rows*cols elements, keep is uint8 0/1. */
int jf_philox_keep(uint64_t key0, uint64_t key1, double p, int64_t total, uint8_t *keep, jf_stream_t stream);
int jf_dropout(const int8_t *q, const float *s, const uint8_t *keep, float keep_factor,
               int64_t n, int64_t c, int8_t *oq, float *os, int32_t *err, jf_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* JETFIRE_H_ */
