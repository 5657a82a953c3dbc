// ce.cu — the loss head's softmax cross-entropy, fused (model step, trainer.py:387-406).
//
// The reference computes, per token row r of the logits,
//   logp = log_softmax(logits);  loss = -sum_r mask_r * logp[r, y_r] / n_live
//   dlogits = (exp(logp) - onehot(y)) * mask_r / n_live
// (trainer.py:388-404).  With the BF16 head the logits arrive as bf16 [n x ld];
// (columns v..ld must hold -inf: the vocabulary padding), one CTA per row finds
// the row max and sum of exponentials, writes the row's loss term,
// and a third pass writes dlogits as bf16 — the operand the two head-gradient
// GEMMs consume — so no FP32 logits/probabilities ever reach HBM.  Padded
// vocabulary columns carry -inf logits and get exactly zero gradient.
#include "common.cuh"

namespace jf {

JF_DEV float bf16_to_f32(uint32_t h16) { return __uint_as_float(h16 << 16); }

JF_DEV float block_reduce(float v, bool is_max, float *sm) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float u = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmaxf(v, u) : v + u;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sm[warp] = v;
  __syncthreads();
  float r = sm[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) r = is_max ? fmaxf(r, sm[w]) : r + sm[w];
  __syncthreads();
  return r;
}

JF_DEV float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Three passes over the row (the 100 KB bf16 row stays in L1/L2 after the first):
// max, sum of 2^((x - max) log2 e), then dlogits = 2^(x log2 e - log2-sum-exp) - [col == y],
// scaled by mask / n_live, as bf16.  One FFMA + one ex2 per element per exp pass, no
// per-element branch (padding columns are -inf: 2^-inf = 0).
__global__ void __launch_bounds__(256) ce_bf16_kernel(const uint16_t *__restrict__ logits, int64_t v, int64_t ld,
                                                      const int64_t *__restrict__ y, const float *__restrict__ mask,
                                                      const float *__restrict__ n_live, float *row_loss,
                                                      uint16_t *dl) {
  __shared__ float sm[8];
  constexpr float kLog2e = 1.4426950408889634f;
  const int64_t row = blockIdx.x;
  const uint16_t *x = logits + row * ld;
  // pass 1: row max
  float m = -INFINITY;
  for (int64_t j = (int64_t)threadIdx.x * 8; j < ld; j += (int64_t)blockDim.x * 8) {
    const uint4 w = __ldg(reinterpret_cast<const uint4 *>(x + j));
    const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) m = fmaxf(m, fmaxf(bf16_to_f32(u[k] & 0xffffu), bf16_to_f32(u[k] >> 16)));
  }
  m = block_reduce(m, true, sm);
  const float mb = m * kLog2e;
  // pass 2: sum of exp
  float s0 = 0.f, s1 = 0.f;
  for (int64_t j = (int64_t)threadIdx.x * 8; j < ld; j += (int64_t)blockDim.x * 8) {
    const uint4 w = __ldg(reinterpret_cast<const uint4 *>(x + j));
    const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      s0 += ex2f(fmaf(bf16_to_f32(u[k] & 0xffffu), kLog2e, -mb));
      s1 += ex2f(fmaf(bf16_to_f32(u[k] >> 16), kLog2e, -mb));
    }
  }
  const float ssum = block_reduce(s0 + s1, false, sm);
  const float l2 = mb + __log2f(ssum);         // log2 of sum exp(x)
  const float lse = l2 * 0.6931471805599453f;  // natural-log LSE
  const float wgt = (mask ? mask[row] : 1.f) / *n_live;
  const int64_t t = y[row];
  if (threadIdx.x == 0) row_loss[row] = -(bf16_to_f32(x[t]) - lse) * wgt;
  // pass 3: dlogits = (softmax - onehot) * mask / n_live, bf16 (RNE)
  uint16_t *d = dl + row * ld;
  for (int64_t j = (int64_t)threadIdx.x * 8; j < ld; j += (int64_t)blockDim.x * 8) {
    uint32_t o[4];
    const uint4 w = __ldg(reinterpret_cast<const uint4 *>(x + j));
    const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float a = ex2f(fmaf(bf16_to_f32(u[k] & 0xffffu), kLog2e, -l2));
      float b = ex2f(fmaf(bf16_to_f32(u[k] >> 16), kLog2e, -l2));
      if (j + 2 * k == t) a -= 1.f;
      if (j + 2 * k + 1 == t) b -= 1.f;
      __nv_bfloat162 h = __floats2bfloat162_rn(a * wgt, b * wgt);
      o[k] = *reinterpret_cast<uint32_t *>(&h);
    }
    *reinterpret_cast<uint4 *>(d + j) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

}  // namespace jf

int jf_launch_check(const char *what);

extern "C" int jf_cross_entropy_bf16(const uint16_t *logits, int64_t n, int64_t v, int64_t ld, const int64_t *y,
                                     const float *mask, const float *n_live, float *row_loss, uint16_t *dlogits,
                                     jf_stream_t stream) {
  if (n <= 0 || v <= 0 || ld % 8 || ld < v) return JF_ERR_ARG;
  jf::ce_bf16_kernel<<<(unsigned)n, 256, 0, (cudaStream_t)stream>>>(logits, v, ld, y, mask, n_live, row_loss,
                                                                     dlogits);
  return jf_launch_check("cross_entropy_bf16");
}
