// ce.cu — the loss head's softmax cross-entropy, fused (model step, trainer.py:387-406).
//
// The reference computes, per token row r of the logits,
//   logp = log_softmax(logits);  loss = -sum_r mask_r * logp[r, y_r] / n_live
//   dlogits = (exp(logp) - onehot(y)) * mask_r / n_live
// (trainer.py:388-404).  With the BF16 head the logits arrive as bf16 [n x ld];
// (columns v..ld must hold -inf: the vocabulary padding), one CTA per row does
// an online max/sum-exp pass, writes the row's loss term,
// and a second pass writes dlogits as bf16 — the operand the two head-gradient
// GEMMs consume — so no FP32 logits/probabilities ever reach HBM.  Padded
// vocabulary columns carry -inf logits and get exactly zero gradient.
#include "common.cuh"

namespace jf {

JF_DEV void online_merge(float &m, float &s, float m2, float s2) {
  if (m2 == -INFINITY) return;
  if (m == -INFINITY) {
    m = m2;
    s = s2;
    return;
  }
  const float mx = fmaxf(m, m2);
  s = s * expf(m - mx) + s2 * expf(m2 - mx);
  m = mx;
}

JF_DEV float bf16_to_f32(uint32_t h16) { return __uint_as_float(h16 << 16); }

__global__ void __launch_bounds__(256) ce_bf16_kernel(const uint16_t *__restrict__ logits, int64_t v, int64_t ld,
                                                      const int64_t *__restrict__ y, const float *__restrict__ mask,
                                                      const float *__restrict__ n_live, float *row_loss,
                                                      uint16_t *dl) {
  __shared__ float sm_m[8], sm_s[8];
  __shared__ float s_lse;
  const int64_t row = blockIdx.x;
  const uint16_t *x = logits + row * ld;
  // pass 1: online max / sum of exp, 8 bf16 per thread per step
  float m = -INFINITY, s = 0.f;
  for (int64_t j = (int64_t)threadIdx.x * 8; j < ld; j += (int64_t)blockDim.x * 8) {  // padding is -inf
    const uint4 w = __ldg(reinterpret_cast<const uint4 *>(x + j));
    const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float val = bf16_to_f32(k & 1 ? u[k >> 1] >> 16 : u[k >> 1] & 0xffffu);
      if (val > m) {
        s = (m == -INFINITY ? 0.f : s * expf(m - val)) + 1.f;
        m = val;
      } else if (val != -INFINITY) {
        s += expf(val - m);
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) online_merge(m, s, __shfl_xor_sync(0xffffffffu, m, o), __shfl_xor_sync(0xffffffffu, s, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sm_m[warp] = m;
    sm_s[warp] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = sm_m[0], S = sm_s[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) online_merge(M, S, sm_m[w], sm_s[w]);
    s_lse = M + logf(S);
    const float wgt = (mask ? mask[row] : 1.f) / *n_live;
    const int64_t t = y[row];
    row_loss[row] = -(bf16_to_f32(x[t]) - s_lse) * wgt;
  }
  __syncthreads();
  const float lse = s_lse;
  const float wgt = (mask ? mask[row] : 1.f) / *n_live;
  const int64_t t = y[row];
  uint16_t *d = dl + row * ld;
  // pass 2: dlogits = (softmax - onehot) * mask / n_live, bf16 (RNE)
  for (int64_t j = (int64_t)threadIdx.x * 8; j < ld; j += (int64_t)blockDim.x * 8) {
    uint32_t o[4];
    const uint4 w = __ldg(reinterpret_cast<const uint4 *>(x + j));
    const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {  // exp(-inf - lse) = 0: padded columns get exactly zero
      float a = expf(bf16_to_f32(u[k] & 0xffffu) - lse), b = expf(bf16_to_f32(u[k] >> 16) - lse);
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
