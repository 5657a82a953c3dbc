// quant.cu — K1 quantizer, K2 dequantizer, block-tensor transpose.
//
// K1 (qtensor.py:219-246): HBM-bound, 4 B read + 1 B (+1/256 B scale) written
// per FP32 element; 2 B read for bf16 input.  One 32x256 tile per CTA.
#include "tile.cuh"

namespace jf {

template <typename T>
JF_DEV float to_f32(T v);
template <>
JF_DEV float to_f32<float>(float v) { return v; }
template <>
JF_DEV float to_f32<uint16_t>(uint16_t v) { return __uint_as_float((uint32_t)v << 16); }

__global__ void __launch_bounds__(kTileThreads) quantize_f32_kernel(const float *__restrict__ x,
                                                                    int64_t n, int64_t c,
                                                                    int64_t ldx, int8_t *q,
                                                                    float *s, int32_t *err) {
  __shared__ uint32_t red[64];
  const TilePos t = tile_pos(n, c);
  float v[4][8];
  if (t.active) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4 *p = reinterpret_cast<const float4 *>(x + t.row(i) * ldx + t.col());
      const float4 a = __ldg(p), b = __ldg(p + 1);
      v[i][0] = a.x; v[i][1] = a.y; v[i][2] = a.z; v[i][3] = a.w;
      v[i][4] = b.x; v[i][5] = b.y; v[i][6] = b.z; v[i][7] = b.w;
    }
  }
  quant_store(t, v, q, s, red, err);
}

__global__ void __launch_bounds__(kTileThreads) quantize_bf16_kernel(
    const uint16_t *__restrict__ x, int64_t n, int64_t c, int64_t ldx, int8_t *q, float *s,
    int32_t *err) {
  __shared__ uint32_t red[64];
  const TilePos t = tile_pos(n, c);
  float v[4][8];
  if (t.active) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint4 w = __ldg(reinterpret_cast<const uint4 *>(x + t.row(i) * ldx + t.col()));
      const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        v[i][2 * j] = __uint_as_float(u[j] << 16);
        v[i][2 * j + 1] = __uint_as_float(u[j] & 0xffff0000u);
      }
    }
  }
  quant_store(t, v, q, s, red, err);
}

// K2: 16 codes per thread (one 16-byte load, one scale), grid-stride.
template <bool BF16>
__global__ void __launch_bounds__(256) dequantize_kernel(const int8_t *__restrict__ q,
                                                         const float *__restrict__ s, int64_t n,
                                                         int64_t c, void *y) {
  const int64_t total = n * c / 16;
  const int64_t cb = c >> 5;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i * 16;
    const int64_t r = e / c, cc = e - r * c;
    const DeqScale dk = deq_scale(__ldg(s + (r >> 5) * cb + (cc >> 5)));
    const uint4 w = __ldg(reinterpret_cast<const uint4 *>(q) + i);
    const uint32_t u[4] = {w.x, w.y, w.z, w.w};
    if (BF16) {
      uint32_t o[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        // products are exact in fp32; bf16 output rounds them RNE
        float f[4];
        deq4(u[k], dk, f);
        __nv_bfloat162 a = __floats2bfloat162_rn(f[0], f[1]), b = __floats2bfloat162_rn(f[2], f[3]);
        o[2 * k] = *reinterpret_cast<uint32_t *>(&a);
        o[2 * k + 1] = *reinterpret_cast<uint32_t *>(&b);
      }
      uint4 *dst = reinterpret_cast<uint4 *>(static_cast<uint16_t *>(y) + e);
      dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
      dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
    } else {
      float4 *dst = reinterpret_cast<float4 *>(static_cast<float *>(y) + e);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float f[4];
        deq4(u[k], dk, f);
        dst[k] = make_float4(f[0], f[1], f[2], f[3]);
      }
    }
  }
}

// ── the attention boundary (qlayers.py:350-351, 406-408) ────────────────
// The FP island runs torch SDPA on per-head [batch, heads, seq, head_dim]
// bf16 tensors.  These two kernels move between that layout and the INT8
// [tokens, channels] BlockQuantTensors directly, so no transposed / sliced
// copies are materialized around the attention call.

// QKV codes [n x 3c] (n = batch*seq, c = heads*hd) -> q, k, v bf16, each
// contiguous [batch, heads, seq, hd].  16 codes per thread (hd % 16 == 0).
__global__ void __launch_bounds__(256) dequant_qkv_heads_kernel(const int8_t *__restrict__ q,
                                                                const float *__restrict__ s, int64_t n,
                                                                int64_t c, int64_t seq, int64_t heads,
                                                                int64_t hd, uint16_t *yq, uint16_t *yk,
                                                                uint16_t *yv) {
  const int64_t c3 = 3 * c;
  const int64_t total = n * c3 / 16;
  const int64_t cb = c3 >> 5;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i * 16;
    const int64_t r = e / c3, cc = e - r * c3;
    const DeqScale dk = deq_scale(__ldg(s + (r >> 5) * cb + (cc >> 5)));
    const uint4 w = __ldg(reinterpret_cast<const uint4 *>(q) + i);
    const uint32_t u[4] = {w.x, w.y, w.z, w.w};
    uint32_t o[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float f[4];
      deq4(u[k], dk, f);
      __nv_bfloat162 a = __floats2bfloat162_rn(f[0], f[1]), b = __floats2bfloat162_rn(f[2], f[3]);
      o[2 * k] = *reinterpret_cast<uint32_t *>(&a);
      o[2 * k + 1] = *reinterpret_cast<uint32_t *>(&b);
    }
    const int64_t which = cc / c, jj = cc - which * c;
    const int64_t h = jj / hd, d = jj - h * hd;
    const int64_t b = r / seq, sq = r - b * seq;
    uint16_t *base = which == 0 ? yq : (which == 1 ? yk : yv);
    uint4 *dst = reinterpret_cast<uint4 *>(base + ((b * heads + h) * seq + sq) * hd + d);
    dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
    dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
  }
}

// bf16 x[batch, seq, heads, hd] with element strides (sb, ss, sh, 1) -> INT8
// [n x c] block tensor written into a column slice (codes stride ldq, grid
// stride lds).  Quantization as K1 (qtensor.py:219-246).
__global__ void __launch_bounds__(kTileThreads) quantize_heads_kernel(
    const uint16_t *__restrict__ x, int64_t n, int64_t c, int64_t seq, int64_t hd, int64_t sb, int64_t ss,
    int64_t sh, int8_t *q, int64_t ldq, float *s, int64_t lds, int32_t *err) {
  __shared__ uint32_t red[64];
  const TilePos t = tile_pos(n, c);
  float v[4][8];
  if (t.active) {
    const int64_t j = t.col(), h = j / hd, d = j - h * hd;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t r = t.row(i), b = r / seq, sq = r - b * seq;
      const uint4 w = __ldg(reinterpret_cast<const uint4 *>(x + b * sb + sq * ss + h * sh + d));
      const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        v[i][2 * k] = __uint_as_float(u[k] << 16);
        v[i][2 * k + 1] = __uint_as_float(u[k] & 0xffff0000u);
      }
    }
  }
  quant_store_ld(t, v, q, ldq, s, lds, red, err);
}

// Transpose codes [n x c] -> [c x n] via a 64x64 smem tile; scales transpose
// alongside (the 2x2 scale blocks of the tile).
__global__ void __launch_bounds__(256) transpose_kernel(const int8_t *__restrict__ q,
                                                        const float *__restrict__ s, int64_t n,
                                                        int64_t c, int8_t *qt, float *st) {
  __shared__ uint32_t tile[64][17];  // 64 rows x 64 bytes (+pad word)
  const int64_t r0 = (int64_t)blockIdx.y * 64, c0 = (int64_t)blockIdx.x * 64;
  const int tid = threadIdx.x;
  // load: 64 rows x 16 words; 256 threads -> 4 words each
  for (int k = tid; k < 64 * 16; k += 256) {
    const int rr = k >> 4, ww = k & 15;
    const int64_t r = r0 + rr, cc = c0 + ww * 4;
    uint32_t val = 0;
    if (r < n && cc < c) val = *reinterpret_cast<const uint32_t *>(q + r * c + cc);
    tile[rr][ww] = val;
  }
  __syncthreads();
  // store: output row = input column (c0 + oc), 64 output rows x 16 words
  for (int k = tid; k < 64 * 16; k += 256) {
    const int oc = k >> 4, ow = k & 15;  // output row oc, word ow (input rows 4ow..4ow+3)
    const int64_t orow = c0 + oc, ocol = r0 + ow * 4;
    if (orow < c && ocol < n) {
      uint32_t out = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const uint32_t word = tile[ow * 4 + b][oc >> 2];
        out |= ((word >> (8 * (oc & 3))) & 0xffu) << (8 * b);
      }
      *reinterpret_cast<uint32_t *>(qt + orow * n + ocol) = out;
    }
  }
  if (tid < 4 && st != nullptr) {
    const int64_t br = (r0 >> 5) + (tid >> 1), bc = (c0 >> 5) + (tid & 1);
    if (br < (n >> 5) && bc < (c >> 5)) st[bc * (n >> 5) + br] = s[br * (c >> 5) + bc];
  }
}

}  // namespace jf

using namespace jf;

int jf_launch_check(const char *what);

extern "C" int jf_quantize_f32(const float *x, int64_t n, int64_t c, int64_t ldx, int8_t *q,
                               float *s, int32_t *err, jf_stream_t stream) {
  if (n % 32 || c % 32 || n <= 0 || c <= 0 || ldx < c || ldx % 4) return JF_ERR_ARG;
  quantize_f32_kernel<<<tile_grid(n, c), kTileThreads, 0, (cudaStream_t)stream>>>(x, n, c, ldx,
                                                                                  q, s, err);
  return jf_launch_check("quantize_f32");
}

extern "C" int jf_quantize_bf16(const uint16_t *x, int64_t n, int64_t c, int64_t ldx, int8_t *q,
                                float *s, int32_t *err, jf_stream_t stream) {
  if (n % 32 || c % 32 || n <= 0 || c <= 0 || ldx < c || ldx % 8) return JF_ERR_ARG;
  quantize_bf16_kernel<<<tile_grid(n, c), kTileThreads, 0, (cudaStream_t)stream>>>(x, n, c, ldx,
                                                                                   q, s, err);
  return jf_launch_check("quantize_bf16");
}

static int dq_grid(int64_t n, int64_t c) {
  int64_t th = n * c / 16;
  int64_t b = (th + 255) / 256;
  int64_t cap = 148LL * 16;
  return (int)(b < cap ? (b > 0 ? b : 1) : cap);
}

extern "C" int jf_dequantize_f32(const int8_t *q, const float *s, int64_t n, int64_t c, float *y,
                                 jf_stream_t stream) {
  if (n % 32 || c % 32 || n <= 0 || c <= 0) return JF_ERR_ARG;
  dequantize_kernel<false><<<dq_grid(n, c), 256, 0, (cudaStream_t)stream>>>(q, s, n, c, y);
  return jf_launch_check("dequantize_f32");
}

extern "C" int jf_dequantize_bf16(const int8_t *q, const float *s, int64_t n, int64_t c,
                                  uint16_t *y, jf_stream_t stream) {
  if (n % 32 || c % 32 || n <= 0 || c <= 0) return JF_ERR_ARG;
  dequantize_kernel<true><<<dq_grid(n, c), 256, 0, (cudaStream_t)stream>>>(q, s, n, c, y);
  return jf_launch_check("dequantize_bf16");
}

extern "C" int jf_dequantize_qkv_heads(const int8_t *q, const float *s, int64_t batch, int64_t seq,
                                       int64_t heads, int64_t head_dim, uint16_t *yq, uint16_t *yk, uint16_t *yv,
                                       jf_stream_t stream) {
  const int64_t n = batch * seq, c = heads * head_dim;
  if (n % 32 || c % 32 || n <= 0 || c <= 0 || head_dim % 16) return JF_ERR_ARG;
  dequant_qkv_heads_kernel<<<dq_grid(n, 3 * c), 256, 0, (cudaStream_t)stream>>>(q, s, n, c, seq, heads, head_dim,
                                                                              yq, yk, yv);
  return jf_launch_check("dequant_qkv_heads");
}

extern "C" int jf_quantize_heads_bf16(const uint16_t *x, int64_t batch, int64_t seq, int64_t heads,
                                      int64_t head_dim, int64_t sb, int64_t ss, int64_t sh, int8_t *q, int64_t ldq,
                                      float *s, int64_t lds, int32_t *err, jf_stream_t stream) {
  const int64_t n = batch * seq, c = heads * head_dim;
  if (n % 32 || c % 32 || n <= 0 || c <= 0 || head_dim % 8 || ldq < c || (sb | ss | sh) % 8) return JF_ERR_ARG;
  quantize_heads_kernel<<<tile_grid(n, c), kTileThreads, 0, (cudaStream_t)stream>>>(
      x, n, c, seq, head_dim, sb, ss, sh, q, ldq, s, lds, err);
  return jf_launch_check("quantize_heads");
}

extern "C" int jf_transpose(const int8_t *q, const float *s, int64_t n, int64_t c, int8_t *qt,
                            float *st, jf_stream_t stream) {
  if (n % 32 || c % 32 || n <= 0 || c <= 0) return JF_ERR_ARG;
  dim3 grid((unsigned)((c + 63) / 64), (unsigned)((n + 63) / 64));
  transpose_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(q, s, n, c, qt, st);
  return jf_launch_check("transpose");
}
