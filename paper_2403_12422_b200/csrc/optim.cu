// optim.cu — AdamW (trainer.py:225-262) with the INT8 weight re-quantization fused in.
//
// Per element, in the reference's float32 operation order (numpy, scalars
// rounded to float32 as NEP 50 does for Python floats):
//   m = fl(fl(m*b1) + fl(omb1*g))            omb1 = f32(1 - b1)
//   v = fl(fl(v*b2) + fl(fl(omb2*g)*g))      omb2 = f32(1 - b2)
//   u = fl(fl(m/bc1) / fl(sqrt(fl(v/bc2)) + eps))
//   u = fl(u + fl(wd*p))                     (decayed keys only; wd = 0 skips it)
//   p = fl(p - fl(lr*u))
// Matrix parameters then leave the kernel with their INT8 copy already made
// (quantize_per_block of the updated master, qlayers.py:139-143) — one pass
// over p, g, m, v instead of an optimizer pass plus a quantizer pass.
#include "tile.cuh"

namespace jf {

struct AdamArgs {
  float b1, b2, omb1, omb2, bc1, bc2, eps, wd, lr;
};

JF_DEV float adam_elem(const AdamArgs &a, float &p, float g, float &m, float &v) {
  m = __fadd_rn(__fmul_rn(m, a.b1), __fmul_rn(a.omb1, g));
  v = __fadd_rn(__fmul_rn(v, a.b2), __fmul_rn(__fmul_rn(a.omb2, g), g));
  float u = __fdiv_rn(__fdiv_rn(m, a.bc1), __fadd_rn(__fsqrt_rn(__fdiv_rn(v, a.bc2)), a.eps));
  if (a.wd != 0.0f) u = __fadd_rn(u, __fmul_rn(a.wd, p));
  p = __fsub_rn(p, __fmul_rn(a.lr, u));
  return p;
}

// Flat update (vectors, or matrices without an INT8 copy): 4 elements per thread.
__global__ void __launch_bounds__(256) adamw_kernel(float *p, const float *__restrict__ g, float *m, float *v,
                                                    int64_t count, AdamArgs a) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    float pp = p[i], mm = m[i], vv = v[i];
    adam_elem(a, pp, __ldg(g + i), mm, vv);
    p[i] = pp;
    m[i] = mm;
    v[i] = vv;
  }
}

// Matrix update + per-block re-quantization of one 32 x 256 tile (tile.cuh).
JF_DEV void adamw_quant_tile(const TilePos &t, float *__restrict__ p, const float *__restrict__ g,
                             float *__restrict__ m, float *__restrict__ v, int64_t c, const AdamArgs &a,
                             int8_t *q, float *s, int32_t *err, uint32_t *red) {
  float w[4][8];
  if (t.active) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t off = t.row(i) * c + t.col();
      float4 p4[2], g4[2], m4[2], v4[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        p4[h] = reinterpret_cast<const float4 *>(p + off)[h];
        g4[h] = __ldg(reinterpret_cast<const float4 *>(g + off) + h);
        m4[h] = reinterpret_cast<const float4 *>(m + off)[h];
        v4[h] = reinterpret_cast<const float4 *>(v + off)[h];
      }
      float *pp = reinterpret_cast<float *>(p4), *gg = reinterpret_cast<float *>(g4);
      float *mm = reinterpret_cast<float *>(m4), *vv = reinterpret_cast<float *>(v4);
#pragma unroll
      for (int j = 0; j < 8; ++j) w[i][j] = adam_elem(a, pp[j], gg[j], mm[j], vv[j]);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        reinterpret_cast<float4 *>(p + off)[h] = p4[h];
        reinterpret_cast<float4 *>(m + off)[h] = m4[h];
        reinterpret_cast<float4 *>(v + off)[h] = v4[h];
      }
    }
  }
  quant_store(t, w, q, s, red, err);
}

__global__ void __launch_bounds__(kTileThreads) adamw_quant_kernel(float *__restrict__ p,
                                                                   const float *__restrict__ g,
                                                                   float *__restrict__ m, float *__restrict__ v,
                                                                   int64_t n, int64_t c, AdamArgs a,
                                                                   int8_t *q, float *s, int32_t *err) {
  __shared__ uint32_t red[64];
  adamw_quant_tile(tile_pos(n, c), p, g, m, v, c, a, q, s, err, red);
}

// All block weight matrices in one launch: a device table of tensors, each with the
// global index of its first 32 x 256 tile; CTA = one tile (the tensor found by a
// binary search over the tile starts).  Same per-tile work as adamw_quant_kernel, but
// no per-matrix launch and no per-matrix wave tail (a 1024 x 1024 matrix alone is 128
// tiles on 148 SMs).
struct AdamQTensor {
  float *p;
  const float *g;
  float *m;
  float *v;
  int8_t *q;
  float *s;
  int64_t n, c;
  float wd;
  int32_t pad;
  int64_t tile_start;
};
static_assert(sizeof(AdamQTensor) == 80, "AdamQTensor layout (mirrored in model.py)");

__global__ void __launch_bounds__(kTileThreads, 3) adamw_quant_multi_kernel(const AdamQTensor *__restrict__ tab,
                                                                         int32_t ntensors, AdamArgs a,
                                                                         int32_t *err) {
  __shared__ uint32_t red[64];
  const int64_t tile = blockIdx.x;
  int lo = 0, hi = ntensors - 1;  // last tensor whose tile_start <= tile
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(&tab[mid].tile_start) <= tile) lo = mid;
    else hi = mid - 1;
  }
  const AdamQTensor &T = tab[lo];
  const int64_t n = T.n, c = T.c, local = tile - T.tile_start;
  const int64_t gx = (c + kTileCols - 1) / kTileCols;
  TilePos t;
  t.r0 = (local / gx) * kTileRows;
  t.c0 = (local % gx) * kTileCols;
  t.n = n;
  t.c = c;
  t.warp = threadIdx.x >> 5;
  t.lane = threadIdx.x & 31;
  t.active = t.col() < c;
  AdamArgs aa = a;
  aa.wd = T.wd;
  adamw_quant_tile(t, T.p, T.g, T.m, T.v, c, aa, T.q, T.s, err, red);
}

// Many small tensors (biases, LayerNorm γ/β) in one launch: a table of tensors
// and a table of fixed-length chunks (tensor index, first element); one CTA
// per chunk.  Per-element arithmetic identical to adamw_kernel.
struct AdamTensor {
  float *p;
  const float *g;
  float *m;
  float *v;
  int64_t count;
  float wd;
  int32_t pad;
};
static_assert(sizeof(AdamTensor) == 48, "AdamTensor layout (mirrored in model.py)");

__global__ void __launch_bounds__(256) adamw_multi_kernel(const AdamTensor *__restrict__ tab,
                                                          const int32_t *__restrict__ chunk_tensor,
                                                          const int64_t *__restrict__ chunk_start,
                                                          int64_t chunk_len, AdamArgs a) {
  const AdamTensor T = tab[chunk_tensor[blockIdx.x]];
  const int64_t s = chunk_start[blockIdx.x];
  const int64_t e = min(s + chunk_len, T.count);
  AdamArgs aa = a;
  aa.wd = T.wd;
  for (int64_t i = s + threadIdx.x; i < e; i += blockDim.x) {
    float pp = T.p[i], mm = T.m[i], vv = T.v[i];
    adam_elem(aa, pp, __ldg(T.g + i), mm, vv);
    T.p[i] = pp;
    T.m[i] = mm;
    T.v[i] = vv;
  }
}

}  // namespace jf

using namespace jf;
int jf_launch_check(const char *what);

// b1, b2 arrive as doubles: the reference forms (1 - b1) in float64 before
// rounding it to float32, which differs from 1 - f32(b1) for b1 = 0.9.
static AdamArgs adam_args(float lr, double b1, double b2, float eps, float wd, float bc1, float bc2) {
  AdamArgs a;
  a.b1 = (float)b1;
  a.b2 = (float)b2;
  a.omb1 = (float)(1.0 - b1);
  a.omb2 = (float)(1.0 - b2);
  a.bc1 = bc1;
  a.bc2 = bc2;
  a.eps = eps;
  a.wd = wd;
  a.lr = lr;
  return a;
}

extern "C" int jf_adamw(float *p, const float *g, float *m, float *v, int64_t count, float lr, double b1, double b2,
                        float eps, float wd, float bc1, float bc2, jf_stream_t stream) {
  if (count <= 0) return JF_ERR_ARG;
  int64_t blocks = (count + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  adamw_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(p, g, m, v, count,
                                                                  adam_args(lr, b1, b2, eps, wd, bc1, bc2));
  return jf_launch_check("adamw");
}

extern "C" int jf_adamw_quantize(float *p, const float *g, float *m, float *v, int64_t n, int64_t c, float lr,
                                 double b1, double b2, float eps, float wd, float bc1, float bc2, int8_t *q, float *s,
                                 int32_t *err, jf_stream_t stream) {
  if (n % 32 || c % 32 || n <= 0 || c <= 0) return JF_ERR_ARG;
  adamw_quant_kernel<<<tile_grid(n, c), kTileThreads, 0, (cudaStream_t)stream>>>(
      p, g, m, v, n, c, adam_args(lr, b1, b2, eps, wd, bc1, bc2), q, s, err);
  return jf_launch_check("adamw_quantize");
}

extern "C" int jf_adamw_quantize_multi(const void *tensors, int32_t ntensors, int64_t total_tiles, float lr,
                                       double b1, double b2, float eps, float bc1, float bc2, int32_t *err,
                                       jf_stream_t stream) {
  if (ntensors <= 0 || total_tiles <= 0 || total_tiles > 0x7fffffff) return JF_ERR_ARG;
  adamw_quant_multi_kernel<<<(unsigned)total_tiles, kTileThreads, 0, (cudaStream_t)stream>>>(
      static_cast<const AdamQTensor *>(tensors), ntensors, adam_args(lr, b1, b2, eps, 0.0f, bc1, bc2), err);
  return jf_launch_check("adamw_quantize_multi");
}

extern "C" int jf_adamw_multi(const void *tensors, const int32_t *chunk_tensor, const int64_t *chunk_start,
                              int32_t nchunks, int64_t chunk_len, float lr, double b1, double b2, float eps,
                              float bc1, float bc2, jf_stream_t stream) {
  if (nchunks <= 0 || chunk_len <= 0) return JF_ERR_ARG;
  adamw_multi_kernel<<<(unsigned)nchunks, 256, 0, (cudaStream_t)stream>>>(
      static_cast<const AdamTensor *>(tensors), chunk_tensor, chunk_start, chunk_len,
      adam_args(lr, b1, b2, eps, 0.0f, bc1, bc2));
  return jf_launch_check("adamw_multi");
}
