// tile.cuh — the 32 x 256 register tile shared by every memory-bound kernel.
//
// One CTA of 256 threads owns a 32-row strip x 256 columns (8 quantization
// blocks).  Warp w holds rows 4w..4w+3, lane l holds columns 8l..8l+7 of
// each of those rows, i.e. 32 FP32 values per thread, so every global
// access is a fully used 256-byte row segment per warp (int8) and the
// 32 x 32 block absmax needs one 4-lane shuffle + one cross-warp smem step.
#pragma once

#include "common.cuh"

namespace jf {

constexpr int kTileRows = 32;
constexpr int kTileCols = 256;
constexpr int kTileThreads = 256;

struct TilePos {
  int64_t r0;   // first row of the strip
  int64_t c0;   // first column of the tile
  int64_t n, c; // matrix shape
  int warp, lane;
  bool active;  // this thread's 8 columns lie inside the matrix

  JF_DEV int64_t row(int i) const { return r0 + 4 * warp + i; }
  JF_DEV int64_t col() const { return c0 + 8 * lane; }
  JF_DEV int64_t scale_idx(int64_t r, int64_t cc) const { return (r >> 5) * (c >> 5) + (cc >> 5); }
};

JF_DEV TilePos tile_pos(int64_t n, int64_t c) {
  TilePos t;
  t.r0 = (int64_t)blockIdx.y * kTileRows;
  t.c0 = (int64_t)blockIdx.x * kTileCols;
  t.n = n;
  t.c = c;
  t.warp = threadIdx.x >> 5;
  t.lane = threadIdx.x & 31;
  t.active = t.col() < c;  // c is a multiple of 32 -> whole quant blocks
  return t;
}

// Load 4 rows x 8 int8 codes and dequantize them (exact: code * scale).
JF_DEV void load_deq(const TilePos &t, const int8_t *__restrict__ q, const float *__restrict__ s,
                     float (&v)[4][8]) {
  if (!t.active) return;
  const DeqScale k = deq_scale(__ldg(s + t.scale_idx(t.r0, t.col())));  // 4 rows share one row block
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint2 w = __ldg(reinterpret_cast<const uint2 *>(q + t.row(i) * t.c + t.col()));
    deq8_packed(w.x, w.y, k, v[i]);
  }
}

// Requantize the FP32 tile per 32x32 block and store codes + scales into a column
// slice of a BlockQuantTensor (quantize_per_block semantics, qtensor.py:219-246):
// codes row stride ldq, scale grid row stride lds (q and s already offset to the
// slice).  `red` is >= 64 words of shared memory.  Ends with the CTA synchronized.
//
// Common path, per element ~3 issue slots: y = fl(x * fl(1/s)) and its magic-number
// rounding t = fl(y + 1.5*2^23) in packed f32x2 ops (the product is an FFMA2 with an
// opaque +0 addend so ptxas cannot contract it into the add), the row's largest
// distance |y - rint(y)| by 3-input max, and the code bytes taken straight from the
// low bytes of t (t = 1.5*2^23 + q exactly, |y| < 2^22).  Exact exactly when the
// scale is a normal binary16 value (then |x/s| <= 127 * (1 + 2^-11) < 127.5: the
// reference's clip is a no-op) and no y lies within 3e-5 of a half-integer
// (quant_code_try's argument).  Otherwise the row takes the exact per-element path.
JF_DEV void quant_store_ld(const TilePos &t, const float (&v)[4][8], int8_t *__restrict__ q, int64_t ldq,
                           float *__restrict__ s, int64_t lds, uint32_t *red, int32_t *err) {
  uint32_t m = 0;
  if (t.active) {
    float mf = absmax3_nan(v[0][0], v[0][1], v[0][2]);
#pragma unroll
    for (int e = 3; e < 31; e += 2) mf = absmax3_nan(mf, v[e >> 3][e & 7], v[(e + 1) >> 3][(e + 1) & 7]);
    mf = absmax3_nan(mf, v[3][7], 0.0f);
    m = __float_as_uint(mf);  // NaN -> >= 0x7f800000 like the integer max of |bits|
  }
  m = max(m, __shfl_xor_sync(0xffffffffu, m, 1));
  m = max(m, __shfl_xor_sync(0xffffffffu, m, 2));
  const int qb = t.lane >> 2;
  if ((t.lane & 3) == 0) red[t.warp * 8 + qb] = m;
  __syncthreads();
  uint32_t am = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) am = max(am, red[w * 8 + qb]);
  int flags = 0;
  const float sc = block_scale(am, flags);
  const float rc = __frcp_rn(sc);
  const bool fast_ok = flags == 0 && sc >= 6.103515625e-05f;  // normal binary16 scale
  if (t.active) {
    const float zero = opaque_zero();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint2 w;
      float tt[8], emax = 0.0f;
#pragma unroll
      for (int j = 0; j < 8; j += 2) {
        float y0, y1, u0, u1, e0, e1;
        ffma2_rn(y0, y1, v[i][j], v[i][j + 1], rc, rc, zero, zero);
        fadd2_rn(tt[j], tt[j + 1], y0, y1, 12582912.0f, 12582912.0f);
        fsub2_rn(u0, u1, tt[j], tt[j + 1], 12582912.0f, 12582912.0f);
        fsub2_rn(e0, e1, y0, y1, u0, u1);
        emax = absmax3_nan(emax, e0, e1);
      }
      if (fast_ok && emax < 0.49997f) {
        w.x = prmt(prmt(__float_as_uint(tt[0]), __float_as_uint(tt[1]), 0x0040u),
                   prmt(__float_as_uint(tt[2]), __float_as_uint(tt[3]), 0x0040u), 0x5410u);
        w.y = prmt(prmt(__float_as_uint(tt[4]), __float_as_uint(tt[5]), 0x0040u),
                   prmt(__float_as_uint(tt[6]), __float_as_uint(tt[7]), 0x0040u), 0x5410u);
      } else {  // rare: near-tie, subnormal scale or flagged block -> exact per element
        w.x = pack4(quant_code_fast(v[i][0], sc, rc), quant_code_fast(v[i][1], sc, rc),
                    quant_code_fast(v[i][2], sc, rc), quant_code_fast(v[i][3], sc, rc));
        w.y = pack4(quant_code_fast(v[i][4], sc, rc), quant_code_fast(v[i][5], sc, rc),
                    quant_code_fast(v[i][6], sc, rc), quant_code_fast(v[i][7], sc, rc));
      }
      *reinterpret_cast<uint2 *>(q + t.row(i) * ldq + t.col()) = w;
    }
    if (t.warp == 0 && (t.lane & 3) == 0) {
      s[(t.r0 >> 5) * lds + (t.col() >> 5)] = sc;
      raise_flags(err, flags);
    }
  }
  __syncthreads();
}

// quant_store into a whole [n x c] BlockQuantTensor.
JF_DEV void quant_store(const TilePos &t, const float (&v)[4][8], int8_t *__restrict__ q,
                        float *__restrict__ s, uint32_t *red, int32_t *err) {
  quant_store_ld(t, v, q, t.c, s, t.c >> 5, red, err);
}

inline dim3 tile_grid(int64_t n, int64_t c) {
  return dim3((unsigned)((c + kTileCols - 1) / kTileCols), (unsigned)(n / kTileRows));
}

}  // namespace jf
