// eltwise.cu — K6..K11: the INT8-in / INT8-out memory-bound operators.
//
// Every kernel reads INT8 codes + block scales, computes in FP32 in the
// reference's exact operation order (qnonlinear.py), and requantizes per
// 32x32 block in registers before writing INT8 back: no FP16/FP32
// activation ever reaches HBM.  Reductions mirror numpy's float32
// pairwise order (see oracle.pairwise_sum) so codes, scales and statistics
// are bit-exact; column (axis-0) parameter-gradient sums are reduced
// strip-wise (tolerance).
#include <algorithm>

#include "tile.cuh"

namespace jf {

// ── K6: residual Add + RowStats (qnonlinear.py:246-267, :134-144) ───────
// Stats of the FP32 sum y (before requantization), per (row, width block):
// mean = fl(pairwise(y)/w), sumsq = pairwise(fl(y*y)).  y is staged in smem
// (row stride 257 floats: conflict-free column walks).
__global__ void __launch_bounds__(kTileThreads) add_stats_kernel(
    const int8_t *__restrict__ a, const float *__restrict__ as, const int8_t *__restrict__ b,
    const float *__restrict__ bs, int64_t n, int64_t c, int width, int tile_w, int8_t *yq,
    float *ys, float *mean, float *sumsq, int32_t *err) {
  extern __shared__ float ysm[];  // [32][257]
  __shared__ uint32_t red[64];
  TilePos t = tile_pos(n, c);
  t.c0 = (int64_t)blockIdx.x * tile_w;
  t.active = (8 * t.lane < tile_w) && (t.col() < c);
  float v[4][8];
  float w2[4][8];
  load_deq(t, a, as, v);
  if (b != nullptr) {
    load_deq(t, b, bs, w2);
    if (t.active) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; j += 2) fadd2_rn(v[i][j], v[i][j + 1], v[i][j], v[i][j + 1], w2[i][j], w2[i][j + 1]);
    }
  } else if (t.active) {
    // Add(x, zeros_like(x)): x + 0.0 (turns -0.0 into +0.0 exactly like numpy)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; j += 2) fadd2_rn(v[i][j], v[i][j + 1], v[i][j], v[i][j + 1], 0.0f, 0.0f);
  }
  if (t.active) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) ysm[(4 * t.warp + i) * 257 + 8 * t.lane + j] = v[i][j];
  }
  __syncthreads();
  // one thread per (row, stats block): row = tid % 32, block = tid / 32 (+ 8k)
  const int64_t valid_w = min((int64_t)tile_w, c - t.c0);
  const int nblk = (int)(valid_w / width);
  const int64_t cw = c / width;
  if (width == 64 && 2 * 32 * nblk <= kTileThreads) {
    // pairwise_leaf(64) unrolled, both sums in one pass over shared memory, two threads
    // per (row, block): thread half h owns numpy's chains 4h..4h+3 (r[j] = a[j], then
    // r[j] += a[j + 8i] in order); ((r0+r1)+(r2+r3)) + ((r4+r5)+(r6+r7)) across the pair.
    const int item = threadIdx.x >> 1, hh = threadIdx.x & 1;
    const int row = item & 31, blk = item >> 5;
    const bool ok = item < 32 * nblk;
    float r1[4], r2[4];
    if (ok) {
      const float *pb = ysm + row * 257 + blk * 64 + 4 * hh;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float a0 = pb[j];
        r1[j] = a0;
        r2[j] = __fmul_rn(a0, a0);
      }
#pragma unroll
      for (int i = 8; i < 64; i += 8)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float a0 = pb[i + j];
          r1[j] = __fadd_rn(r1[j], a0);
          r2[j] = __fadd_rn(r2[j], __fmul_rn(a0, a0));
        }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) r1[j] = r2[j] = 0.f;
    }
    float h1 = __fadd_rn(__fadd_rn(r1[0], r1[1]), __fadd_rn(r1[2], r1[3]));
    float h2 = __fadd_rn(__fadd_rn(r2[0], r2[1]), __fadd_rn(r2[2], r2[3]));
    const float o1 = __shfl_xor_sync(0xffffffffu, h1, 1), o2 = __shfl_xor_sync(0xffffffffu, h2, 1);
    if (ok && hh == 0) {
      const int64_t oi = (t.r0 + row) * cw + t.c0 / width + blk;
      mean[oi] = __fdiv_rn(__fadd_rn(h1, o1), (float)width);
      sumsq[oi] = __fadd_rn(h2, o2);
    }
  } else
  for (int item = threadIdx.x; item < 32 * nblk; item += kTileThreads) {
    const int row = item & 31, blk = item >> 5;
    const float *base = ysm + row * 257 + blk * width;
    const float s1 = pairwise_sum([&](int k) { return base[k]; }, 0, width);
    const float s2 = pairwise_sum([&](int k) { return __fmul_rn(base[k], base[k]); }, 0, width);
    const int64_t oi = (t.r0 + row) * cw + t.c0 / width + blk;
    mean[oi] = __fdiv_rn(s1, (float)width);
    sumsq[oi] = s2;
  }
  quant_store(t, v, yq, ys, red, err);
}

// ── K7: LayerNorm forward (qnonlinear.py:300-330) ──────────────────────
// Per-row moments from the Add statistics: 8 lanes per row reproduce the
// 8-accumulator pairwise sum over the c/width block means / sums of squares.
JF_DEV float pairwise_small_8lanes(const float *__restrict__ p, int nb, int sub) {
  // valid for 8 <= nb <= 128; lanes sub=0..7 of an aligned 8-lane group
  float r = p[sub];
  const int lim = nb - (nb % 8);
  for (int i = 8; i < lim; i += 8) r = __fadd_rn(r, p[i + sub]);
  r = __fadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
  r = __fadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
  r = __fadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
  for (int i = lim; i < nb; ++i) r = __fadd_rn(r, p[i]);
  return r;
}

__global__ void __launch_bounds__(256) ln_moments_kernel(const float *__restrict__ mean,
                                                         const float *__restrict__ sumsq,
                                                         int64_t n, int64_t c, int nb, float eps,
                                                         float *mu, float *inv_std) {
  const int64_t row = (int64_t)blockIdx.x * 32 + (threadIdx.x >> 3);
  const int sub = threadIdx.x & 7;
  if (row >= n) return;  // whole 8-lane groups exit together
  const float *pm = mean + row * nb;
  const float *ps = sumsq + row * nb;
  float sm, ss;
  if (nb >= 8 && nb <= 128) {
    sm = pairwise_small_8lanes(pm, nb, sub);
    ss = pairwise_small_8lanes(ps, nb, sub);
  } else {
    sm = pairwise_sum([&](int k) { return pm[k]; }, 0, nb);
    ss = pairwise_sum([&](int k) { return ps[k]; }, 0, nb);
  }
  if (sub == 0) {
    const float m = __fdiv_rn(sm, (float)nb);                          // row_mean
    float var = __fsub_rn(__fdiv_rn(ss, (float)c), __fmul_rn(m, m));   // row_var
    var = var > 0.0f ? var : 0.0f;  // np.maximum(var, 0.0) (NaN cannot occur: finite stats)
    const float sd = __fsqrt_rn(__fadd_rn(var, eps));
    mu[row] = m;
    inv_std[row] = __fdiv_rn(1.0f, sd);
  }
}

// 8 consecutive floats; kVec: as two 16-byte loads (p 16-byte aligned)
template <bool kVec>
JF_DEV void ldg8(const float *__restrict__ p, float (&d)[8]) {
  if (kVec) {
    const float4 a = __ldg(reinterpret_cast<const float4 *>(p)), b = __ldg(reinterpret_cast<const float4 *>(p) + 1);
    d[0] = a.x, d[1] = a.y, d[2] = a.z, d[3] = a.w, d[4] = b.x, d[5] = b.y, d[6] = b.z, d[7] = b.w;
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) d[j] = __ldg(p + j);
  }
}

// 4 consecutive floats (the warp's 4 rows of a per-row vector; p 16-byte aligned if kVec)
template <bool kVec>
JF_DEV void ldg4(const float *__restrict__ p, float (&d)[4]) {
  if (kVec) {
    const float4 a = __ldg(reinterpret_cast<const float4 *>(p));
    d[0] = a.x, d[1] = a.y, d[2] = a.z, d[3] = a.w;
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) d[j] = __ldg(p + j);
  }
}

// kVec: gamma, beta, mu, inv_std 16-byte aligned (per-lane float4 loads instead of 16 strided
// scalar loads that touch 8 cache lines per warp each).  mu / inv_std of the warp's 4
// rows are one broadcast float4 each (kVec also requires mu / inv_std 16-byte aligned).
template <bool kVec>
__global__ void __launch_bounds__(kTileThreads) ln_fwd_kernel(
    const int8_t *__restrict__ x, const float *__restrict__ xs, const float *__restrict__ mu,
    const float *__restrict__ inv_std, const float *__restrict__ gamma,
    const float *__restrict__ beta, int64_t n, int64_t c, int8_t *yq, float *ys, int32_t *err) {
  __shared__ uint32_t red[64];
  const TilePos t = tile_pos(n, c);
  float v[4][8];
  load_deq(t, x, xs, v);
  if (t.active) {
    float g[8], bb[8];
    ldg8<kVec>(gamma + t.col(), g);
    ldg8<kVec>(beta + t.col(), bb);
    float mv[4], sv[4];
    ldg4<kVec>(mu + t.row(0), mv);
    ldg4<kVec>(inv_std + t.row(0), sv);
    const float zero = opaque_zero();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float m = mv[i], is = sv[i];
#pragma unroll
      for (int j = 0; j < 8; j += 2) {  // packed, same roundings: fl(fl(g*fl(fl(x-m)*is)) + b)
        float x0, x1;
        fsub2_rn(x0, x1, v[i][j], v[i][j + 1], m, m);
        fmul2_rn(x0, x1, x0, x1, is, is);
        ffma2_rn(x0, x1, g[j], g[j + 1], x0, x1, zero, zero);  // rounded product: no contraction
        fadd2_rn(v[i][j], v[i][j + 1], x0, x1, bb[j], bb[j + 1]);
      }
    }
  }
  quant_store(t, v, yq, ys, red, err);
}

// ── K8: LayerNorm backward (qnonlinear.py:333-355) ─────────────────────
// Pass A (per row): m1 = mean(dxhat), m2 = mean(dxhat*xhat) over C in numpy's
// pairwise tree.  The tree of a row is "perfect" (all leaves at one depth)
// for every C used here; leaf i goes to lane i*L/32.. and the butterfly over
// lanes reproduces the upper levels.  Non-perfect C falls back to lane 0.
struct LnRowArgs {
  const int8_t *x;
  const float *xs;
  const float *mu, *inv_std;
  const int8_t *dy;
  const float *dys;
  const float *gamma;
  int64_t n, c;
};

JF_DEV void ln_row_vals(const LnRowArgs &A, int64_t row, int64_t col, float mrow, float isrow,
                        float &dxhat, float &xhat) {
  const int64_t cb = A.c >> 5;
  const float sx = __ldg(A.xs + (row >> 5) * cb + (col >> 5));
  const float sd = __ldg(A.dys + (row >> 5) * cb + (col >> 5));
  const float xv = __fmul_rn((float)A.x[row * A.c + col], sx);
  const float dv = __fmul_rn((float)A.dy[row * A.c + col], sd);
  xhat = __fmul_rn(__fsub_rn(xv, mrow), isrow);
  dxhat = __fmul_rn(dv, __ldg(A.gamma + col));
}

// Fast path (perfect tree, all NL = 2^depth leaves of equal size Lf, Lf % 8 == 0):
// numpy's leaf sum is ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) with r_j the
// sequential sum of elements j, j+8, ..., so the whole row is a balanced tree
// over 8*NL sequential "chains".  Lane (g = lane>>3, j = lane&7) sums chain j
// of leaf 4*it + g; xor-butterflies over j (1,2,4) give leaf sums, over g (8,16)
// pairs/quads of leaves, and the per-iteration values are combined in index
// order in registers — the exact numpy association, with all 32 lanes busy.
__global__ void __launch_bounds__(256) ln_bwd_rows_fast_kernel(LnRowArgs A, int nleaf, int leaf_len,
                                                               float *m1, float *m2) {
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= A.n) return;
  const float mr = __ldg(A.mu + row), ir = __ldg(A.inv_std + row);
  const int g = lane >> 3, j = lane & 7;
  const int64_t cb = A.c >> 5;
  const int8_t *xr = A.x + row * A.c;
  const int8_t *dr = A.dy + row * A.c;
  const float *sxr = A.xs + (row >> 5) * cb;
  const float *sdr = A.dys + (row >> 5) * cb;
  const int iters = (nleaf + 3) >> 2;
  const int gl = nleaf < 4 ? nleaf : 4;  // leaves per iteration
  float v1[32], v2[32];  // per-iteration partial trees (nleaf <= 128)
  for (int it = 0; it < iters; ++it) {
    const int L = it * 4 + g;
    float c1 = 0.f, c2 = 0.f;
    if (L < nleaf) {
      const int base = L * leaf_len + j;
      for (int i = 0; i < leaf_len / 8; ++i) {
        const int k = base + 8 * i;
        const float xv = __fmul_rn((float)xr[k], __ldg(sxr + (k >> 5)));
        const float dv = __fmul_rn((float)dr[k], __ldg(sdr + (k >> 5)));
        const float xh = __fmul_rn(__fsub_rn(xv, mr), ir);
        const float dxh = __fmul_rn(dv, __ldg(A.gamma + k));
        const float pr = __fmul_rn(dxh, xh);
        c1 = (i == 0) ? dxh : __fadd_rn(c1, dxh);
        c2 = (i == 0) ? pr : __fadd_rn(c2, pr);
      }
    }
    // leaf tree over the 8 chains
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      c1 = __fadd_rn(c1, __shfl_xor_sync(0xffffffffu, c1, o));
      c2 = __fadd_rn(c2, __shfl_xor_sync(0xffffffffu, c2, o));
    }
    // pairs / quads of leaves (only as many levels as leaves present)
    for (int o = 8; o < 8 * gl; o <<= 1) {
      c1 = __fadd_rn(c1, __shfl_xor_sync(0xffffffffu, c1, o));
      c2 = __fadd_rn(c2, __shfl_xor_sync(0xffffffffu, c2, o));
    }
    v1[it & 31] = c1;
    v2[it & 31] = c2;
  }
  // combine iteration values in tree (index) order: iters is a power of two
  for (int step = 1; step < iters; step <<= 1)
    for (int t = 0; t < iters; t += 2 * step) {
      v1[t] = __fadd_rn(v1[t], v1[t + step]);
      v2[t] = __fadd_rn(v2[t], v2[t + step]);
    }
  if (lane == 0) {
    m1[row] = __fdiv_rn(v1[0], (float)A.c);
    m2[row] = __fdiv_rn(v2[0], (float)A.c);
  }
}

// Leaf-per-lane path (perfect tree, nleaf | 32, leaf_len % 16 == 0 -- every
// hidden size used here).  The warp stages its rows' x and dY codes in shared
// memory with coalesced 16-byte loads (leaf stride leaf_len + 16 bytes: the
// leaf-per-lane 16-byte reads below are then bank-conflict free), then lane =
// (row, leaf) keeps all 8 chains of its leaf in registers and walks the leaf
// two chain elements per 16-byte read, in ascending order.  Leaf sum
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then an xor-butterfly over the row's
// nleaf lanes: numpy's pairwise association exactly.
__global__ void __launch_bounds__(256) ln_bwd_rows_leaf_kernel(LnRowArgs A, int nleaf, int leaf_len,
                                                               float *m1, float *m2) {
  extern __shared__ __align__(16) uint8_t lsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rpw = 32 / nleaf;
  const int stride = leaf_len + 16;                 // smem bytes per leaf
  const int row_bytes = nleaf * stride;             // smem bytes per row and array
  const int gstride = leaf_len + 4;                 // gamma: floats per leaf (padded)
  float *gsm = reinterpret_cast<float *>(lsm);      // [nleaf][gstride]
  uint8_t *wx = lsm + (size_t)nleaf * gstride * 4 + (size_t)warp * rpw * row_bytes * 2;
  uint8_t *wd = wx + (size_t)rpw * row_bytes;
  for (int q = threadIdx.x; q < (int)(A.c >> 2); q += blockDim.x) {  // gamma, once per CTA
    const int e = q * 4, lf = e / leaf_len;
    *reinterpret_cast<float4 *>(gsm + lf * gstride + (e - lf * leaf_len)) =
        __ldg(reinterpret_cast<const float4 *>(A.gamma) + q);
  }
  const int64_t row0 = ((int64_t)blockIdx.x * 8 + warp) * rpw;
  // stage: chunk q (16 bytes) of row r -> leaf (16q)/leaf_len, offset (16q)%leaf_len
  const int chunks = (int)(A.c >> 4);
  for (int r = 0; r < rpw; ++r) {
    const int64_t row = row0 + r;
    if (row >= A.n) break;
    const uint4 *gx = reinterpret_cast<const uint4 *>(A.x + row * A.c);
    const uint4 *gd = reinterpret_cast<const uint4 *>(A.dy + row * A.c);
    for (int q = lane; q < chunks; q += 32) {
      const int byte = q * 16, lf = byte / leaf_len;
      const int off = r * row_bytes + lf * stride + (byte - lf * leaf_len);
      *reinterpret_cast<uint4 *>(wx + off) = __ldg(gx + q);
      *reinterpret_cast<uint4 *>(wd + off) = __ldg(gd + q);
    }
  }
  __syncthreads();
  const int lr = lane / nleaf, leaf = lane % nleaf;
  const int64_t row = row0 + lr;
  const bool valid = row < A.n;
  float c1[8], c2[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) c1[j] = c2[j] = 0.f;
  if (valid) {
    const float mr = __ldg(A.mu + row), ir = __ldg(A.inv_std + row);
    const float zero = opaque_zero();
    const int64_t cb = A.c >> 5;
    const int64_t col0 = (int64_t)leaf * leaf_len;
    const uint8_t *sx_ = wx + lr * row_bytes + leaf * stride;
    const uint8_t *sd_ = wd + lr * row_bytes + leaf * stride;
    const float *sxr = A.xs + (row >> 5) * cb;
    const float *sdr = A.dys + (row >> 5) * cb;
    for (int seg = 0; seg < leaf_len / 16; ++seg) {
      const int64_t k0 = col0 + seg * 16;
      const uint4 xq = *reinterpret_cast<const uint4 *>(sx_ + seg * 16);
      const uint4 dq = *reinterpret_cast<const uint4 *>(sd_ + seg * 16);
      const DeqScale kx = deq_scale(__ldg(sxr + (k0 >> 5))), kd = deq_scale(__ldg(sdr + (k0 >> 5)));
      float g[16];
      const float *gl = gsm + leaf * gstride + seg * 16;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 g4 = *reinterpret_cast<const float4 *>(gl + 4 * q);
        g[4 * q] = g4.x;
        g[4 * q + 1] = g4.y;
        g[4 * q + 2] = g4.z;
        g[4 * q + 3] = g4.w;
      }
      const uint32_t xw[4] = {xq.x ^ 0x80808080u, xq.y ^ 0x80808080u, xq.z ^ 0x80808080u, xq.w ^ 0x80808080u};
      const uint32_t dw[4] = {dq.x ^ 0x80808080u, dq.y ^ 0x80808080u, dq.z ^ 0x80808080u, dq.w ^ 0x80808080u};
#pragma unroll
      for (int e = 0; e < 16; e += 2) {  // packed f32x2 pairs (chains j, j+1); same roundings
        float xv0, xv1, dv0, dv1, xh0, xh1, dh0, dh1, pr0, pr1;
        ffma2_rn(xv0, xv1, __uint_as_float(prmt_raw(xw[e >> 2], 0x4B000000u, 0x7404u | ((e & 3) << 4))),
                 __uint_as_float(prmt_raw(xw[e >> 2], 0x4B000000u, 0x7404u | (((e + 1) & 3) << 4))), kx.s8, kx.s8,
                 kx.c, kx.c);
        ffma2_rn(dv0, dv1, __uint_as_float(prmt_raw(dw[e >> 2], 0x4B000000u, 0x7404u | ((e & 3) << 4))),
                 __uint_as_float(prmt_raw(dw[e >> 2], 0x4B000000u, 0x7404u | (((e + 1) & 3) << 4))), kd.s8, kd.s8,
                 kd.c, kd.c);
        fsub2_rn(xh0, xh1, xv0, xv1, mr, mr);
        fmul2_rn(xh0, xh1, xh0, xh1, ir, ir);
        ffma2_rn(dh0, dh1, dv0, dv1, g[e], g[e + 1], zero, zero);  // rounded products (they feed adds)
        ffma2_rn(pr0, pr1, dh0, dh1, xh0, xh1, zero, zero);
        const int j = e & 7;
        if (seg == 0 && e < 8) {  // r[j] = a[j]: the chain starts at its first element
          c1[j] = dh0;
          c1[j + 1] = dh1;
          c2[j] = pr0;
          c2[j + 1] = pr1;
        } else {
          fadd2_rn(c1[j], c1[j + 1], c1[j], c1[j + 1], dh0, dh1);
          fadd2_rn(c2[j], c2[j + 1], c2[j], c2[j + 1], pr0, pr1);
        }
      }
    }
  }
  float s1 = __fadd_rn(__fadd_rn(__fadd_rn(c1[0], c1[1]), __fadd_rn(c1[2], c1[3])),
                       __fadd_rn(__fadd_rn(c1[4], c1[5]), __fadd_rn(c1[6], c1[7])));
  float s2 = __fadd_rn(__fadd_rn(__fadd_rn(c2[0], c2[1]), __fadd_rn(c2[2], c2[3])),
                       __fadd_rn(__fadd_rn(c2[4], c2[5]), __fadd_rn(c2[6], c2[7])));
  for (int o = 1; o < nleaf; o <<= 1) {
    s1 = __fadd_rn(s1, __shfl_xor_sync(0xffffffffu, s1, o));
    s2 = __fadd_rn(s2, __shfl_xor_sync(0xffffffffu, s2, o));
  }
  if (valid && leaf == 0) {
    m1[row] = __fdiv_rn(s1, (float)A.c);
    m2[row] = __fdiv_rn(s2, (float)A.c);
  }
}

__global__ void __launch_bounds__(256) ln_bwd_rows_kernel(LnRowArgs A, int depth, int perfect,
                                                          float *m1, float *m2) {
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= A.n) return;
  const float mr = __ldg(A.mu + row), ir = __ldg(A.inv_std + row);
  auto g1 = [&](int k) {
    float d, h;
    ln_row_vals(A, row, k, mr, ir, d, h);
    return d;
  };
  auto g2 = [&](int k) {
    float d, h;
    ln_row_vals(A, row, k, mr, ir, d, h);
    return __fmul_rn(d, h);
  };
  float s1 = 0.f, s2 = 0.f;
  if (perfect) {
    const int nleaf = 1 << depth;
    const int per = nleaf > 32 ? nleaf / 32 : 1;         // leaves per lane
    const int lanes = nleaf > 32 ? 32 : nleaf;
    if (lane < lanes) {
      // combine this lane's `per` consecutive leaves in tree order (per is 2^k)
      float acc1[8], acc2[8];  // per <= 8 supported (depth <= 8)
      for (int li = 0; li < per; ++li) {
        const int leaf = lane * per + li;
        int base = 0, len = (int)A.c;
        for (int lev = depth - 1; lev >= 0; --lev) {
          int h = len / 2;
          h -= h % 8;
          if ((leaf >> lev) & 1) {
            base += h;
            len -= h;
          } else {
            len = h;
          }
        }
        acc1[li] = pairwise_leaf(g1, base, len);
        acc2[li] = pairwise_leaf(g2, base, len);
      }
      for (int step = 1; step < per; step <<= 1)
        for (int li = 0; li < per; li += 2 * step) {
          acc1[li] = __fadd_rn(acc1[li], acc1[li + step]);
          acc2[li] = __fadd_rn(acc2[li], acc2[li + step]);
        }
      s1 = acc1[0];
      s2 = acc2[0];
    }
    for (int off = 1; off < lanes; off <<= 1) {
      s1 = __fadd_rn(s1, __shfl_xor_sync(0xffffffffu, s1, off));
      s2 = __fadd_rn(s2, __shfl_xor_sync(0xffffffffu, s2, off));
    }
  } else if (lane == 0) {
    s1 = pairwise_sum(g1, 0, (int)A.c);
    s2 = pairwise_sum(g2, 0, (int)A.c);
  }
  if (lane == 0) {
    m1[row] = __fdiv_rn(s1, (float)A.c);
    m2[row] = __fdiv_rn(s2, (float)A.c);
  }
}

// Pass B (32x256 tiles): dx = inv_std * ((dxhat - m1) - xhat*m2) -> requant,
// plus per-strip column partials of dgamma = sum(dy*xhat), dbeta = sum(dy).
template <bool kVec>
__global__ void __launch_bounds__(kTileThreads) ln_bwd_tile_kernel(
    LnRowArgs A, const float *__restrict__ m1, const float *__restrict__ m2, int8_t *dxq,
    float *dxs, float *part_g, float *part_b, int32_t *err) {
  __shared__ uint32_t red[64];
  __shared__ __align__(16) float colg[8][256], colb[8][256];
  const TilePos t = tile_pos(A.n, A.c);
  float xv[4][8], dv[4][8];
  load_deq(t, A.x, A.xs, xv);
  load_deq(t, A.dy, A.dys, dv);
  float pg[8], pb[8];
  if (t.active) {
    float g[8];
    ldg8<kVec>(A.gamma + t.col(), g);
#pragma unroll
    for (int j = 0; j < 8; ++j) pg[j] = pb[j] = 0.f;
    // the warp's 4 rows of each per-row vector: one broadcast 16-byte load each
    const int64_t r0 = t.row(0);
    float muv[4], isv[4], m1v[4], m2v[4];
    ldg4<kVec>(A.mu + r0, muv);
    ldg4<kVec>(A.inv_std + r0, isv);
    ldg4<kVec>(m1 + r0, m1v);
    ldg4<kVec>(m2 + r0, m2v);
    // packed f32x2, the reference's roundings in order; every product that feeds an
    // add is an FFMA2 with an opaque +0 (ptxas must not contract it)
    const float zero = opaque_zero();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float mr = muv[i], ir = isv[i], a1 = m1v[i], a2 = m2v[i];
#pragma unroll
      for (int j = 0; j < 8; j += 2) {
        float xh0, xh1, d0, d1, t0, t1, p0, p1;
        fsub2_rn(xh0, xh1, xv[i][j], xv[i][j + 1], mr, mr);
        fmul2_rn(xh0, xh1, xh0, xh1, ir, ir);                               // xhat
        ffma2_rn(d0, d1, dv[i][j], dv[i][j + 1], g[j], g[j + 1], zero, zero); // dxhat
        fsub2_rn(d0, d1, d0, d1, a1, a1);                                    // dxhat - m1
        ffma2_rn(t0, t1, xh0, xh1, a2, a2, zero, zero);                      // xhat * m2
        ffma2_rn(p0, p1, dv[i][j], dv[i][j + 1], xh0, xh1, zero, zero);      // dy * xhat
        if (i == 0) {
          pg[j] = p0;
          pg[j + 1] = p1;
          pb[j] = dv[i][j];
          pb[j + 1] = dv[i][j + 1];
        } else {
          fadd2_rn(pg[j], pg[j + 1], pg[j], pg[j + 1], p0, p1);
          fadd2_rn(pb[j], pb[j + 1], pb[j], pb[j + 1], dv[i][j], dv[i][j + 1]);
        }
        fsub2_rn(d0, d1, d0, d1, t0, t1);
        fmul2_rn(xv[i][j], xv[i][j + 1], ir, ir, d0, d1);  // reuse xv as dx
      }
    }
    float4 *cg4 = reinterpret_cast<float4 *>(&colg[t.warp][8 * t.lane]);
    float4 *cb4 = reinterpret_cast<float4 *>(&colb[t.warp][8 * t.lane]);
    cg4[0] = make_float4(pg[0], pg[1], pg[2], pg[3]);
    cg4[1] = make_float4(pg[4], pg[5], pg[6], pg[7]);
    cb4[0] = make_float4(pb[0], pb[1], pb[2], pb[3]);
    cb4[1] = make_float4(pb[4], pb[5], pb[6], pb[7]);
  }
  quant_store(t, xv, dxq, dxs, red, err);  // contains __syncthreads
  // rows in order: warp 0 rows 0..3, warp 1 rows 4..7, ... (sequential over warps)
  const int col = threadIdx.x;
  if (t.c0 + col < A.c) {
    float sg = colg[0][col], sb = colb[0][col];
#pragma unroll
    for (int w = 1; w < 8; ++w) {
      sg = __fadd_rn(sg, colg[w][col]);
      sb = __fadd_rn(sb, colb[w][col]);
    }
    part_g[(int64_t)blockIdx.y * A.c + t.c0 + col] = sg;
    part_b[(int64_t)blockIdx.y * A.c + t.c0 + col] = sb;
  }
}

// Sum per-strip partials: out[j] = sum_s part[s, j].  CTA = 32 columns x 8
// warps; warp w sums strips [w*S/8, (w+1)*S/8) in order (loads unrolled so
// they stay in flight), then the 8 warp sums are added in warp order.
__global__ void __launch_bounds__(512) strip_reduce_kernel(const float *__restrict__ part0,
                                                           const float *__restrict__ part1, int64_t strips,
                                                           int64_t c, float *out0, float *out1) {
  // blockIdx.y selects the array (LN backward reduces dgamma and dbeta in one launch);
  // 16 warps split the strips in order, then the 16 warp sums are added in warp order.
  __shared__ float ws[16][32];
  const float *part = blockIdx.y ? part1 : part0;
  float *out = blockIdx.y ? out1 : out0;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int64_t j = (int64_t)blockIdx.x * 32 + l;
  const int64_t s0 = strips * w / 16, s1 = strips * (w + 1) / 16;
  float acc = 0.f;
  if (j < c) {
    int64_t s = s0;
    for (; s + 8 <= s1; s += 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(part + (s + u) * c + j);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = __fadd_rn(acc, v[u]);
    }
    for (; s < s1; ++s) acc = __fadd_rn(acc, __ldg(part + s * c + j));
  }
  ws[w][l] = acc;
  __syncthreads();
  if (w == 0 && j < c) {
    float t = ws[0][l];
#pragma unroll
    for (int u = 1; u < 16; ++u) t = __fadd_rn(t, ws[u][l]);
    out[j] = t;
  }
}

// ── K11: dbias partials (qlayers.py:180) ───────────────────────────────
__global__ void __launch_bounds__(kTileThreads) colsum_tile_kernel(const int8_t *__restrict__ q,
                                                                   const float *__restrict__ s,
                                                                   int64_t n, int64_t c,
                                                                   float *part) {
  __shared__ float colp[8][256];
  const TilePos t = tile_pos(n, c);
  float v[4][8];
  load_deq(t, q, s, v);
  if (t.active) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float acc = v[0][j];
#pragma unroll
      for (int i = 1; i < 4; ++i) acc = __fadd_rn(acc, v[i][j]);
      colp[t.warp][8 * t.lane + j] = acc;
    }
  }
  __syncthreads();
  const int col = threadIdx.x;
  if (t.c0 + col < c) {
    float acc = colp[0][col];
#pragma unroll
    for (int w = 1; w < 8; ++w) acc = __fadd_rn(acc, colp[w][col]);
    part[(int64_t)blockIdx.y * c + t.c0 + col] = acc;
  }
}

// ── K9 / K10: GELU (qnonlinear.py:27-46, 150-175) ──────────────────────
// cdf(x) = fl(0.5 * fl(1 + fl32(erf_f64(fl(x * 0.70710677f)))))  — scipy's
// float32 erf is the double erf rounded (verified), so erf runs in FP64.
JF_DEV float norm_cdf_f32(float x) {
  const float z = __fmul_rn(x, 0.7071067811865476f);
  const float e = __double2float_rn(erf((double)z));
  return __fmul_rn(0.5f, __fadd_rn(1.0f, e));
}

// GELU input values are code * block_scale: a 32x32 block holds at most 255
// distinct values, so each tile first tabulates f(code) for its 8 blocks
// (8 x 255 evaluations of the FP64 erf instead of 8 x 1024) and every element
// then looks its result up — bit-identical to evaluating f per element.
JF_DEV void load_codes(const TilePos &t, const int8_t *__restrict__ q, int (&k)[4][8]) {
  if (!t.active) return;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint2 w = __ldg(reinterpret_cast<const uint2 *>(q + t.row(i) * t.c + t.col()));
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      k[i][j] = (int)(int8_t)((w.x >> (8 * j)) & 0xffu);
      k[i][4 + j] = (int)(int8_t)((w.y >> (8 * j)) & 0xffu);
    }
  }
}

// Global GELU tables: every block scale is a positive binary16 value, so all
// possible GELU inputs are code * s for s in the 31744 positive f16 values.
// Row (f16 bits of s) holds f(code * s) for code = -127..127 (+1 pad):
//   table 0: fl(x * cdf(x))            (gelu_forward, qnonlinear.py:150-158)
//   table 1: fl(fl(x * pdf) + cdf(x))  (gelu_grad_f32, qnonlinear.py:43-46)
// Built once per process (8M FP64 erf evaluations, ~ms); the kernels then do
// one L1-resident lookup per element — bit-identical to per-element math.
constexpr int kF16Rows = 0x7C00;  // positive finite binary16 bit patterns (incl. subnormals)

JF_DEV float gelu_val(float xv) { return __fmul_rn(xv, norm_cdf_f32(xv)); }
JF_DEV float gelu_grad(float xv) {
  const float ex = expf(__fmul_rn(__fmul_rn(-0.5f, xv), xv));
  const float pdf = __fmul_rn(0.3989422804014327f, ex);
  return __fadd_rn(__fmul_rn(xv, pdf), norm_cdf_f32(xv));
}

__global__ void __launch_bounds__(256) gelu_table_kernel(float *tab) {
  const int64_t total = (int64_t)kF16Rows * 256;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(e >> 8), k = (int)(e & 255);
    const float s = __half2float(__ushort_as_half((unsigned short)row));
    const float xv = __fmul_rn((float)(k - 127), s);
    tab[e] = k == 255 ? 0.f : gelu_val(xv);
    tab[total + e] = k == 255 ? 0.f : gelu_grad(xv);
  }
}

JF_DEV const float *gelu_row(const float *tab, float s) {
  return tab + ((int64_t)__half_as_ushort(__float2half_rn(s)) << 8) + 127;
}

// Copy the 8 table rows of this tile's 32x32 blocks (one per scale) into shared
// memory with coalesced 16-byte loads; the per-element lookups then gather from
// shared memory instead of L1 (a gather over up to 32 lines per warp load).
JF_DEV void stage_gelu_rows(const TilePos &t, const float *__restrict__ gtab,
                            const float *__restrict__ xs, float (*tab)[256]) {
  const int b = threadIdx.x >> 5, q0 = (threadIdx.x & 31) * 8;
  if (t.c0 + 32 * b < t.c) {
    const float *row = gelu_row(gtab, __ldg(xs + t.scale_idx(t.r0, t.c0 + 32 * b))) - 127;
    const float4 lo = __ldg(reinterpret_cast<const float4 *>(row + q0));
    const float4 hi = __ldg(reinterpret_cast<const float4 *>(row + q0) + 1);
    *reinterpret_cast<float4 *>(&tab[b][q0]) = lo;
    *reinterpret_cast<float4 *>(&tab[b][q0 + 4]) = hi;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kTileThreads) gelu_fwd_kernel(const int8_t *__restrict__ x,
                                                                const float *__restrict__ xs,
                                                                int64_t n, int64_t c, int8_t *yq,
                                                                float *ys, int32_t *err,
                                                                const float *__restrict__ gtab) {
  __shared__ uint32_t red[64];
  __shared__ float tab[8][256];  // tab[block][code + 127] = fl(x * cdf(x)), x = fl(code * s)
  const TilePos t = tile_pos(n, c);
  if (gtab != nullptr) {
    int k[4][8];
    float v[4][8];
    load_codes(t, x, k);
    stage_gelu_rows(t, gtab, xs, tab);
    if (t.active) {
      const float *tb = tab[t.lane >> 2] + 127;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) v[i][j] = tb[k[i][j]];
    }
    quant_store(t, v, yq, ys, red, err);
    return;
  }
  for (int e = threadIdx.x; e < 8 * 255; e += kTileThreads) {
    const int b = e / 255, q = e % 255 - 127;
    if (t.c0 + 32 * b < c) {
      tab[b][q + 127] = gelu_val(__fmul_rn((float)q, __ldg(xs + t.scale_idx(t.r0, t.c0 + 32 * b))));
    }
  }
  __syncthreads();
  int k[4][8];
  float v[4][8];
  load_codes(t, x, k);
  if (t.active) {
    const float *tb = tab[t.lane >> 2] + 127;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) v[i][j] = tb[k[i][j]];
  }
  quant_store(t, v, yq, ys, red, err);
}

// gelu'(x) = fl(fl(x * pdf) + cdf), pdf = fl(0.39894228f * exp(fl(fl(-0.5f*x)*x))).
// numpy's SIMD expf is not correctly rounded; expf here is (<=2 ulp) — the
// one documented tolerance-only op.
__global__ void __launch_bounds__(kTileThreads) gelu_bwd_kernel(
    const int8_t *__restrict__ x, const float *__restrict__ xs, const int8_t *__restrict__ dy,
    const float *__restrict__ dys, int64_t n, int64_t c, int8_t *dxq, float *dxs, int32_t *err,
    const float *__restrict__ gtab) {
  __shared__ uint32_t red[64];
  __shared__ float tab[8][256];  // tab[block][code + 127] = gelu'(fl(code * s_x))
  const TilePos t = tile_pos(n, c);
  if (gtab != nullptr) {
    int k[4][8];
    float d[4][8], v[4][8];
    load_codes(t, x, k);
    load_deq(t, dy, dys, d);
    if (t.active) {
      const float *tb = gelu_row(gtab + (int64_t)kF16Rows * 256, __ldg(xs + t.scale_idx(t.r0, t.col())));
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; j += 2)
          fmul2_rn(v[i][j], v[i][j + 1], d[i][j], d[i][j + 1], __ldg(tb + k[i][j]), __ldg(tb + k[i][j + 1]));
    }
    quant_store(t, v, dxq, dxs, red, err);
    return;
  }
  for (int e = threadIdx.x; e < 8 * 255; e += kTileThreads) {
    const int b = e / 255, q = e % 255 - 127;
    if (t.c0 + 32 * b < c) {
      tab[b][q + 127] = gelu_grad(__fmul_rn((float)q, __ldg(xs + t.scale_idx(t.r0, t.c0 + 32 * b))));
    }
  }
  __syncthreads();
  int k[4][8];
  float d[4][8], v[4][8];
  load_codes(t, x, k);
  load_deq(t, dy, dys, d);
  if (t.active) {
    const float *tb = tab[t.lane >> 2] + 127;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) v[i][j] = __fmul_rn(d[i][j], tb[k[i][j]]);
  }
  quant_store(t, v, dxq, dxs, red, err);
}

// ── Dropout by scale folding (qnonlinear.py:207-220) ───────────────────
__global__ void __launch_bounds__(256) dropout_kernel(const int8_t *__restrict__ q,
                                                      const float *__restrict__ s,
                                                      const uint8_t *__restrict__ keep,
                                                      float keep_factor, int64_t n, int64_t c,
                                                      int8_t *oq, float *os, int32_t *err) {
  const int64_t total = n * c / 16;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 w = reinterpret_cast<const uint4 *>(q)[i];
    const uint4 k = reinterpret_cast<const uint4 *>(keep)[i];
    const uint32_t wv[4] = {w.x, w.y, w.z, w.w}, kv[4] = {k.x, k.y, k.z, k.w};
    uint32_t o[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      uint32_t r = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if ((kv[b] >> (8 * e)) & 0xffu) r |= wv[b] & (0xffu << (8 * e));
      o[b] = r;
    }
    reinterpret_cast<uint4 *>(oq)[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
  const int64_t nb = (n >> 5) * (c >> 5);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nb;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = __half2float(__float2half_rn(__fmul_rn(s[i], keep_factor)));
    if (isinf(v)) raise_flags(err, JF_EFLAG_OVERFLOW);
    os[i] = v;
  }
}

// ── DropoutState.generate's keep mask on the device (qnonlinear.py:190-200) ──
// numpy's Generator(Philox(key=seed)).random(shape) >= p, bit for bit: Philox4x64-10
// (Random123), 128-bit counter starting at 1 for the first block of four outputs
// (numpy increments before generating), element i = word i % 4 of block i / 4 + 1,
// random() = (u64 >> 11) * 2^-53 in double precision.
JF_DEV void philox4x64_10(uint64_t (&c)[4], uint64_t k0, uint64_t k1) {
  constexpr uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B97F4A7C15ull;
      k1 += 0xBB67AE8584CAA73Bull;
    }
    const uint64_t lo0 = M0 * c[0], hi0 = __umul64hi(M0, c[0]);
    const uint64_t lo1 = M1 * c[2], hi1 = __umul64hi(M1, c[2]);
    const uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
  }
}

__global__ void __launch_bounds__(256) philox_keep_kernel(uint64_t k0, uint64_t k1, double p, int64_t total,
                                                          uint8_t *keep) {
  const int64_t groups = (total + 3) / 4;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < groups;
       g += (int64_t)gridDim.x * blockDim.x) {
    uint64_t c[4] = {(uint64_t)g + 1, 0, 0, 0};
    philox4x64_10(c, k0, k1);
    uint32_t w = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const double u = (double)(c[e] >> 11) * (1.0 / 9007199254740992.0);
      w |= (uint32_t)(u >= p) << (8 * e);
    }
    if (4 * g + 3 < total) {
      reinterpret_cast<uint32_t *>(keep)[g] = w;
    } else {
      for (int e = 0; 4 * g + e < total; ++e) keep[4 * g + e] = (w >> (8 * e)) & 1u;
    }
  }
}

}  // namespace jf

using namespace jf;
int jf_launch_check(const char *what);
int jf_set_smem_attr(const void *func, int bytes, const char *what);

static bool aligned16(const void *a, const void *b) {
  return ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0;
}

static bool ok_shape(int64_t n, int64_t c) { return n > 0 && c > 0 && n % 32 == 0 && c % 32 == 0; }

static int gcd_i(int a, int b) { return b ? gcd_i(b, a % b) : a; }

extern "C" int jf_add_stats(const int8_t *a, const float *as, const int8_t *b, const float *bs,
                            int64_t n, int64_t c, int64_t width, int8_t *yq, float *ys,
                            float *mean, float *sumsq, int32_t *err, jf_stream_t stream) {
  if (!ok_shape(n, c) || width <= 0 || c % width) return JF_ERR_ARG;
  const int w = (int)width;
  const int l = 32 / gcd_i(32, w) * w;  // lcm(32, width)
  if (l > kTileCols) return JF_ERR_UNSUPPORTED;
  const int tile_w = (kTileCols / l) * l;
  dim3 grid((unsigned)((c + tile_w - 1) / tile_w), (unsigned)(n / 32));
  const size_t smem = 32 * 257 * sizeof(float);
  if (int rc = jf_set_smem_attr((const void *)add_stats_kernel, (int)smem, "add_stats attr")) return rc;
  add_stats_kernel<<<grid, kTileThreads, smem, (cudaStream_t)stream>>>(
      a, as, b, bs, n, c, w, tile_w, yq, ys, mean, sumsq, err);
  return jf_launch_check("add_stats");
}

extern "C" int jf_ln_fwd(const int8_t *x, const float *xs, const float *mean, const float *sumsq,
                         int64_t n, int64_t c, int64_t width, const float *gamma,
                         const float *beta, float eps, int8_t *yq, float *ys, float *mu,
                         float *inv_std, int32_t *err, jf_stream_t stream) {
  if (!ok_shape(n, c) || width <= 0 || c % width) return JF_ERR_ARG;
  const int nb = (int)(c / width);
  ln_moments_kernel<<<(unsigned)((n + 31) / 32), 256, 0, (cudaStream_t)stream>>>(
      mean, sumsq, n, c, nb, eps, mu, inv_std);
  int rc = jf_launch_check("ln_moments");
  if (rc) return rc;
  const bool vec = aligned16(gamma, beta) && aligned16(mu, inv_std);
  auto kern = vec ? ln_fwd_kernel<true> : ln_fwd_kernel<false>;
  kern<<<tile_grid(n, c), kTileThreads, 0, (cudaStream_t)stream>>>(x, xs, mu, inv_std, gamma, beta, n, c,
                                                                   yq, ys, err);
  return jf_launch_check("ln_fwd");
}

// numpy pairwise tree of length c: perfect iff every leaf sits at one depth.
static int pw_depth(int64_t len) {
  if (len <= 128) return 0;
  int64_t h = len / 2;
  h -= h % 8;
  const int a = pw_depth(h), b = pw_depth(len - h);
  if (a < 0 || b < 0 || a != b) return -1;
  return a + 1;
}

// every leaf of the (perfect) tree has the same length
static bool pw_equal_leaves(int64_t len, int depth) {
  if (depth == 0) return true;
  int64_t h = len / 2;
  h -= h % 8;
  return h == len - h && pw_equal_leaves(h, depth - 1);
}

// A/B switch for the leaf-per-lane row reduction (default on; JF_LN_LEAF=0 disables).
static bool g_ln_leaf = [] {
  const char *e = getenv("JF_LN_LEAF");
  return !(e && e[0] == '0');
}();

extern "C" size_t jf_ln_bwd_workspace_bytes(int64_t n, int64_t c) {
  return (size_t)(2 * n + 2 * (n / 32) * c) * sizeof(float);
}

extern "C" int jf_ln_bwd(const int8_t *x, const float *xs, const float *mu, const float *inv_std,
                         const int8_t *dy, const float *dys, const float *gamma, int64_t n,
                         int64_t c, int8_t *dxq, float *dxs, float *dgamma, float *dbeta,
                         void *workspace, int32_t *err, jf_stream_t stream) {
  if (!ok_shape(n, c)) return JF_ERR_ARG;
  float *ws = static_cast<float *>(workspace);
  float *m1 = ws, *m2 = ws + n, *pg = ws + 2 * n, *pb = pg + (n / 32) * c;
  LnRowArgs A{x, xs, mu, inv_std, dy, dys, gamma, n, c};
  int depth = pw_depth(c);
  int perfect = depth >= 0 && depth <= 8;
  if (!perfect) depth = 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t leaf_len = perfect ? (c >> depth) : 0;
  const bool fast = perfect && depth <= 7 && (leaf_len << depth) == c && leaf_len % 8 == 0 &&
                    pw_equal_leaves(c, depth) && ((1 << depth) <= 4 || true);
  const int nleaf = 1 << depth;
  const bool leafp = fast && nleaf <= 32 && leaf_len % 16 == 0 && ((uintptr_t)x % 16 == 0) &&
                     ((uintptr_t)dy % 16 == 0) && ((uintptr_t)gamma % 16 == 0) && g_ln_leaf;
  // staged rows: 8 warps x (32/nleaf) rows x 2 arrays x nleaf x (leaf_len + 16) bytes
  const size_t leaf_smem = leafp ? (size_t)8 * 32 * 2 * (leaf_len + 16) + (size_t)nleaf * (leaf_len + 4) * 4 : 0;
  if (leafp && leaf_smem <= 200 * 1024) {
    if (leaf_smem > 48 * 1024)
      if (int rc = jf_set_smem_attr((const void *)ln_bwd_rows_leaf_kernel, 200 * 1024, "ln_bwd attr")) return rc;
    const int64_t rows_per_cta = 8 * (32 / nleaf);
    ln_bwd_rows_leaf_kernel<<<(unsigned)((n + rows_per_cta - 1) / rows_per_cta), 256, leaf_smem, st>>>(
        A, nleaf, (int)leaf_len, m1, m2);
  } else if (fast)
    ln_bwd_rows_fast_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(A, 1 << depth, (int)leaf_len, m1, m2);
  else
    ln_bwd_rows_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(A, depth, perfect, m1, m2);
  int rc = jf_launch_check("ln_bwd_rows");
  if (rc) return rc;
  const bool vec = aligned16(gamma, ws) && aligned16(mu, inv_std);
  auto tk = vec ? ln_bwd_tile_kernel<true> : ln_bwd_tile_kernel<false>;
  tk<<<tile_grid(n, c), kTileThreads, 0, st>>>(A, m1, m2, dxq, dxs, pg, pb, err);
  rc = jf_launch_check("ln_bwd_tile");
  if (rc) return rc;
  const unsigned g = (unsigned)((c + 31) / 32);
  strip_reduce_kernel<<<dim3(g, 2), 512, 0, st>>>(pg, pb, n / 32, c, dgamma, dbeta);
  return jf_launch_check("ln_bwd_reduce");
}

extern "C" size_t jf_colsum_workspace_bytes(int64_t n, int64_t c) {
  return (size_t)((n / 32) * c) * sizeof(float);
}

extern "C" int jf_colsum(const int8_t *q, const float *s, int64_t n, int64_t c, float *out,
                         void *workspace, jf_stream_t stream) {
  if (!ok_shape(n, c)) return JF_ERR_ARG;
  float *part = static_cast<float *>(workspace);
  cudaStream_t st = (cudaStream_t)stream;
  colsum_tile_kernel<<<tile_grid(n, c), kTileThreads, 0, st>>>(q, s, n, c, part);
  int rc = jf_launch_check("colsum_tile");
  if (rc) return rc;
  strip_reduce_kernel<<<dim3((unsigned)((c + 31) / 32), 1), 512, 0, st>>>(part, part, n / 32, c, out, out);
  return jf_launch_check("colsum_reduce");
}

extern "C" size_t jf_gelu_tables_bytes(void) { return (size_t)2 * kF16Rows * 256 * sizeof(float); }

extern "C" int jf_gelu_build_tables(float *tables, jf_stream_t stream) {
  gelu_table_kernel<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(tables);
  return jf_launch_check("gelu_tables");
}

extern "C" int jf_gelu_fwd(const int8_t *x, const float *xs, int64_t n, int64_t c, int8_t *yq,
                           float *ys, const float *tables, int32_t *err, jf_stream_t stream) {
  if (!ok_shape(n, c)) return JF_ERR_ARG;
  gelu_fwd_kernel<<<tile_grid(n, c), kTileThreads, 0, (cudaStream_t)stream>>>(x, xs, n, c, yq, ys,
                                                                              err, tables);
  return jf_launch_check("gelu_fwd");
}

extern "C" int jf_gelu_bwd(const int8_t *x, const float *xs, const int8_t *dy, const float *dys,
                           int64_t n, int64_t c, int8_t *dxq, float *dxs, const float *tables,
                           int32_t *err, jf_stream_t stream) {
  if (!ok_shape(n, c)) return JF_ERR_ARG;
  gelu_bwd_kernel<<<tile_grid(n, c), kTileThreads, 0, (cudaStream_t)stream>>>(x, xs, dy, dys, n,
                                                                              c, dxq, dxs, err, tables);
  return jf_launch_check("gelu_bwd");
}

extern "C" int jf_philox_keep(uint64_t key0, uint64_t key1, double p, int64_t total, uint8_t *keep,
                              jf_stream_t stream) {
  if (total <= 0 || !(p >= 0.0 && p < 1.0)) return JF_ERR_ARG;
  const int64_t groups = (total + 3) / 4;
  const int blocks = (int)std::min<int64_t>((groups + 255) / 256, 148 * 16);
  philox_keep_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(key0, key1, p, total, keep);
  return jf_launch_check("philox_keep");
}

extern "C" int jf_dropout(const int8_t *q, const float *s, const uint8_t *keep, float keep_factor,
                          int64_t n, int64_t c, int8_t *oq, float *os, int32_t *err,
                          jf_stream_t stream) {
  if (!ok_shape(n, c)) return JF_ERR_ARG;
  int64_t th = n * c / 16;
  unsigned blocks = (unsigned)((th + 255) / 256 < 148 * 8 ? (th + 255) / 256 : 148 * 8);
  dropout_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(q, s, keep, keep_factor, n, c, oq, os,
                                                           err);
  return jf_launch_check("dropout");
}
