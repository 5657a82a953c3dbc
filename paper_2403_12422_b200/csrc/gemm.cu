// gemm.cu — K3/K4/K5: the per-block INT8 GEMM on tcgen05 (sm_100a).
//
// Y[M x N] = sum over 32-deep K chunks ci (ascending) of
//            sA(I, ci) * sB(ci, J) * P_ci,   P_ci = A[:, 32ci:+32] . B[32ci:+32, :]
// exactly as qgemm.py:193-229 (_mm_core / _scaled_accumulate), then +bias and
// a 32x32 block requantization (qgemm.py:266-279).
//
// Design (one persistent CTA per SM, warp-specialized):
//   warp 0      TMA producer: 128x128-byte tiles of A and B (K-major, SW128)
//               into a 4-stage smem ring (4 K chunks per stage).
//   warp 1      TMEM owner + MMA issuer: one tcgen05.mma.kind::i8 (M=128,
//               N=128, K=32) per K chunk into one of 4 TMEM int32 buffers;
//               every chunk is a fresh product (accumulate=0), because the
//               reference promotes each 32-deep partial separately.
//   warps 2-17  promotion/epilogue: 4 warpgroups x 32 columns.  Each thread
//               owns one row x 32 columns of the FP32 accumulator in
//               registers; per chunk it tcgen05.ld's its int32 partials,
//               frees the TMEM buffer, and promotes:
//                 EXACT: acc = fl(acc + fl(fl(P*sa)*sb))   (bit-exact)
//                 FAST : acc = fma(P, sa*sb, acc)          (sa*sb exact)
//               After the last chunk: +bias, 32x32 absmax (warp = 32 rows),
//               binary16 scale, RNE codes, store INT8 + scale.
// The promotion (one FP32 op chain per output per 32 MACs) is what bounds
// this kernel on B200 — see DESIGN.md §GEMM roofline.
#include "common.cuh"

namespace jf {
namespace gemm {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int BK = 128;  // bytes of K per stage (4 chunks)
constexpr int kStages = 4;
constexpr int kChunksPerStage = BK / 32;
constexpr int kTmemBufs = 4;
constexpr int kEpiWarps = 16;
constexpr int kCtrlWarps = 2;  // TMA warp + MMA warp; epilogue warps use lane quarter warp%4
constexpr int kThreads = (kCtrlWarps + kEpiWarps) * 32;
constexpr uint32_t kStageBytesA = BM * BK;
constexpr uint32_t kStageBytesB = BN * BK;

enum OutKind { OUT_INT8 = 0, OUT_F32 = 1, OUT_INT8_DEQ = 2, OUT_I32 = 3 };

struct Params {
  int64_t M, N, K;
  const float *sa;
  int64_t sa_s0, sa_s1;  // sA(I, ci) = sa[I*s0 + ci*s1]
  const float *sb;
  int64_t sb_s0, sb_s1;  // sB(ci, J) = sb[J*s0 + ci*s1]
  const float *bias;     // [N] or nullptr
  int8_t *yq;
  float *ys;
  float *yf;   // FP32 output (OUT_F32 / OUT_INT8_DEQ) — int32 for OUT_I32
  int32_t *err;
  int out_kind;
  float zero;  // always 0.0f; opaque to ptxas (blocks FMUL2+FADD2 contraction)
};

struct Smem {
  uint64_t full[kStages];
  uint64_t empty[kStages];
  uint64_t tfull[kTmemBufs];
  uint64_t tempty[kTmemBufs];
  uint32_t tmem_base;
};

constexpr size_t kSmemBytes = 1024 /*align slack*/ + kStages * (kStageBytesA + kStageBytesB) + 256;

template <bool kFast>
__global__ void __maxnreg__(96)
    gemm_i8_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *base = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sA = base;
  uint8_t *sB = base + kStages * kStageBytesA;
  Smem &S = *reinterpret_cast<Smem *>(sB + kStages * kStageBytesB);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t mt = (p.M + BM - 1) / BM, nt = (p.N + BN - 1) / BN;
  const int64_t ntiles = mt * nt;
  const int nchunks = (int)(p.K / 32);
  const int nstages_k = (nchunks + kChunksPerStage - 1) / kChunksPerStage;

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], 1);
    }
    for (int b = 0; b < kTmemBufs; ++b) {
      mbar_init(&S.tfull[b], 1);
      mbar_init(&S.tempty[b], kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&S.tmem_base, kTmemBufs * BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;

  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp == 0) {
    // ───────────── TMA producer ─────────────
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int m0 = (int)((tile % mt) * BM), n0 = (int)((tile / mt) * BN);
        for (int ks = 0; ks < nstages_k; ++ks) {
          mbar_wait(&S.empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&S.full[stage], kStageBytesA + kStageBytesB);
          tma_load_2d(sA + stage * kStageBytesA, &tmA, &S.full[stage], ks * BK, m0);
          tma_load_2d(sB + stage * kStageBytesB, &tmB, &S.full[stage], ks * BK, n0);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ───────────── MMA issuer ─────────────
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_i8(BM, BN, 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t g = 0;  // global chunk counter (TMEM ring position)
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int ks = 0; ks < nstages_k; ++ks) {
          mbar_wait(&S.full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * kStageBytesA);
          const uint32_t b0 = smem_u32(sB + stage * kStageBytesB);
          const int nch = min(kChunksPerStage, nchunks - ks * kChunksPerStage);
          for (int c = 0; c < nch; ++c, ++g) {
            const uint32_t buf = g % kTmemBufs;
            mbar_wait(&S.tempty[buf], ((g / kTmemBufs) & 1) ^ 1);
            tc_fence_after();
            const uint64_t ad = smem_desc_sw128(a0 + c * 32, 16, 1024);
            const uint64_t bd = smem_desc_sw128(b0 + c * 32, 16, 1024);
            mma_i8_ss(tmem + buf * BN, ad, bd, idesc, 0u);  // fresh int32 partial per chunk
            mma_commit(&S.tfull[buf]);
          }
          mma_commit(&S.empty[stage]);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp >= kCtrlWarps) {
    // ───────────── promotion + epilogue ─────────────
    const int lq = warp & 3;                   // TMEM lane quarter == row block in tile
    const int cg = (warp - kCtrlWarps) >> 2;   // 32-column group
    const uint32_t t_lane = (uint32_t)(lq * 32) << 16;
    uint32_t g = 0;
    int flags = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t I = (tile % mt) * (BM / 32) + lq;  // 32-row block index
      const int64_t J = (tile / mt) * (BN / 32) + cg;  // 32-col block index
      const bool valid = (I * 32 < p.M) && (J * 32 < p.N);
      const bool scaled = valid && p.out_kind != OUT_I32;
      const float *pa = scaled ? p.sa + I * p.sa_s0 : nullptr;
      const float *pb = scaled ? p.sb + J * p.sb_s0 : nullptr;
      float acc[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = 0.0f;
      float sa_n = scaled ? __ldg(pa) : 0.f, sb_n = scaled ? __ldg(pb) : 0.f;
      uint32_t r[32];
      for (int ci = 0; ci < nchunks; ++ci, ++g) {
        const float sa = sa_n, sb = sb_n;
        if (scaled && ci + 1 < nchunks) {  // prefetch next chunk's scales
          sa_n = __ldg(pa + (ci + 1) * p.sa_s1);
          sb_n = __ldg(pb + (ci + 1) * p.sb_s1);
        }
        const uint32_t buf = g % kTmemBufs;
        mbar_wait(&S.tfull[buf], (g / kTmemBufs) & 1);
        tc_fence_after();
        const uint32_t taddr = tmem + t_lane + buf * BN + cg * 32;
        tmem_ld_32x32b_x32(taddr, r);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.tempty[buf]);
        if (p.out_kind == OUT_I32) {
          // debug: raw int32 partial of the (single) chunk
          if (valid) {
            int32_t *dst = reinterpret_cast<int32_t *>(p.yf) + (I * 32 + lane) * p.N + J * 32;
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              *reinterpret_cast<int4 *>(dst + j) =
                  make_int4((int)r[j], (int)r[j + 1], (int)r[j + 2], (int)r[j + 3]);
          }
          continue;
        }
        if (kFast) {
          const float s = __fmul_rn(sa, sb);  // exact: 11 x 11 significant bits
#pragma unroll
          for (int j = 0; j < 32; j += 2)
            ffma2_rn(acc[j], acc[j + 1], __int2float_rn((int)r[j]), __int2float_rn((int)r[j + 1]), s, s,
                     acc[j], acc[j + 1]);
        } else {
          // packed f32x2, every op an IEEE-rounded fp32 op in the reference order.
          // ptxas contracts mul.rn.f32x2 + add.rn.f32x2 into FFMA2 (not equivalent);
          // an fma with a runtime +0 addend is a correctly rounded product it cannot fuse.
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            float t0, t1;
            fmul2_rn(t0, t1, __int2float_rn((int)r[j]), __int2float_rn((int)r[j + 1]), sa, sa);
            ffma2_rn(t0, t1, t0, t1, sb, sb, p.zero, p.zero);
            fadd2_rn(acc[j], acc[j + 1], acc[j], acc[j + 1], t0, t1);
          }
        }
      }
      if (!valid || p.out_kind == OUT_I32) continue;
      // ── epilogue: bias, requantization, stores ──
      const int64_t row = I * 32 + lane;
      const int64_t col0 = J * 32;
      if (p.bias != nullptr) {
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = __fadd_rn(acc[j], __ldg(p.bias + col0 + j));
      }
      if (p.out_kind == OUT_F32) {
        float *dst = p.yf + row * p.N + col0;
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4 *>(dst + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
        continue;
      }
      uint32_t m = 0;
#pragma unroll
      for (int j = 0; j < 32; ++j) m = max(m, abs_bits(acc[j]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
      int f = 0;
      const float sc = block_scale(m, f);
      uint32_t w[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        w[k] = pack4(quant_code(acc[4 * k], sc), quant_code(acc[4 * k + 1], sc),
                     quant_code(acc[4 * k + 2], sc), quant_code(acc[4 * k + 3], sc));
      int8_t *dq = p.yq + row * p.N + col0;
      reinterpret_cast<uint4 *>(dq)[0] = make_uint4(w[0], w[1], w[2], w[3]);
      reinterpret_cast<uint4 *>(dq)[1] = make_uint4(w[4], w[5], w[6], w[7]);
      if (lane == 0) {
        p.ys[I * (p.N >> 5) + J] = sc;
        flags |= f;
      }
      if (p.out_kind == OUT_INT8_DEQ) {
        float *dst = p.yf + row * p.N + col0;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          *reinterpret_cast<float4 *>(dst + 4 * k) =
              make_float4(__fmul_rn(code_at(w[k], 0), sc), __fmul_rn(code_at(w[k], 1), sc),
                          __fmul_rn(code_at(w[k], 2), sc), __fmul_rn(code_at(w[k], 3), sc));
      }
    }
    if (lane == 0) raise_flags(p.err, flags);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, kTmemBufs * BN);
}

}  // namespace gemm
}  // namespace jf

// ─────────────────────────── host side ───────────────────────────
using namespace jf;

int jf_launch_check(const char *what);
void jf_set_error(const char *msg);
int jf_num_sms();
bool jf_make_tmap_i8(CUtensorMap *map, const void *ptr, int64_t rows, int64_t cols, int64_t ld,
                     int box_cols, int box_rows);

// Core launcher: A [M x K] (row stride lda), Bt [N x K] (row stride ldb), both K-major codes.
int jf_gemm_launch(const int8_t *A, int64_t lda, const int8_t *Bt, int64_t ldb, int64_t M,
                   int64_t N, int64_t K, const float *sa, int64_t sa_s0, int64_t sa_s1,
                   const float *sb, int64_t sb_s0, int64_t sb_s1, const float *bias, int mode,
                   int out_kind, int8_t *yq, float *ys, void *yf, int32_t *err,
                   cudaStream_t stream) {
  using namespace jf::gemm;
  if (M <= 0 || N <= 0 || K <= 0 || M % 32 || N % 32 || K % 32 || lda % 16 || ldb % 16) {
    jf_set_error("gemm: dims must be positive multiples of 32, strides multiples of 16");
    return JF_ERR_ARG;
  }
  CUtensorMap ta, tb;
  if (!jf_make_tmap_i8(&ta, A, M, K, lda, BK, BM) || !jf_make_tmap_i8(&tb, Bt, N, K, ldb, BK, BN))
    return JF_ERR_LAUNCH;
  Params p{M, N, K, sa, sa_s0, sa_s1, sb, sb_s0, sb_s1, bias, yq, ys, (float *)yf, err, out_kind, 0.0f};
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int grid = (int)(tiles < jf_num_sms() ? tiles : jf_num_sms());
  const bool fast = mode == JF_MODE_FAST;
  auto kern = fast ? gemm_i8_kernel<true> : gemm_i8_kernel<false>;
  static bool attr_done[2] = {false, false};
  const int ki = fast ? 1 : 0;
  if (!attr_done[ki]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes) !=
        cudaSuccess)
      return jf_launch_check("gemm attr");
    attr_done[ki] = true;
  }
  kern<<<grid, kThreads, kSmemBytes, stream>>>(ta, tb, p);
  return jf_launch_check("gemm_i8");
}

extern "C" int jf_gemm_fwd(const int8_t *x, const float *xs, const int8_t *w, const float *ws,
                           const float *bias, int64_t n, int64_t c, int64_t d, int32_t mode,
                           int32_t out_kind, int8_t *yq, float *ys, float *yf, int32_t *err,
                           jf_stream_t stream) {
  const int64_t cb = c / 32;
  return jf_gemm_launch(x, c, w, c, n, d, c, xs, cb, 1, ws, cb, 1, bias, mode, out_kind, yq, ys,
                        yf, err, (cudaStream_t)stream);
}

extern "C" size_t jf_gemm_scratch_bytes(int32_t which, int64_t n, int64_t d, int64_t c) {
  if (which == 1) return (size_t)(c * d);
  return (size_t)(n * d + n * c);
}

extern "C" int jf_gemm_dgrad(const int8_t *dy, const float *dys, const int8_t *w, const float *ws,
                             const int8_t *wt, const float *wts, int64_t n, int64_t d, int64_t c,
                             int32_t mode, int32_t out_kind, int8_t *dxq, float *dxs, float *dxf,
                             void *scratch, int32_t *err, jf_stream_t stream) {
  (void)wts;
  if (wt == nullptr) {
    if (scratch == nullptr) return JF_ERR_ARG;
    int8_t *t = static_cast<int8_t *>(scratch);
    int rc = jf_transpose(w, nullptr, d, c, t, nullptr, stream);
    if (rc) return rc;
    wt = t;
  }
  // A = dY [n x d] (K = d), Bt = W^T [c x d]; sB(ci, J) = W.scales[ci, J]
  return jf_gemm_launch(dy, d, wt, d, n, c, d, dys, d / 32, 1, ws, 1, c / 32, nullptr, mode,
                        out_kind, dxq, dxs, dxf, err, (cudaStream_t)stream);
}

extern "C" int jf_gemm_wgrad(const int8_t *dy, const float *dys, const int8_t *x, const float *xs,
                             const int8_t *dyt, const int8_t *xt, int64_t n, int64_t d, int64_t c,
                             int32_t mode, int32_t out_kind, int8_t *dwq, float *dws, float *dwf,
                             void *scratch, int32_t *err, jf_stream_t stream) {
  int8_t *s8 = static_cast<int8_t *>(scratch);
  if (dyt == nullptr) {
    if (scratch == nullptr) return JF_ERR_ARG;
    int rc = jf_transpose(dy, nullptr, n, d, s8, nullptr, stream);  // [d x n]
    if (rc) return rc;
    dyt = s8;
  }
  if (xt == nullptr) {
    if (scratch == nullptr) return JF_ERR_ARG;
    int8_t *t = s8 + n * d;
    int rc = jf_transpose(x, nullptr, n, c, t, nullptr, stream);  // [c x n]
    if (rc) return rc;
    xt = t;
  }
  // A = dY^T [d x n] (K = n): sA(I, ci) = dY.scales[ci, I]; Bt = X^T [c x n]: sB(ci, J) = X.scales[ci, J]
  return jf_gemm_launch(dyt, n, xt, n, d, c, n, dys, 1, d / 32, xs, 1, c / 32, nullptr, mode,
                        out_kind, dwq, dws, dwf, err, (cudaStream_t)stream);
}

extern "C" int jf_gemm_partials(const int8_t *a, const int8_t *bt, int64_t m, int64_t n,
                                int64_t k, int64_t kblk, int32_t *out, jf_stream_t stream) {
  if (kblk < 0 || kblk * 32 >= k) return JF_ERR_ARG;
  // K restricted to one chunk via pointer offset + row stride = k
  return jf_gemm_launch(a + kblk * 32, k, bt + kblk * 32, k, m, n, 32, nullptr, 0, 0, nullptr, 0,
                        0, nullptr, JF_MODE_EXACT, jf::gemm::OUT_I32, nullptr, nullptr, out,
                        nullptr, (cudaStream_t)stream);
}
