// gemm.cu — K3/K4/K5: the per-block INT8 GEMM on tcgen05 (sm_100a).
//
// Y[M x N] = sum over 32-deep K chunks ci (ascending) of
//            sA(I, ci) * sB(ci, J) * P_ci,   P_ci = A[:, 32ci:+32] . B[32ci:+32, :]
// exactly as qgemm.py:193-229 (_mm_core / _scaled_accumulate), then +bias and
// a 32x32 block requantization (qgemm.py:266-279).
//
// Design (one persistent CTA per SM, warp-specialized, 128x128 output tiles):
//   warp 0        TMA producer: 128x128-byte K-major SW128 tiles of A and B
//                 into a 6-stage smem ring (4 K chunks per stage).
//   warp 1        MMA issuer: one tcgen05.mma.kind::i8 (M=128, N=128, K=32)
//                 per K chunk into TMEM buffer (chunk % 4), accumulate = 0:
//                 every chunk is a fresh int32 partial because the reference
//                 promotes each 32-deep product separately.
//   warps 2..17   promotion/epilogue (16 warps, 32 columns each; TMEM lane
//                 quarter = warp % 4).  Per chunk a thread tcgen05.ld's its 32
//                 int32 partials, frees the buffer, and promotes in packed
//                 f32x2 ops:
//                   EXACT: acc = fl(acc + fl(fl(P*sa)*sb))   (bit-exact)
//                   FAST : acc = fma(P, sa*sb, acc)          (sa*sb exact)
//                 After the last chunk: +bias, 32x32 absmax (warp = 32 rows),
//                 binary16 scale, RNE codes, INT8 + scale stores.
// Bound: per output element per 32 MACs the promotion
// costs one I2F (ALU pipe, half rate) and 3 (exact) / 1 (fast) FP32 ops; at
// 128 FP32 ops/clk/SM exact mode cannot beat 384 clk per 128x128x32 chunk
// (16.7% of the 64-clk tensor rate), fast mode is held to 256 clk by I2F.
// Variants measured A/B in one session (mlp1 fwd, 4096x16384x4096, exact):
// this per-chunk hand-off 1294 us; chunk pairs per barrier 1345 us; MMA issue
// folded into a promotion warp 1842 us; 8 promotion warps x 64 columns 1406
// us; 3 MMA issuers 1318 us; "phase" issue (4 MMAs after all 4 buffers
// drain) 1356 us.  The remaining gap to the 403-clk/chunk standalone
// promotion loop (profiles/r1e_microbench.jsonl) is sub-partition skew: the
// four sub-partitions each serve one TMEM lane quarter, the buffer release
// waits for the slowest, and the one hosting the MMA issuer lags.
#include <stdio.h>
#include <string.h>

#include "common.cuh"

namespace jf {
namespace gemm {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int BK = 128;  // bytes of K per stage (4 chunks)
constexpr int kStages = 6;
constexpr int kChunksPerStage = BK / 32;
constexpr int kTmemBufs = 4;  // == kChunksPerStage: chunk c of a stage uses buffer c
constexpr int kEpiWarps = 16;  // promotion warps (kind::f16 path)
constexpr int kPairSlots = 2;  // kind::f16 path: 2 slots x 2 chunk buffers x 128 f32 columns
constexpr int kTmemCols = kPairSlots * 2 * BN;
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
  long long *trace;  // JF_GEMM_TRACE builds only (f16 path): CTA 0 event clocks [8][512]
  int ctl_kind;      // control-thread waits: 0 spin, 1 try_wait with suspend hint, 2 test + nanosleep
  uint32_t ctl_ns;
};

// mbarrier wait used by the single-thread TMA producer and MMA issuer.
JF_DEV void ctl_wait(const Params &p, uint32_t addr, uint32_t parity) {
#ifdef JF_CTL_RUNTIME
  if (p.ctl_kind == 1) {
    mbar_wait_u32_sleep(addr, parity, p.ctl_ns);
  } else if (p.ctl_kind == 2) {
    while (!mbar_test_u32(addr, parity)) __nanosleep(p.ctl_ns);
  } else {
    mbar_wait_u32(addr, parity);
  }
#else
  // One flavour, compiled in: the control loops stay small enough to share the
  // sub-partition's L0 instruction cache with the promotion loop (a runtime
  // switch between three wait loops at every call site measured 9% slower).
  mbar_wait_u32_sleep(addr, parity, 200);
#endif
}

struct Smem {
  uint64_t full[kStages];
  uint64_t empty[kStages];
  uint64_t tfull[kTmemBufs];
  uint64_t tempty[kTmemBufs];
  uint32_t tmem_base;
};

constexpr size_t kSmemBytes = 1024 /*align slack*/ + kStages * (kStageBytesA + kStageBytesB) + 256;

// Promote one 32-column block of int32 partials into the FP32 accumulator.
template <bool kFast>
JF_DEV void promote32(float *acc, const uint32_t *r, float sa, float sb, float zero) {
  if (kFast) {
    const float s = __fmul_rn(sa, sb);  // exact: 11 x 11 significant bits
#pragma unroll
    for (int j = 0; j < 32; j += 2)
      ffma2_rn(acc[j], acc[j + 1], __int2float_rn((int)r[j]), __int2float_rn((int)r[j + 1]), s, s, acc[j],
               acc[j + 1]);
  } else {
    // packed f32x2, every op an IEEE-rounded fp32 op in the reference order.
    // ptxas contracts mul.rn.f32x2 + add.rn.f32x2 into FFMA2 (not equivalent);
    // an fma with a runtime +0 addend is a correctly rounded product it cannot fuse.
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
      float t0, t1;
      fmul2_rn(t0, t1, __int2float_rn((int)r[j]), __int2float_rn((int)r[j + 1]), sa, sa);
      ffma2_rn(t0, t1, t0, t1, sb, sb, zero, zero);
      fadd2_rn(acc[j], acc[j + 1], acc[j], acc[j + 1], t0, t1);
    }
  }
}

// Same, for f32 partials that hold exact integers (kind::f16 path: no I2F).
template <bool kFast>
JF_DEV void promote32f(float *acc, const uint32_t *r, float sa, float sb, float zero) {
  if (kFast) {
    const float s = __fmul_rn(sa, sb);
#pragma unroll
    for (int j = 0; j < 32; j += 2)
      ffma2_rn(acc[j], acc[j + 1], __uint_as_float(r[j]), __uint_as_float(r[j + 1]), s, s, acc[j], acc[j + 1]);
  } else {
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
      float t0, t1;
      fmul2_rn(t0, t1, __uint_as_float(r[j]), __uint_as_float(r[j + 1]), sa, sa);
      ffma2_rn(t0, t1, t0, t1, sb, sb, zero, zero);
      fadd2_rn(acc[j], acc[j + 1], acc[j], acc[j + 1], t0, t1);
    }
  }
}

// +bias, 32x32 requantization (warp = 32 rows), stores.  Returns error flags.
JF_DEV int finish_block(const Params &p, float *acc, int64_t I, int64_t J, int lane) {
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
    return 0;
  }
  uint32_t m = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) m = max(m, abs_bits(acc[j]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  int f = 0;
  const float sc = block_scale(m, f);
  const float rc = __frcp_rn(sc);
  uint32_t w[8];
#pragma unroll
  for (int k = 0; k < 8; ++k)
    w[k] = pack4(quant_code_fast(acc[4 * k], sc, rc), quant_code_fast(acc[4 * k + 1], sc, rc),
                 quant_code_fast(acc[4 * k + 2], sc, rc), quant_code_fast(acc[4 * k + 3], sc, rc));
  int8_t *dq = p.yq + row * p.N + col0;
  reinterpret_cast<uint4 *>(dq)[0] = make_uint4(w[0], w[1], w[2], w[3]);
  reinterpret_cast<uint4 *>(dq)[1] = make_uint4(w[4], w[5], w[6], w[7]);
  if (lane == 0) p.ys[I * (p.N >> 5) + J] = sc;
  if (p.out_kind == OUT_INT8_DEQ) {
    float *dst = p.yf + row * p.N + col0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      *reinterpret_cast<float4 *>(dst + 4 * k) =
          make_float4(__fmul_rn(code_at(w[k], 0), sc), __fmul_rn(code_at(w[k], 1), sc),
                      __fmul_rn(code_at(w[k], 2), sc), __fmul_rn(code_at(w[k], 3), sc));
  }
  return lane == 0 ? f : 0;
}

// kEpi promotion warps (8 or 16) in (kEpi/4) column groups of kCols = BN*4/kEpi;
// kIss MMA issuer warps (1, or 3 when nchunks % 4 == 0).
template <bool kFast, bool kPartials, int kEpi, int kIss>
__global__ void __launch_bounds__((1 + kIss + kEpi) * 32, 1)
    gemm_i8_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const Params p) {
  constexpr int kCtrl = 1 + kIss;  // warp 0: TMA, warps 1..kIss: MMA issuers
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
  const int my_tiles = (int)((ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x);
  const uint32_t bar_full = smem_u32(&S.full[0]), bar_empty = smem_u32(&S.empty[0]);
  const uint32_t bar_tfull = smem_u32(&S.tfull[0]), bar_tempty = smem_u32(&S.tempty[0]);

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], kIss > 1 ? kChunksPerStage : 1);  // multi-issuer: one commit per chunk
    }
    for (int b = 0; b < kTmemBufs; ++b) {
      mbar_init(&S.tfull[b], 1);
      mbar_init(&S.tempty[b], kEpi);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&S.tmem_base, kTmemBufs * BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;

  if (warp == 0) {
    // ───────────── TMA producer ─────────────
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int m0 = (int)((tile % mt) * BM), n0 = (int)((tile / mt) * BN);
        for (int ks = 0; ks < nstages_k; ++ks) {
          ctl_wait(p, bar_empty + 8 * stage, phase ^ 1);
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
  } else if (warp < kCtrl) {
    // ───────────── MMA issuers ─────────────
    // Descriptors are precomputed: the per-chunk path is wait -> fence -> MMA -> commit.
    const uint64_t adesc0 = smem_desc_sw128(smem_u32(sA), 16, 1024);
    const uint64_t bdesc0 = smem_desc_sw128(smem_u32(sB), 16, 1024);
    constexpr uint32_t idesc = idesc_i8(BM, BN, 0, 0);
    if (kIss > 1) {
      // issuer j takes global chunks g = j, j+kIss, ...: stage seq g/4, buffer (and
      // K slice within the stage) g%4, and this is buffer g%4's (g/4)-th use.
      if (lane == 0) {
        const int total = my_tiles * nchunks;
        for (int g = warp - 1; g < total; g += kIss) {
          const int G = g >> 2, c = g & 3, slot = G % kStages;
          mbar_wait_u32(bar_full + 8 * slot, (uint32_t)(G / kStages) & 1);
          mbar_wait_u32(bar_tempty + 8 * c, ((uint32_t)G & 1) ^ 1);
          tc_fence_after();
          mma_i8_ss(tmem + c * BN, adesc0 + (uint64_t)((slot * kStageBytesA + c * 32) >> 4),
                    bdesc0 + (uint64_t)((slot * kStageBytesB + c * 32) >> 4), idesc, 0u);
          mma_commit(&S.tfull[c]);
          mma_commit(&S.empty[slot]);
        }
      }
    } else if (lane == 0) {
      // single issuer (generic K): chunk ci of every tile lands in TMEM buffer ci % 4
      int stage = 0, gk = 0;
      uint32_t phase = 0, tphase = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int ks = 0; ks < nstages_k; ++ks) {
          ctl_wait(p, bar_full + 8 * stage, phase);
          tc_fence_after();
          const uint64_t ad = adesc0 + (uint64_t)((stage * kStageBytesA) >> 4);
          const uint64_t bd = bdesc0 + (uint64_t)((stage * kStageBytesB) >> 4);
          const int nch = min(kChunksPerStage, nchunks - ks * kChunksPerStage);
#pragma unroll
          for (int c = 0; c < kChunksPerStage; ++c) {
            if (c < nch) {
              ctl_wait(p, bar_tempty + 8 * c, ((tphase >> c) & 1) ^ 1);
              tphase ^= 1u << c;
              tc_fence_after();
              mma_i8_ss(tmem + c * BN, ad + 2 * c, bd + 2 * c, idesc, 0u);
              mma_commit(&S.tfull[c]);
            }
          }
          mma_commit(&S.empty[stage]);
          gk += nch;
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else {
    // ───────────── promotion + epilogue ─────────────
    constexpr int kCols = BN * 4 / kEpi;        // columns per warp: 64 (8 warps) or 32 (16 warps)
    constexpr int kBlk = kCols / 32;            // 32-column blocks per warp
    const int lq = warp & 3;                    // TMEM lane quarter == 32-row block of the tile
    const int cgp = (warp - kCtrl) >> 2;        // column group
    const uint32_t tcol = tmem + ((uint32_t)(lq * 32) << 16) + cgp * kCols;
    const bool vec_scales = (p.sa_s1 == 1) && (p.sb_s1 == 1) && (nchunks % 4 == 0);
    uint32_t tphase = 0;
    int flags = 0;
    int lt = 0;  // this CTA's local tile index
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++lt) {
      const int64_t I = (tile % mt) * (BM / 32) + lq;              // 32-row block index
      const int64_t J0 = (tile / mt) * (BN / 32) + kBlk * cgp;     // first 32-col block
      const bool vrow = I * 32 < p.M;
      bool vb[kBlk];
#pragma unroll
      for (int q = 0; q < kBlk; ++q) vb[q] = vrow && ((J0 + q) * 32 < p.N);
      float acc[kBlk][32];
#pragma unroll
      for (int q = 0; q < kBlk; ++q)
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[q][j] = 0.0f;
      const float *pa = p.sa + (kPartials || !vrow ? 0 : I * p.sa_s0);
      const float *pb[kBlk];
#pragma unroll
      for (int q = 0; q < kBlk; ++q) pb[q] = p.sb + (kPartials || !vb[q] ? 0 : (J0 + q) * p.sb_s0);
      for (int cb = 0; cb < nchunks; cb += kTmemBufs) {
        float sav[4] = {0.f, 0.f, 0.f, 0.f}, sbv[kBlk][4];
#pragma unroll
        for (int q = 0; q < kBlk; ++q) sbv[q][0] = sbv[q][1] = sbv[q][2] = sbv[q][3] = 0.f;
        if (!kPartials) {
          if (vec_scales) {  // K-contiguous scale grids: 4 chunks per 16-byte load
            if (vrow) {
              const float4 t = __ldg(reinterpret_cast<const float4 *>(pa + cb));
              sav[0] = t.x; sav[1] = t.y; sav[2] = t.z; sav[3] = t.w;
            }
#pragma unroll
            for (int q = 0; q < kBlk; ++q)
              if (vb[q]) {
                const float4 t = __ldg(reinterpret_cast<const float4 *>(pb[q] + cb));
                sbv[q][0] = t.x; sbv[q][1] = t.y; sbv[q][2] = t.z; sbv[q][3] = t.w;
              }
          } else {
#pragma unroll
            for (int b = 0; b < kTmemBufs; ++b)
              if (cb + b < nchunks) {
                if (vrow) sav[b] = __ldg(pa + (cb + b) * p.sa_s1);
#pragma unroll
                for (int q = 0; q < kBlk; ++q)
                  if (vb[q]) sbv[q][b] = __ldg(pb[q] + (cb + b) * p.sb_s1);
              }
          }
        }
#pragma unroll
        for (int b = 0; b < kTmemBufs; ++b) {
          if (cb + b >= nchunks) break;
          mbar_wait_u32(bar_tfull + 8 * b, (tphase >> b) & 1);
          tphase ^= 1u << b;
          tc_fence_after();
          uint32_t r[kBlk][32];
#pragma unroll
          for (int q = 0; q < kBlk; ++q) tmem_ld_32x32b_x32(tcol + b * BN + 32 * q, r[q]);
          tmem_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_u32(bar_tempty + 8 * b);
          if (kPartials) {
            // debug: raw int32 partials of the (single) chunk
#pragma unroll
            for (int q = 0; q < kBlk; ++q)
              if (vb[q]) {
                int32_t *dst = reinterpret_cast<int32_t *>(p.yf) + (I * 32 + lane) * p.N + (J0 + q) * 32;
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                  *reinterpret_cast<int4 *>(dst + j) =
                      make_int4((int)r[q][j], (int)r[q][j + 1], (int)r[q][j + 2], (int)r[q][j + 3]);
              }
          } else {
#pragma unroll
            for (int q = 0; q < kBlk; ++q) promote32<kFast>(acc[q], r[q], sav[b], sbv[q][b], p.zero);
          }
        }
      }
      if (kPartials) continue;
#pragma unroll
      for (int q = 0; q < kBlk; ++q)
        if (vb[q]) flags |= finish_block(p, acc[q], I, J0 + q, lane);
    }
    if (lane == 0) raise_flags(p.err, flags);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, kTmemBufs * BN);
}


// ─────────────── gemm_i8s_kernel: the same pipeline, scales staged by TMA ───────────────
// Used when M, N, K are multiples of 128 (every transformer-block shape).  The
// TMA producer also brings each stage's 4x4 sub-grids of sA and sB (64 B each)
// into shared memory, so the promotion warps read their scale factors with
// one LDS per 4 chunks instead of two L2-latency LDGs (hand-off microbenchmark:
// 471 clk/chunk floor, +66 with global scale loads).  A stage is released only
// when the MMAs consumed its tiles AND all promotion warps read its scales
// (empty barrier count 1 + 16).  No partial tiles, so no validity predicates.
struct SmemS {
  uint64_t full[kStages];
  uint64_t empty[kStages];
  uint64_t tfull[kTmemBufs];
  uint64_t tempty[kTmemBufs];
  uint32_t tmem_base;
};
constexpr uint32_t kScaleBytes = 256;  // per stage: A box at +0, B box at +128 (16 floats each)
constexpr size_t kSmemBytesS =
    1024 + kStages * (kStageBytesA + kStageBytesB) + kStages * kScaleBytes + sizeof(SmemS) + 64;

// kAmn / kBmn: the operand is MN-major in memory (the UMMA reads int8
// MN-major tiles directly, so dgrad consumes W [d x c] and wgrad consumes
// dY [n x d] and X [n x c] as stored -- no transposed copies).  An MN-major
// stage is a TMA box of 128 K-rows x 128 MN-bytes (SW128); chunk c starts
// 32 rows = 4096 bytes further, versus 32 bytes for a K-major stage.
template <bool kFast, bool kAmn, bool kBmn>
__global__ void __launch_bounds__((2 + 16) * 32, 1)
    gemm_i8s_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmSA, const __grid_constant__ CUtensorMap tmSB,
                    const Params p, const int saT, const int sbT) {
  constexpr int kEpi = 16;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *base = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sA = base;
  uint8_t *sB = base + kStages * kStageBytesA;
  uint8_t *sS = sB + kStages * kStageBytesB;  // scale boxes, 128-byte aligned
  SmemS &S = *reinterpret_cast<SmemS *>(sS + kStages * kScaleBytes);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t mt = p.M / BM, nt = p.N / BN;
  const int64_t ntiles = mt * nt;
  const int nstages_k = (int)(p.K / BK);
  const uint32_t bar_full = smem_u32(&S.full[0]), bar_empty = smem_u32(&S.empty[0]);
  const uint32_t bar_tfull = smem_u32(&S.tfull[0]), bar_tempty = smem_u32(&S.tempty[0]);

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    prefetch_tmap(&tmSA);
    prefetch_tmap(&tmSB);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], 1 + kEpi);
    }
    for (int b = 0; b < kTmemBufs; ++b) {
      mbar_init(&S.tfull[b], 1);
      mbar_init(&S.tempty[b], kEpi);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&S.tmem_base, kTmemBufs * BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;

  if (warp == 0) {
    // ───────────── TMA producer: int8 tiles + scale sub-grids ─────────────
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
#pragma unroll 1
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int m0 = (int)((tile % mt) * BM), n0 = (int)((tile / mt) * BN);
#pragma unroll 1  // (control loops stay compact: they share the L0 I-cache with the promotion loop)
        for (int ks = 0; ks < nstages_k; ++ks) {
          ctl_wait(p, bar_empty + 8 * stage, phase ^ 1);
          mbar_arrive_expect_tx(&S.full[stage], kStageBytesA + kStageBytesB + 128);
          // tensor-map coordinates are {inner, outer}
          if (kAmn) tma_load_2d(sA + stage * kStageBytesA, &tmA, &S.full[stage], m0, ks * BK);
          else tma_load_2d(sA + stage * kStageBytesA, &tmA, &S.full[stage], ks * BK, m0);
          if (kBmn) tma_load_2d(sB + stage * kStageBytesB, &tmB, &S.full[stage], n0, ks * BK);
          else tma_load_2d(sB + stage * kStageBytesB, &tmB, &S.full[stage], ks * BK, n0);
          uint8_t *ss = sS + stage * kScaleBytes;
          // box {4, 4}: K-contiguous grids -> [row block][chunk], else [chunk][row block]
          if (saT) tma_load_2d(ss, &tmSA, &S.full[stage], m0 / 32, ks * 4);
          else tma_load_2d(ss, &tmSA, &S.full[stage], ks * 4, m0 / 32);
          if (sbT) tma_load_2d(ss + 128, &tmSB, &S.full[stage], n0 / 32, ks * 4);
          else tma_load_2d(ss + 128, &tmSB, &S.full[stage], ks * 4, n0 / 32);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ───────────── MMA issuer: chunk c of every stage -> TMEM buffer c ─────────────
    if (lane == 0) {
      const uint64_t adesc0 = smem_desc_sw128(smem_u32(sA), 16, 1024);
      const uint64_t bdesc0 = smem_desc_sw128(smem_u32(sB), 16, 1024);
      constexpr uint32_t idesc = idesc_i8(BM, BN, kAmn ? 1 : 0, kBmn ? 1 : 0);
      constexpr uint32_t kStepA = kAmn ? (32 * 128) >> 4 : 2;  // descriptor units (16 B) per chunk
      constexpr uint32_t kStepB = kBmn ? (32 * 128) >> 4 : 2;
      int stage = 0;
      uint32_t phase = 0, tphase = 0;
#pragma unroll 1
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
#pragma unroll 1
        for (int ks = 0; ks < nstages_k; ++ks) {
          ctl_wait(p, bar_full + 8 * stage, phase);
          tc_fence_after();
          const uint64_t ad = adesc0 + (uint64_t)((stage * kStageBytesA) >> 4);
          const uint64_t bd = bdesc0 + (uint64_t)((stage * kStageBytesB) >> 4);
#pragma unroll
          for (int c = 0; c < kChunksPerStage; ++c) {
            ctl_wait(p, bar_tempty + 8 * c, ((tphase >> c) & 1) ^ 1);
            tphase ^= 1u << c;
            tc_fence_after();
            mma_i8_ss(tmem + c * BN, ad + kStepA * c, bd + kStepB * c, idesc, 0u);
            mma_commit(&S.tfull[c]);
          }
          mma_commit(&S.empty[stage]);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else {
    // ───────────── promotion + epilogue ─────────────
    const int lq = warp & 3;          // TMEM lane quarter == 32-row block of the tile
    const int cg = (warp - 2) >> 2;   // 32-column group of the tile
    const uint32_t tcol = tmem + ((uint32_t)(lq * 32) << 16) + cg * 32;
    const uint32_t ssa0 = smem_u32(sS), ssb0 = ssa0 + 128;
    // float offsets of this warp's 4 scale factors inside the 4x4 boxes
    const uint32_t oa = saT ? (uint32_t)lq * 4 : (uint32_t)lq * 16;
    const uint32_t ob = sbT ? (uint32_t)cg * 4 : (uint32_t)cg * 16;
    const uint32_t da = saT ? 16 : 4, db = sbT ? 16 : 4;  // byte step between chunks
    uint32_t tphase = 0;
    int flags = 0;
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t I = (tile % mt) * (BM / 32) + lq;
      const int64_t J = (tile / mt) * (BN / 32) + cg;
      float acc[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = 0.0f;
#pragma unroll 2
      for (int ks = 0; ks < nstages_k; ++ks) {
        // the stage's scales: acquire the TMA writes, read, release the stage
        mbar_wait_u32(bar_full + 8 * stage, phase);
        const uint32_t sa_addr = ssa0 + stage * kScaleBytes + oa, sb_addr = ssb0 + stage * kScaleBytes + ob;
        float sav[4], sbv[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          sav[b] = lds_f32(sa_addr + b * da);
          sbv[b] = lds_f32(sb_addr + b * db);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_u32(bar_empty + 8 * stage);
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
#pragma unroll
        for (int b = 0; b < kTmemBufs; ++b) {
          mbar_wait_u32(bar_tfull + 8 * b, (tphase >> b) & 1);
          tphase ^= 1u << b;
          tc_fence_after();
          uint32_t r[32];
          tmem_ld_32x32b_x32(tcol + b * BN, r);
          tmem_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_u32(bar_tempty + 8 * b);
          promote32<kFast>(acc, r, sav[b], sbv[b], p.zero);
        }
      }
      flags |= finish_block(p, acc, I, J, lane);
    }
    if (lane == 0) raise_flags(p.err, flags);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, kTmemBufs * BN);
}

// ─────────────── gemm_f16s_kernel: f16-widened codes, kind::f16 MMA ───────────────
// Same pipeline, scale staging and promotion as gemm_i8s_kernel (K-major A and
// B), but the operands are the int8 codes widened to f16 in HBM
// (jf_widen_codes): the f32 accumulator of the kind::f16 MMA holds the exact
// integer partial (every product and partial sum is an integer below 2^20),
// so the promotion skips the 32 I2F per chunk -- the kernel's issue-slot
// bottleneck.  Bit-identical to the int8 kernels.  A stage (128 K) is two
// 64-wide SW128 boxes per operand; a 32-deep chunk is two K=16 MMAs.
constexpr int kStagesF = 3;
constexpr uint32_t kBoxBytesF = 128 * 128;         // 128 rows x 64 f16
constexpr uint32_t kStageBytesF = 2 * kBoxBytesF;  // per operand
constexpr size_t kSmemBytesF = 1024 + kStagesF * 2 * kStageBytesF + kStagesF * kScaleBytes + sizeof(SmemS) + 64;

template <bool kFast>
__global__ void __launch_bounds__((2 + 16) * 32, 1)
    gemm_f16s_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmSA, const __grid_constant__ CUtensorMap tmSB,
                     const Params p, const int saT, const int sbT) {
  constexpr int kEpi = 16;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *base = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sA = base;
  uint8_t *sB = base + kStagesF * kStageBytesF;
  uint8_t *sS = sB + kStagesF * kStageBytesF;
  SmemS &S = *reinterpret_cast<SmemS *>(sS + kStagesF * kScaleBytes);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t mt = p.M / BM, nt = p.N / BN;
  const int64_t ntiles = mt * nt;
  const int nstages_k = (int)(p.K / BK);
  const uint32_t bar_full = smem_u32(&S.full[0]), bar_empty = smem_u32(&S.empty[0]);
  const uint32_t bar_tfull = smem_u32(&S.tfull[0]), bar_tempty = smem_u32(&S.tempty[0]);

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    prefetch_tmap(&tmSA);
    prefetch_tmap(&tmSB);
    for (int s = 0; s < kStagesF; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], 1 + kEpi);
    }
    for (int b = 0; b < kTmemBufs; ++b) {
      mbar_init(&S.tfull[b], 1);
      mbar_init(&S.tempty[b], kEpi);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&S.tmem_base, kTmemBufs * BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;

  if (warp == 0) {
    // ───────────── TMA producer: f16 tiles (2 boxes each) + scale sub-grids ─────────────
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int m0 = (int)((tile % mt) * BM), n0 = (int)((tile / mt) * BN);
        for (int ks = 0; ks < nstages_k; ++ks) {
          ctl_wait(p, bar_empty + 8 * stage, phase ^ 1);
          mbar_arrive_expect_tx(&S.full[stage], 2 * kStageBytesF + 128);
          uint8_t *a = sA + stage * kStageBytesF, *b = sB + stage * kStageBytesF;
          tma_load_2d(a, &tmA, &S.full[stage], ks * BK, m0);
          tma_load_2d(a + kBoxBytesF, &tmA, &S.full[stage], ks * BK + 64, m0);
          tma_load_2d(b, &tmB, &S.full[stage], ks * BK, n0);
          tma_load_2d(b + kBoxBytesF, &tmB, &S.full[stage], ks * BK + 64, n0);
          uint8_t *ss = sS + stage * kScaleBytes;
          if (saT) tma_load_2d(ss, &tmSA, &S.full[stage], m0 / 32, ks * 4);
          else tma_load_2d(ss, &tmSA, &S.full[stage], ks * 4, m0 / 32);
          if (sbT) tma_load_2d(ss + 128, &tmSB, &S.full[stage], n0 / 32, ks * 4);
          else tma_load_2d(ss + 128, &tmSB, &S.full[stage], ks * 4, n0 / 32);
          if (++stage == kStagesF) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ───────────── MMA issuer: chunk c -> TMEM buffer c, two K=16 MMAs ─────────────
    if (lane == 0) {
      const uint64_t adesc0 = smem_desc_sw128(smem_u32(sA), 16, 1024);
      const uint64_t bdesc0 = smem_desc_sw128(smem_u32(sB), 16, 1024);
      constexpr uint32_t idesc = idesc_f16_f32(BM, BN);
      int stage = 0;
      uint32_t phase = 0, tphase = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int ks = 0; ks < nstages_k; ++ks) {
          ctl_wait(p, bar_full + 8 * stage, phase);
          tc_fence_after();
          const uint64_t ad = adesc0 + (uint64_t)((stage * kStageBytesF) >> 4);
          const uint64_t bd = bdesc0 + (uint64_t)((stage * kStageBytesF) >> 4);
#pragma unroll
          for (int c = 0; c < kChunksPerStage; ++c) {
            ctl_wait(p, bar_tempty + 8 * c, ((tphase >> c) & 1) ^ 1);
            tphase ^= 1u << c;
            tc_fence_after();
            // chunk c: box c/2, byte offset (c%2)*64 in the 128-byte row; K=16 step = 32 bytes
            const uint32_t off = ((c >> 1) * kBoxBytesF + (c & 1) * 64) >> 4;
            mma_f16_ss(tmem + c * BN, ad + off, bd + off, idesc, 0u);
            mma_f16_ss(tmem + c * BN, ad + off + 2, bd + off + 2, idesc, 1u);
            mma_commit(&S.tfull[c]);
          }
          mma_commit(&S.empty[stage]);
          if (++stage == kStagesF) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else {
    // ───────────── promotion + epilogue (as gemm_i8s_kernel, f32 partials) ─────────────
    const int lq = warp & 3;
    const int cg = (warp - 2) >> 2;
    const uint32_t tcol = tmem + ((uint32_t)(lq * 32) << 16) + cg * 32;
    const uint32_t ssa0 = smem_u32(sS), ssb0 = ssa0 + 128;
    const uint32_t oa = saT ? (uint32_t)lq * 4 : (uint32_t)lq * 16;
    const uint32_t ob = sbT ? (uint32_t)cg * 4 : (uint32_t)cg * 16;
    const uint32_t da = saT ? 16 : 4, db = sbT ? 16 : 4;
    uint32_t tphase = 0;
    int flags = 0;
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t I = (tile % mt) * (BM / 32) + lq;
      const int64_t J = (tile / mt) * (BN / 32) + cg;
      float acc[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = 0.0f;
      for (int ks = 0; ks < nstages_k; ++ks) {
        mbar_wait_u32(bar_full + 8 * stage, phase);
        const uint32_t sa_addr = ssa0 + stage * kScaleBytes + oa, sb_addr = ssb0 + stage * kScaleBytes + ob;
        float sav[4], sbv[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          sav[b] = lds_f32(sa_addr + b * da);
          sbv[b] = lds_f32(sb_addr + b * db);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_u32(bar_empty + 8 * stage);
        if (++stage == kStagesF) {
          stage = 0;
          phase ^= 1;
        }
#pragma unroll
        for (int b = 0; b < kTmemBufs; ++b) {
          mbar_wait_u32(bar_tfull + 8 * b, (tphase >> b) & 1);
          tphase ^= 1u << b;
          tc_fence_after();
          uint32_t r[32];
          tmem_ld_32x32b_x32(tcol + b * BN, r);
          tmem_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_u32(bar_tempty + 8 * b);
          promote32f<kFast>(acc, r, sav[b], sbv[b], p.zero);
        }
      }
      flags |= finish_block(p, acc, I, J, lane);
    }
    if (lane == 0) raise_flags(p.err, flags);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, kTmemBufs * BN);
}

// int8 codes -> f16 (exact), 16 codes per thread.
__global__ void widen_codes_kernel(const int8_t *__restrict__ x, __half *__restrict__ y, int64_t n16) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n16) return;
  const int4 v = reinterpret_cast<const int4 *>(x)[i];
  uint32_t o[8];
  i8x4_to_f16x4((uint32_t)v.x, o[0], o[1]);
  i8x4_to_f16x4((uint32_t)v.y, o[2], o[3]);
  i8x4_to_f16x4((uint32_t)v.z, o[4], o[5]);
  i8x4_to_f16x4((uint32_t)v.w, o[6], o[7]);
  int4 *d = reinterpret_cast<int4 *>(y) + 2 * i;
  d[0] = make_int4((int)o[0], (int)o[1], (int)o[2], (int)o[3]);
  d[1] = make_int4((int)o[4], (int)o[5], (int)o[6], (int)o[7]);
}

// int8 codes [rows x cols] -> f16 transposed [cols x rows]; 64 x 64 tiles via shared memory.
__global__ void __launch_bounds__(256) widen_codes_t_kernel(const int8_t *__restrict__ x, __half *__restrict__ y,
                                                            int64_t rows, int64_t cols) {
  __shared__ uint8_t t[64][64 + 4];
  const int64_t r0 = (int64_t)blockIdx.y * 64, c0 = (int64_t)blockIdx.x * 64;
  {
    const int r = threadIdx.x >> 2, seg = threadIdx.x & 3;  // 64 rows x 4 segments of 16 bytes
    const int4 v = *reinterpret_cast<const int4 *>(x + (r0 + r) * cols + c0 + seg * 16);
    uint32_t *d = reinterpret_cast<uint32_t *>(&t[r][seg * 16]);
    d[0] = (uint32_t)v.x;
    d[1] = (uint32_t)v.y;
    d[2] = (uint32_t)v.z;
    d[3] = (uint32_t)v.w;
  }
  __syncthreads();
  const int oc = threadIdx.x >> 2, seg = threadIdx.x & 3;  // output row oc (= input column), 16 codes
  uint32_t w[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int rr = seg * 16 + q * 4;
    w[q] = (uint32_t)t[rr][oc] | ((uint32_t)t[rr + 1][oc] << 8) | ((uint32_t)t[rr + 2][oc] << 16) |
           ((uint32_t)t[rr + 3][oc] << 24);
  }
  uint32_t o[8];
  i8x4_to_f16x4(w[0], o[0], o[1]);
  i8x4_to_f16x4(w[1], o[2], o[3]);
  i8x4_to_f16x4(w[2], o[4], o[5]);
  i8x4_to_f16x4(w[3], o[6], o[7]);
  int4 *d = reinterpret_cast<int4 *>(y + (c0 + oc) * rows + r0 + seg * 16);
  d[0] = make_int4((int)o[0], (int)o[1], (int)o[2], (int)o[3]);
  d[1] = make_int4((int)o[4], (int)o[5], (int)o[6], (int)o[7]);
}

#ifdef JF_GEMM_TRACE
#define JF_TR(ev, i)                                                                        \
  do {                                                                                      \
    if (blockIdx.x == 0 && (i) < 512 && p.trace) p.trace[(ev) * 512 + (i)] = clock64();     \
  } while (0)
#else
#define JF_TR(ev, i) \
  do {               \
  } while (0)
#endif

// ─────────────── kind::f16 variant: int8 codes in HBM, f16 tiles in smem ───────────────
// The tensor core's int32 output forces one I2F per output element per chunk
// (ALU pipe, half rate): on B200 that, not the MMA, bounds the kind::i8
// kernel (ncu: ALU 65% / issue 68% busy in fast mode, tensor 12%).  Here the
// int8 codes are widened to f16 in shared memory (every code is exact in
// binary16) and tcgen05.mma.kind::f16 accumulates in f32: each 32-deep chunk's
// partial is an integer of magnitude <= 32*127^2 < 2^24, so the f32 partial
// IS the int32 partial, exactly, and the promotion reads it without any
// conversion.  The widening costs ~1.5 instructions per OPERAND element
// (8192 per 128x128x32 chunk) instead of one I2F per OUTPUT element (16384).
//   warps 0..15  promotion/epilogue (as in gemm_i8_kernel); warp 0 lane 0
//                also issues the MMAs right after its TMEM slot is released
//   warps 16..19 converters; warp 16 lane 0 is also the TMA producer
namespace h16 {
constexpr int BKH = 64;                       // K per stage (2 chunks)
constexpr int kHStages = 3;                   // f16 ring depth (tensor-core operands)
constexpr int kQStages = 8;                   // int8 ring depth (TMA lookahead)
constexpr int kConvWarps = 4;
constexpr int kWarps = kConvWarps + kEpiWarps;
constexpr uint32_t kI8Bytes = BM * BKH;       // per operand per stage: 8 KB
constexpr uint32_t kF16Bytes = BM * BKH * 2;  // 16 KB (128 rows x 128 B, SW128)
struct Bars {
  uint64_t full8[kQStages], empty8[kQStages], hfull[kHStages], hempty[kHStages];
  uint64_t tfull[kPairSlots], tempty[kPairSlots];
  uint32_t tmem_base;
};
constexpr size_t kSmemBytes = 1024 + kHStages * 2 * kF16Bytes + kQStages * 2 * kI8Bytes + 256;
}  // namespace h16

template <bool kFast, int kProbe = 0>  // diagnostics: kProbe 1 = converters skip the widening, 2 = no TMEM loads
__global__ void __launch_bounds__(h16::kWarps * 32, 1)
    gemm_h16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const Params p) {
  using namespace h16;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *base = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *hA = base;                              // f16 ring (1024-aligned for SW128)
  uint8_t *hB = hA + kHStages * kF16Bytes;
  uint8_t *qA = hB + kHStages * kF16Bytes;          // int8 ring (TMA, no swizzle)
  uint8_t *qB = qA + kQStages * kI8Bytes;
  Bars &S = *reinterpret_cast<Bars *>(qB + kQStages * kI8Bytes);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t mt = (p.M + BM - 1) / BM, nt = (p.N + BN - 1) / BN;
  const int64_t ntiles = mt * nt;
  const int nchunks = (int)(p.K / 32);
  const int nh = (nchunks + 1) / 2;  // stages (chunk pairs) per tile
  const int my_tiles = (int)((ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x);
  const int total = my_tiles * nh;   // stages this CTA streams
  const uint32_t bar_full8 = smem_u32(&S.full8[0]), bar_empty8 = smem_u32(&S.empty8[0]);
  const uint32_t bar_hfull = smem_u32(&S.hfull[0]), bar_hempty = smem_u32(&S.hempty[0]);
  const uint32_t bar_tfull = smem_u32(&S.tfull[0]), bar_tempty = smem_u32(&S.tempty[0]);

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < kQStages; ++s) {
      mbar_init(&S.full8[s], 1);
      mbar_init(&S.empty8[s], kConvWarps);
    }
    for (int s = 0; s < kHStages; ++s) {
      mbar_init(&S.hfull[s], kConvWarps);
      mbar_init(&S.hempty[s], 1);
    }
    for (int b = 0; b < kPairSlots; ++b) {
      mbar_init(&S.tfull[b], 1);
      mbar_init(&S.tempty[b], kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&S.tmem_base, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;

  // Converters take the HIGHEST warp ids: the SMSP arbiter favours high warp
  // ids, and the converters (plus the TMA producer among them) are the
  // latency-critical producers; with low ids they starved behind the
  // promotion warps (trace: 2.6k clk per stage vs ~0.3k of work).
  const int cw = warp - kEpiWarps;  // converter index, valid when >= 0
  if (cw >= 0) {
    // ───────────── converters (converter 0 lane 0 is also the TMA producer) ─────────────
    auto issue_tma = [&](int g) {
      const int s = g % kQStages;
      mbar_wait_u32(bar_empty8 + 8 * s, ((g / kQStages) & 1) ^ 1);
      const int lt = g / nh, kh = g - lt * nh;
      const int64_t tile = blockIdx.x + (int64_t)lt * gridDim.x;
      const int m0 = (int)((tile % mt) * BM), n0 = (int)((tile / mt) * BN), k0 = kh * BKH;
      mbar_arrive_expect_tx(&S.full8[s], 2 * kI8Bytes);
      tma_load_2d(qA + s * kI8Bytes, &tmA, &S.full8[s], k0, m0);
      tma_load_2d(qB + s * kI8Bytes, &tmB, &S.full8[s], k0, n0);
    };
    if (cw == 0 && lane == 0)
      for (int g = 0; g < min(kQStages - 1, total); ++g) issue_tma(g);
    __syncwarp();
    const uint32_t q_base = smem_u32(qA), h_base = smem_u32(hA);
    // item = (row of the 256 A|B rows, 16-byte source chunk c4 of its 64 bytes);
    // thread handles rows 8*j + lane/4 of this warp's 64, chunk c4 = lane % 4
    const int c4 = lane & 3;
    for (int g = 0; g < total; ++g) {
      const int s = g % kHStages, s8 = g % kQStages;
      if (cw == 0 && lane == 0) JF_TR(0, g);
      if (cw == 0 && lane == 0 && g + kQStages - 1 < total) issue_tma(g + kQStages - 1);
      mbar_wait_u32(bar_full8 + 8 * s8, (g / kQStages) & 1);
      if (cw == 0 && lane == 0) JF_TR(1, g);
      mbar_wait_u32(bar_hempty + 8 * s, ((g / kHStages) & 1) ^ 1);
      if (cw == 0 && lane == 0) JF_TR(2, g);
      if (kProbe != 1) {
        uint4 v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int rl = cw * 64 + j * 8 + (lane >> 2);  // 0..255
          const int isB = rl >> 7, r = rl & 127;
          v[j] = lds128(q_base + (uint32_t)(isB * kQStages + s8) * kI8Bytes + r * BKH + c4 * 16);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int rl = cw * 64 + j * 8 + (lane >> 2);
          const int isB = rl >> 7, r = rl & 127;
          const uint32_t row = h_base + (uint32_t)(isB * kHStages + s) * kF16Bytes + r * 128;
          uint32_t h[8];
          i8x4_to_f16x4(v[j].x, h[0], h[1]);
          i8x4_to_f16x4(v[j].y, h[2], h[3]);
          i8x4_to_f16x4(v[j].z, h[4], h[5]);
          i8x4_to_f16x4(v[j].w, h[6], h[7]);
          // f16 chunks 2*c4, 2*c4+1 of the row, 128-byte swizzle (chunk ^ row % 8)
          sts128(row + (((2 * c4) ^ (r & 7)) << 4), h[0], h[1], h[2], h[3]);
          sts128(row + (((2 * c4 + 1) ^ (r & 7)) << 4), h[4], h[5], h[6], h[7]);
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_u32(bar_hfull + 8 * s);
        mbar_arrive_u32(bar_empty8 + 8 * s8);
      }
      if (cw == 0 && lane == 0) JF_TR(3, g);
    }
  } else {
    // ───────────── promotion + epilogue (warp 0 lane 0 also issues the MMAs) ─────────────
    const int ew = warp;
    const int lq = warp & 3;
    const int cg = ew >> 2;
    const uint32_t tcol = tmem + ((uint32_t)(lq * 32) << 16) + cg * 32;
    const bool vec_scales = (p.sa_s1 == 1) && (p.sb_s1 == 1) && (nchunks % 4 == 0);
    const bool issuer = (ew == 0) && (lane == 0);
    const uint64_t adesc0 = smem_desc_sw128(smem_u32(hA), 16, 1024);
    const uint64_t bdesc0 = smem_desc_sw128(smem_u32(hB), 16, 1024);
    constexpr uint32_t idesc = idesc_f16_f32(BM, BN);
    // MMAs of stage g (a chunk pair) into TMEM slot g % 2; slot must be free
    auto issue_mma = [&](int g) {
      const int s = g % kHStages;
      const uint32_t slot = g & 1;
      const bool two = 2 * (g % nh) + 1 < nchunks;
      JF_TR(4, g);
      mbar_wait_u32(bar_hfull + 8 * s, (g / kHStages) & 1);
      JF_TR(5, g);
      mbar_wait_u32(bar_tempty + 8 * slot, ((g >> 1) & 1) ^ 1);
      JF_TR(6, g);
      tc_fence_after();
      const uint64_t ad = adesc0 + (uint64_t)((s * kF16Bytes) >> 4);
      const uint64_t bd = bdesc0 + (uint64_t)((s * kF16Bytes) >> 4);
      const uint32_t d0 = tmem + slot * (2 * BN);
      // chunk 0: K 0..31 = row bytes 0..63 (two K=16 MMAs, +32 B each); chunk 1: bytes 64..127
      mma_f16_ss(d0, ad, bd, idesc, 0u);
      mma_f16_ss(d0, ad + 2, bd + 2, idesc, 1u);
      if (two) {
        mma_f16_ss(d0 + BN, ad + 4, bd + 4, idesc, 0u);
        mma_f16_ss(d0 + BN, ad + 6, bd + 6, idesc, 1u);
      }
      mma_commit(&S.tfull[slot]);
      mma_commit(&S.hempty[s]);
    };
    if (issuer)
      for (int g = 0; g < min(kPairSlots, total); ++g) issue_mma(g);
    __syncwarp();
    uint32_t q = 0;
    int flags = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t I = (tile % mt) * (BM / 32) + lq;
      const int64_t J = (tile / mt) * (BN / 32) + cg;
      const bool valid = (I * 32 < p.M) && (J * 32 < p.N);
      float acc[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = 0.0f;
      const float *pa = p.sa + (valid ? I * p.sa_s0 : 0);
      const float *pb = p.sb + (valid ? J * p.sb_s0 : 0);
      float4 nsa = make_float4(0.f, 0.f, 0.f, 0.f), nsb = nsa;
      auto load_scales = [&](int cb, float4 &a4, float4 &b4) {
        if (!valid || cb >= nchunks) return;
        if (vec_scales) {
          a4 = __ldg(reinterpret_cast<const float4 *>(pa + cb));
          b4 = __ldg(reinterpret_cast<const float4 *>(pb + cb));
        } else {
          float t[4], u[4];
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            t[b] = cb + b < nchunks ? __ldg(pa + (cb + b) * p.sa_s1) : 0.f;
            u[b] = cb + b < nchunks ? __ldg(pb + (cb + b) * p.sb_s1) : 0.f;
          }
          a4 = make_float4(t[0], t[1], t[2], t[3]);
          b4 = make_float4(u[0], u[1], u[2], u[3]);
        }
      };
      load_scales(0, nsa, nsb);
      for (int cb = 0; cb < nchunks; cb += 4) {
        const float sav[4] = {nsa.x, nsa.y, nsa.z, nsa.w};
        const float sbv[4] = {nsb.x, nsb.y, nsb.z, nsb.w};
        load_scales(cb + 4, nsa, nsb);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c0 = cb + 2 * h;
          if (c0 >= nchunks) break;
          const bool two = c0 + 1 < nchunks;
          const uint32_t slot = q & 1;
          mbar_wait_u32(bar_tfull + 8 * slot, (q >> 1) & 1);
          if (issuer) JF_TR(7, (int)q);
          tc_fence_after();
          uint32_t r[32];
          const uint32_t t0 = tcol + slot * (2 * BN);
          if (kProbe != 2) {
            tmem_ld_32x32b_x32(t0, r);
            tmem_wait_ld();
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) r[j] = __float_as_uint((float)(j + lane));
          }
          promote32f<kFast>(acc, r, sav[2 * h], sbv[2 * h], p.zero);
          if (two && kProbe != 2) {
            tmem_ld_32x32b_x32(t0 + BN, r);
            tmem_wait_ld();
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_u32(bar_tempty + 8 * slot);
          if (issuer && (int)q + kPairSlots < total) issue_mma((int)q + kPairSlots);
          __syncwarp();
          ++q;
          if (two) promote32f<kFast>(acc, r, sav[2 * h + 1], sbv[2 * h + 1], p.zero);
        }
      }
      if (valid) flags |= finish_block(p, acc, I, J, lane);
    }
    if (lane == 0) raise_flags(p.err, flags);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, kTmemCols);
}

}  // namespace gemm
}  // namespace jf

// ─────────────────────────── host side ───────────────────────────
using namespace jf;

int jf_launch_check(const char *what);
void jf_set_error(const char *msg);
int jf_num_sms();
bool jf_make_tmap_i8(CUtensorMap *map, const void *ptr, int64_t rows, int64_t cols, int64_t ld,
                     int box_cols, int box_rows, bool swizzle128);
bool jf_make_tmap_f32(CUtensorMap *map, const void *ptr, int64_t rows, int64_t cols, int64_t ld,
                      int box_cols, int box_rows);
bool jf_make_tmap_f16(CUtensorMap *map, const void *ptr, int64_t rows, int64_t cols, int64_t ld,
                      int box_cols, int box_rows);

#ifdef JF_GEMM_TRACE
static long long *g_trace = nullptr;
extern "C" int jf_gemm_trace_read(long long *host) {
  if (!g_trace) return 1;
  return cudaMemcpy(host, g_trace, 8 * 512 * sizeof(long long), cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 2;
}
#endif

// Launch options (diagnostics / A-B experiments).  Defaults are the measured
// best; JF_GEMM_IMPL / JF_GEMM_EPI / JF_GEMM_ISSUERS / JF_GEMM_CTL set them at
// load time, jf_gemm_set_option() at run time.
struct GemmOptions {
  int impl = 0;      // 0 kind::i8, 1 kind::f16 (h16)
  int epi = 16;      // promotion warps (16 or 8)
  int issuers = 1;   // MMA issuer warps (1 or 3)
  int ctl_kind = 1;  // control-thread wait flavour (see ctl_wait; JF_CTL_RUNTIME builds only)
  int ctl_ns = 200;
  int tma_scales = 1;  // gemm_i8s_kernel when the shape allows
  GemmOptions() {
    if (const char *e = getenv("JF_GEMM_IMPL")) impl = strcmp(e, "h16") == 0 ? 1 : 0;
    if (const char *e = getenv("JF_GEMM_EPI")) epi = atoi(e) == 8 ? 8 : 16;
    if (const char *e = getenv("JF_GEMM_ISSUERS")) issuers = atoi(e) == 3 ? 3 : 1;
    if (const char *e = getenv("JF_GEMM_CTL")) sscanf(e, "%d,%d", &ctl_kind, &ctl_ns);
  }
};
static GemmOptions g_opt;

extern "C" int jf_gemm_set_option(const char *key, int value) {
  if (!strcmp(key, "impl")) g_opt.impl = value ? 1 : 0;
  else if (!strcmp(key, "epi")) g_opt.epi = value == 8 ? 8 : 16;
  else if (!strcmp(key, "issuers")) g_opt.issuers = value == 3 ? 3 : 1;
  else if (!strcmp(key, "ctl_kind")) g_opt.ctl_kind = value;
  else if (!strcmp(key, "ctl_ns")) g_opt.ctl_ns = value;
  else if (!strcmp(key, "tma_scales")) g_opt.tma_scales = value;
  else return JF_ERR_ARG;
  return JF_OK;
}

// gemm_i8s_kernel launch.  A is [M x K] (K-major) or [K x M] (a_mn: MN-major), row
// stride lda bytes; likewise B as [N x K] or [K x N].  Returns -1 when the shape
// or the scale-grid layout does not qualify (caller falls back).
static int launch_i8s(const int8_t *A, bool a_mn, int64_t lda, const int8_t *B, bool b_mn, int64_t ldb, int64_t M,
                      int64_t N, int64_t K, const float *sa, int64_t sa_s0, int64_t sa_s1, const float *sb,
                      int64_t sb_s0, int64_t sb_s1, const float *bias, int mode, int out_kind, int8_t *yq,
                      float *ys, void *yf, int32_t *err, cudaStream_t stream) {
  using namespace jf::gemm;
  if (!g_opt.tma_scales || out_kind == OUT_I32 || M % 128 || N % 128 || K % 128 || lda % 16 || ldb % 16 ||
      (uintptr_t)A % 16 || (uintptr_t)B % 16)
    return -1;
  // scale grids: each contiguous along K or along M/N, 16-byte row pitch
  auto grid_ok = [](const float *s, int64_t s0, int64_t s1) {
    return ((uintptr_t)s % 16 == 0) && ((s1 == 1 && s0 % 4 == 0) || (s0 == 1 && s1 % 4 == 0));
  };
  if (!grid_ok(sa, sa_s0, sa_s1) || !grid_ok(sb, sb_s0, sb_s1)) return -1;
  const int64_t kb = K / 32;
  const int saT = sa_s1 != 1, sbT = sb_s1 != 1;
  CUtensorMap ta, tb, tsa, tsb;
  const bool ok =
      (a_mn ? jf_make_tmap_i8(&ta, A, K, M, lda, BM, BK, true) : jf_make_tmap_i8(&ta, A, M, K, lda, BK, BM, true)) &&
      (b_mn ? jf_make_tmap_i8(&tb, B, K, N, ldb, BN, BK, true) : jf_make_tmap_i8(&tb, B, N, K, ldb, BK, BN, true)) &&
      (saT ? jf_make_tmap_f32(&tsa, sa, kb, M / 32, sa_s1, 4, 4) : jf_make_tmap_f32(&tsa, sa, M / 32, kb, sa_s0, 4, 4)) &&
      (sbT ? jf_make_tmap_f32(&tsb, sb, kb, N / 32, sb_s1, 4, 4) : jf_make_tmap_f32(&tsb, sb, N / 32, kb, sb_s0, 4, 4));
  if (!ok) return JF_ERR_LAUNCH;
  Params p{M, N, K, sa, sa_s0, sa_s1, sb, sb_s0, sb_s1, bias, yq, ys, (float *)yf, err, out_kind, 0.0f, nullptr,
           g_opt.ctl_kind, (uint32_t)g_opt.ctl_ns};
  const bool fast = mode == JF_MODE_FAST;
  using KFn = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const CUtensorMap, const Params,
                       const int, const int);
  KFn ks;
  int ki;
  if (!a_mn && !b_mn) {
    ks = fast ? gemm_i8s_kernel<true, false, false> : gemm_i8s_kernel<false, false, false>;
    ki = 0;
  } else if (!a_mn && b_mn) {
    ks = fast ? gemm_i8s_kernel<true, false, true> : gemm_i8s_kernel<false, false, true>;
    ki = 1;
  } else if (a_mn && b_mn) {
    ks = fast ? gemm_i8s_kernel<true, true, true> : gemm_i8s_kernel<false, true, true>;
    ki = 2;
  } else {
    return -1;
  }
  static bool done[3][2] = {};
  if (!done[ki][fast]) {
    if (cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytesS) != cudaSuccess)
      return jf_launch_check("gemm_i8s attr");
    done[ki][fast] = true;
  }
  const int64_t tiles = (M / BM) * (N / BN);
  const int grid = (int)(tiles < jf_num_sms() ? tiles : jf_num_sms());
  ks<<<grid, 18 * 32, kSmemBytesS, stream>>>(ta, tb, tsa, tsb, p, saT, sbT);
  return jf_launch_check("gemm_i8s");
}

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
  const bool h16p = g_opt.impl == 1 && out_kind != OUT_I32;
  CUtensorMap ta, tb;
  if (h16p) {
    if (!jf_make_tmap_i8(&ta, A, M, K, lda, h16::BKH, BM, false) ||
        !jf_make_tmap_i8(&tb, Bt, N, K, ldb, h16::BKH, BN, false))
      return JF_ERR_LAUNCH;
  } else if (!jf_make_tmap_i8(&ta, A, M, K, lda, BK, BM, true) ||
             !jf_make_tmap_i8(&tb, Bt, N, K, ldb, BK, BN, true)) {
    return JF_ERR_LAUNCH;
  }
  Params p{M, N, K, sa, sa_s0, sa_s1, sb, sb_s0, sb_s1, bias, yq, ys, (float *)yf, err, out_kind, 0.0f, nullptr,
           g_opt.ctl_kind, (uint32_t)g_opt.ctl_ns};
#ifdef JF_GEMM_TRACE
  if (!g_trace) cudaMalloc(&g_trace, 8 * 512 * sizeof(long long));
  cudaMemsetAsync(g_trace, 0, 8 * 512 * sizeof(long long), stream);
  p.trace = g_trace;
#endif
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int grid = (int)(tiles < jf_num_sms() ? tiles : jf_num_sms());
  const bool fast = mode == JF_MODE_FAST;
  const bool partials = out_kind == OUT_I32;
  if (h16p) {
    void (*hk)(const CUtensorMap, const CUtensorMap, const Params) =
        fast ? gemm_h16_kernel<true> : gemm_h16_kernel<false>;
    static bool hdone[2] = {};
    if (!hdone[fast]) {
      if (cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h16::kSmemBytes) !=
          cudaSuccess)
        return jf_launch_check("gemm_h16 attr");
      hdone[fast] = true;
    }
    hk<<<grid, h16::kWarps * 32, h16::kSmemBytes, stream>>>(ta, tb, p);
    return jf_launch_check("gemm_h16");
  }
  if (!partials && !h16p) {
    const int rc = launch_i8s(A, false, lda, Bt, false, ldb, M, N, K, sa, sa_s0, sa_s1, sb, sb_s0, sb_s1, bias,
                              mode, out_kind, yq, ys, yf, err, stream);
    if (rc >= 0) return rc;
  }
  const int epi = g_opt.epi, iss_env = g_opt.issuers;
  // multi-issuer pipeline needs whole 4-chunk stages (K % 128 == 0)
  const int iss = (!partials && K % BK == 0) ? iss_env : 1;
  void (*kern)(const CUtensorMap, const CUtensorMap, const Params);
#define JF_PICK(E, IS)                                                                 \
  kern = partials ? gemm_i8_kernel<false, true, E, 1>                                  \
                  : (fast ? gemm_i8_kernel<true, false, E, IS> : gemm_i8_kernel<false, false, E, IS>);
  if (epi == 16) {
    if (iss == 3) { JF_PICK(16, 3) } else { JF_PICK(16, 1) }
  } else {
    if (iss == 3) { JF_PICK(8, 3) } else { JF_PICK(8, 1) }
  }
#undef JF_PICK
  static bool attr_done[2][2][3] = {};
  const int ki = partials ? 2 : (fast ? 1 : 0);
  bool &done = attr_done[epi == 16][iss == 3][ki];
  if (!done) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes) !=
        cudaSuccess)
      return jf_launch_check("gemm attr");
    done = true;
  }
  const int threads = (1 + iss + epi) * 32;
  kern<<<grid, threads, kSmemBytes, stream>>>(ta, tb, p);
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
  // W [d x c] is the MN-major B operand as stored (no W^T needed)
  {
    const int rc = launch_i8s(dy, false, d, w, true, c, n, c, d, dys, d / 32, 1, ws, 1, c / 32, nullptr, mode,
                              out_kind, dxq, dxs, dxf, err, (cudaStream_t)stream);
    if (rc >= 0) return rc;
  }
  if (wt == nullptr) {
    if (scratch == nullptr) return JF_ERR_ARG;
    int8_t *t = static_cast<int8_t *>(scratch);
    int rc = jf_transpose(w, nullptr, d, c, t, nullptr, stream);
    if (rc) return rc;
    wt = t;
    wts = nullptr;
  }
  // A = dY [n x d] (K = d), Bt = W^T [c x d]; sB(ci, J) = W.scales[ci, J] = W^T.scales[J, ci]
  if (wts != nullptr)
    return jf_gemm_launch(dy, d, wt, d, n, c, d, dys, d / 32, 1, wts, d / 32, 1, nullptr, mode,
                          out_kind, dxq, dxs, dxf, err, (cudaStream_t)stream);
  return jf_gemm_launch(dy, d, wt, d, n, c, d, dys, d / 32, 1, ws, 1, c / 32, nullptr, mode,
                        out_kind, dxq, dxs, dxf, err, (cudaStream_t)stream);
}

extern "C" int jf_gemm_wgrad(const int8_t *dy, const float *dys, const int8_t *x, const float *xs,
                             const int8_t *dyt, const float *dyts, const int8_t *xt,
                             const float *xts, int64_t n, int64_t d, int64_t c, int32_t mode,
                             int32_t out_kind, int8_t *dwq, float *dws, float *dwf, void *scratch,
                             int32_t *err, jf_stream_t stream) {
  // dY [n x d] and X [n x c] are the MN-major A and B operands as stored (no transposes)
  {
    const int rc = launch_i8s(dy, true, d, x, true, c, d, c, n, dys, 1, d / 32, xs, 1, c / 32, nullptr, mode,
                              out_kind, dwq, dws, dwf, err, (cudaStream_t)stream);
    if (rc >= 0) return rc;
  }
  int8_t *s8 = static_cast<int8_t *>(scratch);
  if (dyt == nullptr) {
    if (scratch == nullptr) return JF_ERR_ARG;
    int rc = jf_transpose(dy, nullptr, n, d, s8, nullptr, stream);  // [d x n]
    if (rc) return rc;
    dyt = s8;
    dyts = nullptr;
  }
  if (xt == nullptr) {
    if (scratch == nullptr) return JF_ERR_ARG;
    int8_t *t = s8 + n * d;
    int rc = jf_transpose(x, nullptr, n, c, t, nullptr, stream);  // [c x n]
    if (rc) return rc;
    xt = t;
    xts = nullptr;
  }
  // A = dY^T [d x n] (K = n): sA(I, ci) = dY.scales[ci, I] (= dY^T.scales[I, ci]);
  // Bt = X^T [c x n]: sB(ci, J) = X.scales[ci, J] (= X^T.scales[J, ci])
  const float *sa = dyts ? dyts : dys;
  const int64_t sa0 = dyts ? n / 32 : 1, sa1 = dyts ? 1 : d / 32;
  const float *sb = xts ? xts : xs;
  const int64_t sb0 = xts ? n / 32 : 1, sb1 = xts ? 1 : c / 32;
  return jf_gemm_launch(dyt, n, xt, n, d, c, n, sa, sa0, sa1, sb, sb0, sb1, nullptr, mode,
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

// ─────────────── f16-widened operand path (C ABI) ───────────────

extern "C" int jf_widen_codes(const int8_t *x, int64_t rows, int64_t cols, uint16_t *y, int32_t transpose,
                              jf_stream_t stream) {
  using namespace jf::gemm;
  if (rows <= 0 || cols <= 0 || rows % 64 || cols % 64 || (uintptr_t)x % 16 || (uintptr_t)y % 16) {
    jf_set_error("widen_codes: rows/cols must be positive multiples of 64, pointers 16-byte aligned");
    return JF_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (transpose) {
    widen_codes_t_kernel<<<dim3((unsigned)(cols / 64), (unsigned)(rows / 64)), 256, 0, s>>>(
        x, reinterpret_cast<__half *>(y), rows, cols);
  } else {
    const int64_t n16 = rows * cols / 16;
    widen_codes_kernel<<<(unsigned)((n16 + 255) / 256), 256, 0, s>>>(x, reinterpret_cast<__half *>(y), n16);
  }
  return jf_launch_check("widen_codes");
}

extern "C" int jf_gemm_f16(const uint16_t *a, const float *sa, int64_t sa_s0, int64_t sa_s1, const uint16_t *b,
                           const float *sb, int64_t sb_s0, int64_t sb_s1, const float *bias, int64_t m, int64_t n,
                           int64_t k, int32_t mode, int32_t out_kind, int8_t *yq, float *ys, float *yf,
                           int32_t *err, jf_stream_t stream) {
  using namespace jf::gemm;
  auto grid_ok = [](const float *s, int64_t s0, int64_t s1) {
    return ((uintptr_t)s % 16 == 0) && ((s1 == 1 && s0 % 4 == 0) || (s0 == 1 && s1 % 4 == 0));
  };
  if (m <= 0 || n <= 0 || k <= 0 || m % 128 || n % 128 || k % 128 || (uintptr_t)a % 16 || (uintptr_t)b % 16 ||
      !grid_ok(sa, sa_s0, sa_s1) || !grid_ok(sb, sb_s0, sb_s1) || out_kind == OUT_I32) {
    jf_set_error("gemm_f16: dims must be multiples of 128, scale grids contiguous along one axis");
    return JF_ERR_ARG;
  }
  const int64_t kb = k / 32;
  const int saT = sa_s1 != 1, sbT = sb_s1 != 1;
  CUtensorMap ta, tb, tsa, tsb;
  const bool ok = jf_make_tmap_f16(&ta, a, m, k, k, 64, BM) && jf_make_tmap_f16(&tb, b, n, k, k, 64, BN) &&
                  (saT ? jf_make_tmap_f32(&tsa, sa, kb, m / 32, sa_s1, 4, 4)
                       : jf_make_tmap_f32(&tsa, sa, m / 32, kb, sa_s0, 4, 4)) &&
                  (sbT ? jf_make_tmap_f32(&tsb, sb, kb, n / 32, sb_s1, 4, 4)
                       : jf_make_tmap_f32(&tsb, sb, n / 32, kb, sb_s0, 4, 4));
  if (!ok) return JF_ERR_LAUNCH;
  Params p{m, n, k, sa, sa_s0, sa_s1, sb, sb_s0, sb_s1, bias, yq, ys, yf, err, out_kind, 0.0f, nullptr,
           g_opt.ctl_kind, (uint32_t)g_opt.ctl_ns};
  const bool fast = mode == JF_MODE_FAST;
  auto kf = fast ? gemm_f16s_kernel<true> : gemm_f16s_kernel<false>;
  static bool done[2] = {};
  if (!done[fast]) {
    if (cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytesF) != cudaSuccess)
      return jf_launch_check("gemm_f16s attr");
    done[fast] = true;
  }
  const int64_t tiles = (m / BM) * (n / BN);
  const int grid = (int)(tiles < jf_num_sms() ? tiles : jf_num_sms());
  kf<<<grid, 18 * 32, kSmemBytesF, (cudaStream_t)stream>>>(ta, tb, tsa, tsb, p, saT, sbT);
  return jf_launch_check("gemm_f16s");
}
