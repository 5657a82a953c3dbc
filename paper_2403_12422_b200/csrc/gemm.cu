// gemm.cu — K3/K4/K5: the per-block INT8 GEMM on tcgen05 (sm_100a).
//
// Y[M x N] = sum over 32-deep K chunks ci (ascending) of
//            sA(I, ci) * sB(ci, J) * P_ci,   P_ci = A[:, 32ci:+32] . B[32ci:+32, :]
// exactly as qgemm.py:193-229 (_mm_core / _scaled_accumulate), then +bias and
// a 32x32 block requantization (qgemm.py:266-279).
//
// Main kernel (gemm_tc_kernel; every transformer shape: M, N, K multiples of 128):
// one persistent CTA per SM, warp-specialized, 128x128 output tiles.
//   warp 0        TMA producer: each stage = 4 K chunks of A and B (SW128 tiles)
//                 plus the stage's 4x4 sub-grids of both scale grids.
//   warp 1        MMA issuer: per 32-deep chunk one tcgen05.mma.kind::i8
//                 (M=128 N=128 K=32; or two kind::f16 K=16 on f16-widened
//                 codes), accumulate = 0 -- every chunk is a fresh partial
//                 because the reference promotes each 32-deep product
//                 separately -- into TMEM buffer (chunk % 4).
//   warps 2..17   promotion/epilogue: 32 columns x 32 TMEM lanes per warp
//                 (lane quarter = warp % 4).  Per chunk: tcgen05.ld the
//                 partials, release the buffer, promote in packed f32x2 ops:
//                   EXACT: acc = fl(acc + fl(fl(P*sa)*sb))   (bit-exact)
//                   FAST : acc = fma(P, sa*sb, acc)          (sa*sb exact)
//                 After the last chunk: +bias, 32x32 absmax, binary16
//                 scale, RNE codes.  FP32 never reaches HBM (except the FP32
//                 output kinds).
// Bounds per 128x128x32 chunk and SM: MMA 64 clk (i8) / 128
// (f16); TMEM read 64 KB at ~480 B/clk = 136 clk; exact promotion 3 rounded
// FP32 ops x 16384 / 128 lanes = 384 clk; fast 128 clk FMA + (i8 only) one
// I2F per element on the half-rate ALU pipe = 256 clk.
//
// Generic kernel (gemm_i8_kernel): any multiple-of-32 shape (partial tiles,
// scale grids read from global memory), and the int32 partials debug output.
#include <stdio.h>
#include <string.h>

#include "common.cuh"

namespace jf {
namespace gemm {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int BK = 128;  // K per stage (4 chunks)
constexpr int kChunksPerStage = BK / 32;
constexpr int kTmemBufs = 4;  // == kChunksPerStage: chunk c of a stage uses buffer c

enum OutKind { OUT_INT8 = 0, OUT_F32 = 1, OUT_INT8_DEQ = 2, OUT_I32 = 3 };
enum OpKind { OP_I8 = 0, OP_F16 = 1 };

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
  long long *trace;  // JF_GEMM_TRACE builds only: CTA-0 event clocks [8][512]
};

// Diagnostics (JF_GEMM_TRACE builds, `make trace`): clock64 of pipeline events of
// CTA 0's first 256 chunks (tools/gemm_trace.py): [0..2] MMA issuer (tempty wait
// start, buffer free, commit issued), [3..5] warp 2 (tfull wait start, full, data),
// [8 + w] promotion warp w's promotion end.
#ifdef JF_GEMM_TRACE
constexpr int kTrEv = 32, kTrChunks = 256;
#define JF_TR(ev, g)                                                                               \
  do {                                                                                             \
    if (blockIdx.x == 0 && (g) < kTrChunks && p.trace) p.trace[(ev) * kTrChunks + (g)] = clock64(); \
  } while (0)
#else
#define JF_TR(ev, g) \
  do {               \
  } while (0)
#endif

// Single-thread control roles (TMA producer, MMA issuer) wait with a suspend
// hint: they share SM sub-partitions with promotion warps and would otherwise
// steal their issue slots spinning.
JF_DEV void ctl_wait(uint32_t addr, uint32_t parity) { mbar_wait_u32_sleep(addr, parity, 200); }

// One lane of a converged warp (the control roles run their loops on all 32 lanes so
// the loop state stays warp-uniform -- uniform datapath, no per-chunk R2UR -- and
// issue each TMA / MMA / commit from the elected lane).
JF_DEV bool elect_one() {
  uint32_t p;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(p));
  return p != 0;
}

// The partials a tcgen05.ld wrote are only valid after tcgen05.wait::ld; make
// every consumer depend on the wait (the "+r" operands) so the compiler cannot
// hoist any use of them above it.
template <int N>
JF_DEV void tmem_wait_ld_dep(uint32_t (&r)[N]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < N; i += 8)
    asm volatile("" : "+r"(r[i]), "+r"(r[i + 1]), "+r"(r[i + 2]), "+r"(r[i + 3]), "+r"(r[i + 4]),
                 "+r"(r[i + 5]), "+r"(r[i + 6]), "+r"(r[i + 7]));
}

// Promote one 32-column block of partials into the FP32 accumulator.
// kF32: the partials are f32 bit patterns holding exact integers (kind::f16 path).
template <bool kFast, bool kF32>
JF_DEV void promote32(float *acc, const uint32_t *r, float sa, float sb, float zero) {
  auto val = [&](int j) { return kF32 ? __uint_as_float(r[j]) : __int2float_rn((int)r[j]); };
  if (kFast) {
    const float s = __fmul_rn(sa, sb);  // exact: 11 x 11 significant bits
#pragma unroll
    for (int j = 0; j < 32; j += 2) ffma2_rn(acc[j], acc[j + 1], val(j), val(j + 1), s, s, acc[j], acc[j + 1]);
  } else {
    // packed f32x2, every op an IEEE-rounded fp32 op in the reference order.
    // ptxas contracts mul.rn.f32x2 + add.rn.f32x2 into FFMA2 (not equivalent);
    // an fma with a runtime +0 addend is a correctly rounded product it cannot fuse.
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
      float t0, t1;
      fmul2_rn(t0, t1, val(j), val(j + 1), sa, sa);
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
    if ((reinterpret_cast<uintptr_t>(p.bias) & 15) == 0) {  // 8 broadcast 16-byte loads
      const float4 *b4 = reinterpret_cast<const float4 *>(p.bias + col0);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float4 b = __ldg(b4 + k);
        fadd2_rn(acc[4 * k], acc[4 * k + 1], acc[4 * k], acc[4 * k + 1], b.x, b.y);
        fadd2_rn(acc[4 * k + 2], acc[4 * k + 3], acc[4 * k + 2], acc[4 * k + 3], b.z, b.w);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = __fadd_rn(acc[j], __ldg(p.bias + col0 + j));
    }
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
  // XU-free requantization (common.cuh quant_codes32; the per-element FRND + F2I of
  // quant_code_fast, quarter rate, was the exposed part of every tile's epilogue)
  uint32_t w[8];
  quant_codes32(acc, sc, rc, quant_fast_ok(f, sc), p.zero, w);
  int8_t *dq = p.yq + row * p.N + col0;
  reinterpret_cast<uint4 *>(dq)[0] = make_uint4(w[0], w[1], w[2], w[3]);
  reinterpret_cast<uint4 *>(dq)[1] = make_uint4(w[4], w[5], w[6], w[7]);
  if (lane == 0) p.ys[I * (p.N >> 5) + J] = sc;
  if (p.out_kind == OUT_INT8_DEQ) {  // fl(code * sc), exact, PRMT + FFMA2 (no I2F)
    float *dst = p.yf + row * p.N + col0;
    const DeqScale k8 = deq_scale(sc);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float d[8];
      deq8_packed(w[2 * k], w[2 * k + 1], k8, d);
      *reinterpret_cast<float4 *>(dst + 8 * k) = make_float4(d[0], d[1], d[2], d[3]);
      *reinterpret_cast<float4 *>(dst + 8 * k + 4) = make_float4(d[4], d[5], d[6], d[7]);
    }
  }
  return lane == 0 ? f : 0;
}

struct Bars {
  uint64_t full[8];
  uint64_t empty[8];
  uint64_t tfull[kTmemBufs];
  uint64_t tempty[kTmemBufs];
  uint32_t tmem_base;
};

// ───────────────────────── gemm_tc_kernel (main) ─────────────────────────
// Operand staging per stage (4 chunks):
//   OP_I8 : A, B each one 128-row x 128-byte SW128 box (16 KB); K-major (row =
//           M/N index, 128 K bytes) or MN-major (row = K index, 128 M/N bytes;
//           the UMMA reads int8 MN-major tiles directly, so dgrad consumes W
//           [d x c] and wgrad dY [n x d], X [n x c] as stored).  6 stages.
//   OP_F16: A, B each two 128-row x 64-f16 SW128 boxes (32 KB), K-major.  3 stages.
// Scales: per stage the 4x4 sub-grids of sA (row blocks x chunks) and sB, 64 B
// each, by TMA into the stage's 256-byte scale slot.
constexpr int kEpiTC = 16;  // promotion warps of gemm_tc_kernel
// Chunks per tfull commit / wait: the MMA issuer commits tfull only after every
// kGroup-th chunk, and a commit covers all earlier MMAs of the issuing thread, so the
// promotion warps wait once per group.  Each commit costs ~68 clk of tensor pipe
// (r1e microbenchmark); per-chunk commits (1) measured 2-5% slower than pairs (2).
#ifndef JF_GEMM_GROUP
#define JF_GEMM_GROUP 2
#endif
constexpr int kGroup = JF_GEMM_GROUP;

template <int kOp>
struct Cfg {
  static constexpr int kStages = kOp == OP_I8 ? 6 : 3;
  static constexpr uint32_t kStageBytes = kOp == OP_I8 ? BM * BK : 2 * BM * BK;  // per operand
  static constexpr uint32_t kScaleBytes = 256;
  static constexpr size_t kSmem = 1024 + (size_t)kStages * 2 * kStageBytes + kStages * kScaleBytes + sizeof(Bars) + 64;
};

// Warp layout: warp 0 TMA producer (sub-partition 0), warp 1 MMA issuer
// (sub-partition 1), warps 2.. promotion.  Both control roles run their loops on
// the whole warp (uniform loop state) and issue from one elected lane: the MMA
// issuer shares sub-partition 1 with four promotion warps, and every instruction
// it needs per chunk is an issue slot they lose (tools/gemm_trace.py: with a
// lane-0-only issuer, sub-partition 1's warps trail the others by ~2 chunks and
// gate every TMEM buffer release).  Measured and NOT kept (profiles/r2_gemm_ab.md):
// one issuer per sub-partition (4 issuers, 20 warps) -- no skew, but slower;
// software-pipelined TMEM loads (spills at the 96-register cap of 18 warps);
// 64 columns per promotion warp (2 warps per sub-partition hide less latency).
template <int kOp, bool kFast, bool kAmn, bool kBmn>
__global__ void __launch_bounds__((2 + kEpiTC) * 32, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmSA, const __grid_constant__ CUtensorMap tmSB,
                   const Params p, const int saT, const int sbT) {
  using C = Cfg<kOp>;
  constexpr int kStages = C::kStages;
  constexpr int kEpi = kEpiTC;  // promotion warps
  constexpr int kCols = 32;     // columns per promotion warp
  constexpr int kBlk = 1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sA = base;
  uint8_t *sB = base + kStages * C::kStageBytes;
  uint8_t *sS = sB + kStages * C::kStageBytes;  // scale slots, 128-byte aligned
  Bars &S = *reinterpret_cast<Bars *>(sS + kStages * C::kScaleBytes);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t mt = p.M / BM, nt = p.N / BN;
  const int64_t ntiles = mt * nt;
  const int nstages_k = (int)(p.K / BK);
  const uint32_t bar_full = smem_u32(&S.full[0]), bar_empty = smem_u32(&S.empty[0]);
  const uint32_t bar_tfull = smem_u32(&S.tfull[0]), bar_tempty = smem_u32(&S.tempty[0]);
  // warp roles
  const int epi_w = warp - 2;  // promotion warp index
  const bool is_tma = warp == 0;
  const bool is_iss = warp == 1;
  const int alloc_warp = 1;

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    prefetch_tmap(&tmSA);
    prefetch_tmap(&tmSB);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], 1 + kEpi);  // the MMAs consumed the tiles AND every warp read the scales
    }
    for (int b = 0; b < kTmemBufs; ++b) {
      mbar_init(&S.tfull[b], 1);
      mbar_init(&S.tempty[b], kEpi);
    }
    fence_barrier_init();
  }
  if (warp == alloc_warp) tmem_alloc(&S.tmem_base, kTmemBufs * BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;

  // TMA loads of one stage (operand tiles + the 4x4 scale sub-grids)
  auto tma_stage = [&](int stage, int64_t tile, int ks) {
    const int m0 = (int)((tile % mt) * BM), n0 = (int)((tile / mt) * BN);
    mbar_arrive_expect_tx(&S.full[stage], 2 * C::kStageBytes + 128);
    uint8_t *a = sA + stage * C::kStageBytes, *b = sB + stage * C::kStageBytes;
    // tensor-map coordinates are {inner, outer}
    if constexpr (kOp == OP_F16) {
      tma_load_2d(a, &tmA, &S.full[stage], ks * BK, m0);
      tma_load_2d(a + C::kStageBytes / 2, &tmA, &S.full[stage], ks * BK + 64, m0);
      tma_load_2d(b, &tmB, &S.full[stage], ks * BK, n0);
      tma_load_2d(b + C::kStageBytes / 2, &tmB, &S.full[stage], ks * BK + 64, n0);
    } else {
      if (kAmn) tma_load_2d(a, &tmA, &S.full[stage], m0, ks * BK);
      else tma_load_2d(a, &tmA, &S.full[stage], ks * BK, m0);
      if (kBmn) tma_load_2d(b, &tmB, &S.full[stage], n0, ks * BK);
      else tma_load_2d(b, &tmB, &S.full[stage], ks * BK, n0);
    }
    uint8_t *ss = sS + stage * C::kScaleBytes;
    // box {4, 4}: K-contiguous grids -> [row block][chunk], else [chunk][row block]
    if (saT) tma_load_2d(ss, &tmSA, &S.full[stage], m0 / 32, ks * 4);
    else tma_load_2d(ss, &tmSA, &S.full[stage], ks * 4, m0 / 32);
    if (sbT) tma_load_2d(ss + 128, &tmSB, &S.full[stage], n0 / 32, ks * 4);
    else tma_load_2d(ss + 128, &tmSB, &S.full[stage], ks * 4, n0 / 32);
  };
  // one chunk's MMA(s): chunk c of stage `stage` -> TMEM buffer c
  const uint64_t adesc0 = smem_desc_sw128(smem_u32(sA), 16, 1024);
  const uint64_t bdesc0 = smem_desc_sw128(smem_u32(sB), 16, 1024);
  auto mma_chunk = [&](int stage, int c) {
    const uint64_t ad = adesc0 + (uint64_t)((stage * C::kStageBytes) >> 4);
    const uint64_t bd = bdesc0 + (uint64_t)((stage * C::kStageBytes) >> 4);
    if constexpr (kOp == OP_F16) {
      constexpr uint32_t idesc = idesc_f16_f32(BM, BN);
      // chunk c: box c/2, byte offset (c%2)*64 in the 128-byte row; K=16 step = 32 bytes
      const uint32_t off = ((c >> 1) * (C::kStageBytes / 2) + (c & 1) * 64) >> 4;
      mma_f16_ss(tmem + c * BN, ad + off, bd + off, idesc, 0u);
      mma_f16_ss(tmem + c * BN, ad + off + 2, bd + off + 2, idesc, 1u);
    } else {
      constexpr uint32_t idesc = idesc_i8(BM, BN, kAmn ? 1 : 0, kBmn ? 1 : 0);
      constexpr uint32_t kStepA = kAmn ? (32 * 128) >> 4 : 2;  // descriptor units (16 B) per chunk
      constexpr uint32_t kStepB = kBmn ? (32 * 128) >> 4 : 2;
      mma_i8_ss(tmem + c * BN, ad + kStepA * c, bd + kStepB * c, idesc, 0u);
    }
  };

  if (is_tma) {
    // ───────────── TMA producer (basic layout; whole warp, one elected lane issues) ─────────────
    {
      int stage = 0;
      uint32_t phase = 0;
#pragma unroll 1
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
#pragma unroll 1
        for (int ks = 0; ks < nstages_k; ++ks) {
          ctl_wait(bar_empty + 8 * stage, phase ^ 1);
          if (elect_one()) tma_stage(stage, tile, ks);
          __syncwarp();
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (is_iss) {
    // ───────────── single MMA issuer (whole warp): chunk c of every stage -> TMEM buffer c ─────────────
    {
      int stage = 0, gch = 0;
      uint32_t phase = 0, tphase = 0;
#pragma unroll 1
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
#pragma unroll 1
        for (int ks = 0; ks < nstages_k; ++ks) {
          ctl_wait(bar_full + 8 * stage, phase);
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < kChunksPerStage; ++c) {
            if (lane == 0) JF_TR(0, gch + c);
            ctl_wait(bar_tempty + 8 * c, ((tphase >> c) & 1) ^ 1);
            if (lane == 0) JF_TR(1, gch + c);
            tphase ^= 1u << c;
            tc_fence_after();
            if (lane == 0) JF_TR(6, gch + c);
            if (elect_one()) {
              mma_chunk(stage, c);
              if (c % kGroup == kGroup - 1) mma_commit(&S.tfull[c]);
            }
            __syncwarp();
            if (lane == 0) JF_TR(2, gch + c);
          }
          if (elect_one()) mma_commit(&S.empty[stage]);
          __syncwarp();
          gch += kChunksPerStage;
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else {
    // ───────────── promotion + epilogue ─────────────
    const int lq = warp & 3;              // TMEM lane quarter == 32-row block of the tile
    const int cg = epi_w >> 2;            // column group: columns [cg*kCols, +kCols)
    const uint32_t tcol = tmem + ((uint32_t)(lq * 32) << 16) + cg * kCols;
    const uint32_t ssa0 = smem_u32(sS), ssb0 = ssa0 + 128;
    // float offsets of this warp's scale factors inside the 4x4 boxes
    const uint32_t oa = saT ? (uint32_t)lq * 4 : (uint32_t)lq * 16;
    const uint32_t da = saT ? 16 : 4;  // byte step between chunks
    const uint32_t db = sbT ? 16 : 4;
    uint32_t tphase = 0;
    int flags = 0;
    int stage = 0;
    uint32_t phase = 0;
    constexpr bool kF32 = kOp == OP_F16;
    const bool trw = epi_w == 0 && lane == 0;
    int gch = 0;
#pragma unroll 1
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t I = (tile % mt) * (BM / 32) + lq;
      const int64_t J0 = (tile / mt) * (BN / 32) + cg * kBlk;
      float acc[kBlk][32];
#pragma unroll
      for (int q = 0; q < kBlk; ++q)
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[q][j] = 0.0f;
#pragma unroll 1
      for (int ks = 0; ks < nstages_k; ++ks) {
        // the stage's scales: acquire the TMA writes, read, release the stage
        mbar_wait_u32(bar_full + 8 * stage, phase);
        const uint32_t sa_addr = ssa0 + stage * C::kScaleBytes + oa;
        const uint32_t sb_addr = ssb0 + stage * C::kScaleBytes;
        float sav[4], sbv[kBlk][4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          sav[b] = lds_f32(sa_addr + b * da);
#pragma unroll
          for (int q = 0; q < kBlk; ++q)
            sbv[q][b] = lds_f32(sb_addr + (sbT ? (uint32_t)(cg * kBlk + q) * 4 : (uint32_t)(cg * kBlk + q) * 16) +
                                b * db);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_u32(bar_empty + 8 * stage);
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
#pragma unroll
        for (int b = 0; b < kTmemBufs; ++b) {
          uint32_t r[kCols];
          if (trw) JF_TR(3, gch + b);
          if (b % kGroup == 0) {  // the group's last chunk landed => the whole group did
            const int bl = b + kGroup - 1;
            mbar_wait_u32(bar_tfull + 8 * bl, (tphase >> bl) & 1);
            tphase ^= 1u << bl;
          }
          if (trw) JF_TR(4, gch + b);
          tc_fence_after();
          tmem_ld_32x32b_x32(tcol + b * BN, r);
          tmem_wait_ld_dep(r);
          if (trw) JF_TR(5, gch + b);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_u32(bar_tempty + 8 * b);
#pragma unroll
          for (int q = 0; q < kBlk; ++q) promote32<kFast, kF32>(acc[q], r + 32 * q, sav[b], sbv[q][b], p.zero);
#ifdef JF_GEMM_TRACE
          if (lane == 0 && epi_w < 16) JF_TR(8 + epi_w, gch + b + (int)(acc[0][0] == 1.2345f));  // (after the math)
#endif
        }
        gch += kTmemBufs;
      }
#pragma unroll
      for (int q = 0; q < kBlk; ++q) flags |= finish_block(p, acc[q], I, J0 + q, lane);
    }
    if (lane == 0) raise_flags(p.err, flags);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == alloc_warp) tmem_dealloc(tmem, kTmemBufs * BN);
}

// ───────────────────────── gemm_i8_kernel (generic shapes) ─────────────────────────
// Same pipeline, K-major A and B ([rows x K] codes, row stride a multiple of 16),
// scale grids read from global memory, partial tiles predicated.  kPartials:
// the raw int32 partials of a single chunk (jf_gemm_partials, micro_mm_16).
constexpr int kStagesG = 6;
constexpr int kEpiG = 16;
constexpr uint32_t kStageBytesG = BM * BK;
constexpr size_t kSmemG = 1024 + kStagesG * 2 * kStageBytesG + sizeof(Bars) + 64;

template <bool kFast, bool kPartials>
__global__ void __launch_bounds__((2 + kEpiG) * 32, 1)
    gemm_i8_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sA = base;
  uint8_t *sB = base + kStagesG * kStageBytesG;
  Bars &S = *reinterpret_cast<Bars *>(sB + kStagesG * kStageBytesG);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t mt = (p.M + BM - 1) / BM, nt = (p.N + BN - 1) / BN;
  const int64_t ntiles = mt * nt;
  const int nchunks = (int)(p.K / 32);
  const int nstages_k = (nchunks + kChunksPerStage - 1) / kChunksPerStage;
  const uint32_t bar_full = smem_u32(&S.full[0]), bar_empty = smem_u32(&S.empty[0]);
  const uint32_t bar_tfull = smem_u32(&S.tfull[0]), bar_tempty = smem_u32(&S.tempty[0]);

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < kStagesG; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], 1);
    }
    for (int b = 0; b < kTmemBufs; ++b) {
      mbar_init(&S.tfull[b], 1);
      mbar_init(&S.tempty[b], kEpiG);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&S.tmem_base, kTmemBufs * BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int m0 = (int)((tile % mt) * BM), n0 = (int)((tile / mt) * BN);
        for (int ks = 0; ks < nstages_k; ++ks) {
          ctl_wait(bar_empty + 8 * stage, phase ^ 1);
          mbar_arrive_expect_tx(&S.full[stage], 2 * kStageBytesG);
          tma_load_2d(sA + stage * kStageBytesG, &tmA, &S.full[stage], ks * BK, m0);
          tma_load_2d(sB + stage * kStageBytesG, &tmB, &S.full[stage], ks * BK, n0);
          if (++stage == kStagesG) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint64_t adesc0 = smem_desc_sw128(smem_u32(sA), 16, 1024);
      const uint64_t bdesc0 = smem_desc_sw128(smem_u32(sB), 16, 1024);
      constexpr uint32_t idesc = idesc_i8(BM, BN, 0, 0);
      int stage = 0;
      uint32_t phase = 0, tphase = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int ks = 0; ks < nstages_k; ++ks) {
          ctl_wait(bar_full + 8 * stage, phase);
          tc_fence_after();
          const uint64_t ad = adesc0 + (uint64_t)((stage * kStageBytesG) >> 4);
          const uint64_t bd = bdesc0 + (uint64_t)((stage * kStageBytesG) >> 4);
          const int nch = min(kChunksPerStage, nchunks - ks * kChunksPerStage);
#pragma unroll
          for (int c = 0; c < kChunksPerStage; ++c) {
            if (c < nch) {
              ctl_wait(bar_tempty + 8 * c, ((tphase >> c) & 1) ^ 1);
              tphase ^= 1u << c;
              tc_fence_after();
              mma_i8_ss(tmem + c * BN, ad + 2 * c, bd + 2 * c, idesc, 0u);
              mma_commit(&S.tfull[c]);
            }
          }
          mma_commit(&S.empty[stage]);
          if (++stage == kStagesG) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else {
    const int lq = warp & 3;
    const int cg = (warp - 2) >> 2;
    const uint32_t tcol = tmem + ((uint32_t)(lq * 32) << 16) + cg * 32;
    uint32_t tphase = 0;
    int flags = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t I = (tile % mt) * (BM / 32) + lq;
      const int64_t J = (tile / mt) * (BN / 32) + cg;
      const bool valid = I * 32 < p.M && J * 32 < p.N;
      float acc[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = 0.0f;
      const float *pa = p.sa + (kPartials || !valid ? 0 : I * p.sa_s0);
      const float *pb = p.sb + (kPartials || !valid ? 0 : J * p.sb_s0);
      for (int cb = 0; cb < nchunks; cb += kTmemBufs) {
        float sav[4] = {0.f, 0.f, 0.f, 0.f}, sbv[4] = {0.f, 0.f, 0.f, 0.f};
        if (!kPartials && valid) {
#pragma unroll
          for (int b = 0; b < kTmemBufs; ++b)
            if (cb + b < nchunks) {
              sav[b] = __ldg(pa + (cb + b) * p.sa_s1);
              sbv[b] = __ldg(pb + (cb + b) * p.sb_s1);
            }
        }
#pragma unroll
        for (int b = 0; b < kTmemBufs; ++b) {
          if (cb + b >= nchunks) break;
          mbar_wait_u32(bar_tfull + 8 * b, (tphase >> b) & 1);
          tphase ^= 1u << b;
          tc_fence_after();
          uint32_t r[32];
          tmem_ld_32x32b_x32(tcol + b * BN, r);
          tmem_wait_ld_dep(r);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_u32(bar_tempty + 8 * b);
          if (kPartials) {
            if (valid) {
              int32_t *dst = reinterpret_cast<int32_t *>(p.yf) + (I * 32 + lane) * p.N + J * 32;
#pragma unroll
              for (int j = 0; j < 32; j += 4)
                *reinterpret_cast<int4 *>(dst + j) = make_int4((int)r[j], (int)r[j + 1], (int)r[j + 2], (int)r[j + 3]);
            }
          } else {
            promote32<kFast, false>(acc, r, sav[b], sbv[b], p.zero);
          }
        }
      }
      if (!kPartials && valid) flags |= finish_block(p, acc, I, J, lane);
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

}  // namespace gemm
}  // namespace jf

// ─────────────────────────── host side ───────────────────────────
using namespace jf;

int jf_launch_check(const char *what);
void jf_set_error(const char *msg);
int jf_num_sms();
int jf_set_smem_attr(const void *func, int bytes, const char *what);
bool jf_make_tmap_i8(CUtensorMap *map, const void *ptr, int64_t rows, int64_t cols, int64_t ld,
                     int box_cols, int box_rows, bool swizzle128);
bool jf_make_tmap_f32(CUtensorMap *map, const void *ptr, int64_t rows, int64_t cols, int64_t ld,
                      int box_cols, int box_rows);
bool jf_make_tmap_f16(CUtensorMap *map, const void *ptr, int64_t rows, int64_t cols, int64_t ld,
                      int box_cols, int box_rows);

// Launch options (diagnostics / A-B experiments; results are bit-identical for every
// option), set at run time by jf_gemm_set_option().  Defaults are the measured best.
struct GemmOptions {
  int tma_scales = 1;  // 0: every shape on the generic kernel
};
static GemmOptions g_opt;

extern "C" int jf_gemm_set_option(const char *key, int value) {
  if (!strcmp(key, "tma_scales")) g_opt.tma_scales = value;
  else return JF_ERR_ARG;
  return JF_OK;
}

#ifdef JF_GEMM_TRACE
static long long *g_trace = nullptr;
extern "C" int jf_gemm_trace_read(long long *host) {
  if (!g_trace) return 1;
  return cudaMemcpy(host, g_trace, gemm::kTrEv * gemm::kTrChunks * sizeof(long long), cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 2;
}
#endif

namespace {
using TcFn = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const CUtensorMap, const gemm::Params,
                      const int, const int);

template <int kOp, bool kAmn, bool kBmn>
TcFn pick_tc_mode(bool fast) {
  using namespace jf::gemm;
  return fast ? gemm_tc_kernel<kOp, true, kAmn, kBmn> : gemm_tc_kernel<kOp, false, kAmn, kBmn>;
}

bool grid_ok(const float *s, int64_t s0, int64_t s1) {
  return ((uintptr_t)s % 16 == 0) && ((s1 == 1 && s0 % 4 == 0) || (s0 == 1 && s1 % 4 == 0));
}

// gemm_tc_kernel launch.  OP_I8: A is [M x K] (K-major) or [K x M] (a_mn: MN-major),
// row stride lda elements; likewise B as [N x K] or [K x N].  OP_F16: K-major only.
// Returns -1 when the shape or the scale-grid layout does not qualify (caller falls back).
int launch_tc(int op, const void *A, bool a_mn, int64_t lda, const void *B, bool b_mn, int64_t ldb, int64_t M,
              int64_t N, int64_t K, const float *sa, int64_t sa_s0, int64_t sa_s1, const float *sb, int64_t sb_s0,
              int64_t sb_s1, const float *bias, int mode, int out_kind, int8_t *yq, float *ys, void *yf,
              int32_t *err, cudaStream_t stream) {
  using namespace jf::gemm;
  if (!g_opt.tma_scales || out_kind == OUT_I32 || M % 128 || N % 128 || K % 128 || lda % 16 || ldb % 16 ||
      (uintptr_t)A % 16 || (uintptr_t)B % 16 || !grid_ok(sa, sa_s0, sa_s1) || !grid_ok(sb, sb_s0, sb_s1))
    return -1;
  if (op == OP_F16 && (a_mn || b_mn)) return -1;
  const int64_t kb = K / 32;
  const int saT = sa_s1 != 1, sbT = sb_s1 != 1;
  CUtensorMap ta, tb, tsa, tsb;
  bool ok;
  if (op == OP_F16) {
    ok = jf_make_tmap_f16(&ta, A, M, K, lda, 64, BM) && jf_make_tmap_f16(&tb, B, N, K, ldb, 64, BN);
  } else {
    ok = (a_mn ? jf_make_tmap_i8(&ta, A, K, M, lda, BM, BK, true) : jf_make_tmap_i8(&ta, A, M, K, lda, BK, BM, true)) &&
         (b_mn ? jf_make_tmap_i8(&tb, B, K, N, ldb, BN, BK, true) : jf_make_tmap_i8(&tb, B, N, K, ldb, BK, BN, true));
  }
  ok = ok &&
       (saT ? jf_make_tmap_f32(&tsa, sa, kb, M / 32, sa_s1, 4, 4) : jf_make_tmap_f32(&tsa, sa, M / 32, kb, sa_s0, 4, 4)) &&
       (sbT ? jf_make_tmap_f32(&tsb, sb, kb, N / 32, sb_s1, 4, 4) : jf_make_tmap_f32(&tsb, sb, N / 32, kb, sb_s0, 4, 4));
  if (!ok) return JF_ERR_LAUNCH;
  Params p{M, N, K, sa, sa_s0, sa_s1, sb, sb_s0, sb_s1, bias, yq, ys, (float *)yf, err, out_kind, 0.0f, nullptr};
#ifdef JF_GEMM_TRACE
  if (!g_trace) cudaMalloc(&g_trace, gemm::kTrEv * gemm::kTrChunks * sizeof(long long));
  cudaMemsetAsync(g_trace, 0, gemm::kTrEv * gemm::kTrChunks * sizeof(long long), stream);
  p.trace = g_trace;
#endif
  const bool fast = mode == JF_MODE_FAST;
  TcFn k;
  size_t smem;
  if (op == OP_F16) {
    k = pick_tc_mode<OP_F16, false, false>(fast);
    smem = Cfg<OP_F16>::kSmem;
  } else {
    if (!a_mn && !b_mn) k = pick_tc_mode<OP_I8, false, false>(fast);
    else if (!a_mn && b_mn) k = pick_tc_mode<OP_I8, false, true>(fast);
    else if (a_mn && b_mn) k = pick_tc_mode<OP_I8, true, true>(fast);
    else return -1;
    smem = Cfg<OP_I8>::kSmem;
  }
  if (int rc = jf_set_smem_attr((const void *)k, (int)smem, "gemm_tc attr")) return rc;
  const int64_t tiles = (M / BM) * (N / BN);
  const int grid = (int)(tiles < jf_num_sms() ? tiles : jf_num_sms());
  const int threads = (2 + kEpiTC) * 32;
  k<<<grid, threads, smem, stream>>>(ta, tb, tsa, tsb, p, saT, sbT);
  return jf_launch_check("gemm_tc");
}
}  // namespace

// Core launcher: A [M x K] (row stride lda), Bt [N x K] (row stride ldb), both K-major codes.
int jf_gemm_launch(const int8_t *A, int64_t lda, const int8_t *Bt, int64_t ldb, int64_t M, int64_t N, int64_t K,
                   const float *sa, int64_t sa_s0, int64_t sa_s1, const float *sb, int64_t sb_s0, int64_t sb_s1,
                   const float *bias, int mode, int out_kind, int8_t *yq, float *ys, void *yf, int32_t *err,
                   cudaStream_t stream) {
  using namespace jf::gemm;
  if (M <= 0 || N <= 0 || K <= 0 || M % 32 || N % 32 || K % 32 || lda % 16 || ldb % 16) {
    jf_set_error("gemm: dims must be positive multiples of 32, strides multiples of 16");
    return JF_ERR_ARG;
  }
  const bool partials = out_kind == OUT_I32;
  if (!partials) {
    const int rc = launch_tc(OP_I8, A, false, lda, Bt, false, ldb, M, N, K, sa, sa_s0, sa_s1, sb, sb_s0, sb_s1, bias,
                             mode, out_kind, yq, ys, yf, err, stream);
    if (rc >= 0) return rc;
  }
  CUtensorMap ta, tb;
  if (!jf_make_tmap_i8(&ta, A, M, K, lda, BK, BM, true) || !jf_make_tmap_i8(&tb, Bt, N, K, ldb, BK, BN, true))
    return JF_ERR_LAUNCH;
  Params p{M, N, K, sa, sa_s0, sa_s1, sb, sb_s0, sb_s1, bias, yq, ys, (float *)yf, err, out_kind, 0.0f, nullptr};
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int grid = (int)(tiles < jf_num_sms() ? tiles : jf_num_sms());
  const bool fast = mode == JF_MODE_FAST;
  void (*kern)(const CUtensorMap, const CUtensorMap, const Params) =
      partials ? gemm_i8_kernel<false, true> : (fast ? gemm_i8_kernel<true, false> : gemm_i8_kernel<false, false>);
  if (int rc = jf_set_smem_attr((const void *)kern, (int)kSmemG, "gemm attr")) return rc;
  kern<<<grid, (2 + kEpiG) * 32, kSmemG, stream>>>(ta, tb, p);
  return jf_launch_check("gemm_i8");
}

extern "C" int jf_gemm_fwd(const int8_t *x, const float *xs, const int8_t *w, const float *ws, const float *bias,
                           int64_t n, int64_t c, int64_t d, int32_t mode, int32_t out_kind, int8_t *yq, float *ys,
                           float *yf, int32_t *err, jf_stream_t stream) {
  const int64_t cb = c / 32;
  return jf_gemm_launch(x, c, w, c, n, d, c, xs, cb, 1, ws, cb, 1, bias, mode, out_kind, yq, ys, yf, err,
                        (cudaStream_t)stream);
}

extern "C" size_t jf_gemm_scratch_bytes(int32_t which, int64_t n, int64_t d, int64_t c) {
  if (which == 1) return (size_t)(c * d);
  return (size_t)(n * d + n * c);
}

extern "C" int jf_gemm_dgrad(const int8_t *dy, const float *dys, const int8_t *w, const float *ws, const int8_t *wt,
                             const float *wts, int64_t n, int64_t d, int64_t c, int32_t mode, int32_t out_kind,
                             int8_t *dxq, float *dxs, float *dxf, void *scratch, int32_t *err, jf_stream_t stream) {
  using namespace jf::gemm;
  // W [d x c] is the MN-major B operand as stored (no W^T needed)
  {
    const int rc = launch_tc(OP_I8, dy, false, d, w, true, c, n, c, d, dys, d / 32, 1, ws, 1, c / 32, nullptr, mode,
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
    return jf_gemm_launch(dy, d, wt, d, n, c, d, dys, d / 32, 1, wts, d / 32, 1, nullptr, mode, out_kind, dxq, dxs,
                          dxf, err, (cudaStream_t)stream);
  return jf_gemm_launch(dy, d, wt, d, n, c, d, dys, d / 32, 1, ws, 1, c / 32, nullptr, mode, out_kind, dxq, dxs, dxf,
                        err, (cudaStream_t)stream);
}

extern "C" int jf_gemm_wgrad(const int8_t *dy, const float *dys, const int8_t *x, const float *xs, const int8_t *dyt,
                             const float *dyts, const int8_t *xt, const float *xts, int64_t n, int64_t d, int64_t c,
                             int32_t mode, int32_t out_kind, int8_t *dwq, float *dws, float *dwf, void *scratch,
                             int32_t *err, jf_stream_t stream) {
  using namespace jf::gemm;
  // dY [n x d] and X [n x c] are the MN-major A and B operands as stored (no transposes)
  {
    const int rc = launch_tc(OP_I8, dy, true, d, x, true, c, d, c, n, dys, 1, d / 32, xs, 1, c / 32, nullptr, mode,
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
  return jf_gemm_launch(dyt, n, xt, n, d, c, n, sa, sa0, sa1, sb, sb0, sb1, nullptr, mode, out_kind, dwq, dws, dwf,
                        err, (cudaStream_t)stream);
}

extern "C" int jf_gemm_partials(const int8_t *a, const int8_t *bt, int64_t m, int64_t n, int64_t k, int64_t kblk,
                                int32_t *out, jf_stream_t stream) {
  if (kblk < 0 || kblk * 32 >= k) return JF_ERR_ARG;
  // K restricted to one chunk via pointer offset + row stride = k
  return jf_gemm_launch(a + kblk * 32, k, bt + kblk * 32, k, m, n, 32, nullptr, 0, 0, nullptr, 0, 0, nullptr,
                        JF_MODE_EXACT, jf::gemm::OUT_I32, nullptr, nullptr, out, nullptr, (cudaStream_t)stream);
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
                           int64_t k, int32_t mode, int32_t out_kind, int8_t *yq, float *ys, float *yf, int32_t *err,
                           jf_stream_t stream) {
  using namespace jf::gemm;
  if (m <= 0 || n <= 0 || k <= 0 || out_kind == OUT_I32) {
    jf_set_error("gemm_f16: dims must be positive");
    return JF_ERR_ARG;
  }
  const int rc = launch_tc(OP_F16, a, false, k, b, false, k, m, n, k, sa, sa_s0, sa_s1, sb, sb_s0, sb_s1, bias, mode,
                           out_kind, yq, ys, yf, err, (cudaStream_t)stream);
  if (rc < 0) {
    jf_set_error("gemm_f16: dims must be multiples of 128, scale grids contiguous along one axis");
    return JF_ERR_ARG;
  }
  return rc;
}
