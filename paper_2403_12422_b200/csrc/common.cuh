// common.cuh — shared device helpers for libjetfire (sm_100a only).
//
// Numerics follow the reference bit-for-bit (see oracle/int8flow_oracle.py):
// no FMA contraction (explicit __f*_rn intrinsics; the library is built
// with -fmad=false as a second guard), IEEE division in the quantizer,
// round-half-even via __float2int_rn, binary16 RNE scale snapping.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/jetfire.h"

#define JF_DEV __device__ __forceinline__

namespace jf {

constexpr int kBlock = 32;
constexpr int kQmax = 127;

// ── error word ──────────────────────────────────────────────────────────
JF_DEV void raise_flags(int32_t *err, int flags) {
  if (flags && err) atomicOr(err, flags);
}

// ── quantizer scale rule (qtensor.py:198-211) ──────────────────────────
// amax_bits: bit pattern of max|x| over the block, computed as an integer
// max of (bits & 0x7fffffff): any NaN/Inf makes it >= 0x7f800000, which is
// how np.abs(...).max() propagates non-finite values (qtensor.py:239-241).
JF_DEV float block_scale(uint32_t amax_bits, int &flags) {
  if (amax_bits >= 0x7f800000u) {
    flags |= JF_EFLAG_NONFINITE;
    return 1.0f;
  }
  if (amax_bits == 0u) return 1.0f;  // all-zero block -> scale 1
  const float am = __uint_as_float(amax_bits);
  const float raw = __fdiv_rn(am, 127.0f);
  const float s = __half2float(__float2half_rn(raw));  // binary16 RNE snap
  if (isinf(s)) {
    flags |= JF_EFLAG_OVERFLOW;
    return 1.0f;
  }
  return s == 0.0f ? 5.9604644775390625e-08f /* 2**-24 */ : s;
}

// q = clip(rint(x / s), -127, 127) with a true IEEE division (qtensor.py:243-245)
JF_DEV int quant_code(float x, float s) {
  int q = __float2int_rn(__fdiv_rn(x, s));
  q = q > kQmax ? kQmax : q;
  q = q < -kQmax ? -kQmax : q;
  return q;
}

// Same result as quant_code, without a division on the common path:
// y = fl(x * r), r = fl(1/s).  |y - fl(x/s)| <= 1.5 * 2^-23 * |x/s| <= 2.3e-5
// (|x/s| <= 128), so unless y lies within 3e-5 of a half-integer, y and
// fl(x/s) are on the same side of every rounding boundary and fl(x/s) is not a
// tie: rint(y) == rint(fl(x/s)).  The rare near-tie case takes the exact path.
JF_DEV int quant_code_fast(float x, float s, float r) {
  const float y = __fmul_rn(x, r);
  const float d = fabsf(__fsub_rn(__fsub_rn(y, floorf(y)), 0.5f));
  int q = (d > 3.0e-5f) ? __float2int_rn(y) : __float2int_rn(__fdiv_rn(x, s));
  q = q > kQmax ? kQmax : q;
  q = q < -kQmax ? -kQmax : q;
  return q;
}

// quant_code_fast's common path only: the code of fl(x * r), and `tie` raised when
// y is within 3e-5 of a half-integer (the caller then redoes the element with
// quant_code_fast).  Straight-line code: no per-element branch / reconvergence,
// and no XU-pipe instruction (the quarter-rate XU pipe -- F2I, FRND, I2F -- was the
// saturated unit of the memory-bound kernels, ncu r2): round-half-even to an
// integer by adding 1.5 * 2^23 (|y| <= 128 << 2^22: the sum's ulp is 1), the code
// read from the sum's low mantissa bits, the distance to the rounded value exact.
JF_DEV int quant_code_try(float x, float r, bool &tie) {
  const float y = __fmul_rn(x, r);
  const float t = __fadd_rn(y, 12582912.0f);  // 1.5 * 2^23
  const float e = __fsub_rn(y, __fsub_rn(t, 12582912.0f));  // y - rint(y), exact
  tie = tie || !(fabsf(e) < 0.49997f);
  int q = __float_as_int(t) - 0x4B400000;
  q = q > kQmax ? kQmax : q;
  q = q < -kQmax ? -kQmax : q;
  return q;
}

// Exact dequantization fl(code * s) without an int->float conversion (XU pipe):
// the biased code byte u = code + 128 goes into bits 8..15 of 0x4B000000, i.e. the
// float f = 2^23 + 2^15 + 256 * code exactly; then
//   fma(f, s * 2^-8, -(2^15 + 2^7) * s) = fl(code * s)
// with one rounding (s * 2^-8 and the 20-bit constant are exact).  PRMT + FFMA.
struct DeqScale {
  float s8, c;
};
JF_DEV uint32_t prmt_raw(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
JF_DEV DeqScale deq_scale(float s) { return {__fmul_rn(s, 0.00390625f), __fmul_rn(-32896.0f, s)}; }
JF_DEV float deq_code(uint32_t biased_word, int j, DeqScale k) {
  uint32_t bits;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(bits) : "r"(biased_word), "r"(0x4B000000u), "r"(0x7404u | (j << 4)));
  return __fmaf_rn(__uint_as_float(bits), k.s8, k.c);
}
// ── packed / 3-input helpers of the tile kernels ──────────────────────
// fp32x2 ops (defined below the PTX wrappers) are forward-declared here.
JF_DEV void ffma2_rn(float &d0, float &d1, float a0, float a1, float b0, float b1, float c0, float c1);
JF_DEV void fadd2_rn(float &d0, float &d1, float a0, float a1, float b0, float b1);
JF_DEV void fsub2_rn(float &d0, float &d1, float a0, float a1, float b0, float b1);

// max(|a|, |b|, |c|), NaN if any input is NaN (3-input max, sm_100).
JF_DEV float absmax3_nan(float a, float b, float c) {
  float d;
  asm("max.NaN.abs.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// +0.0f from constant memory: a value neither NVVM nor ptxas can fold (the host could
// rewrite it), used as the addend that turns a packed product into an FFMA2 (no mul/add
// contraction).  A constant-cache hit -- not the uncached L2 round trip a volatile
// global read costs on every tile's critical path.
__constant__ float c_opaque_zero = 0.0f;
JF_DEV float opaque_zero() { return c_opaque_zero; }

// 8 codes (two words) -> v[0..7], exact: PRMT into a 2^23 mantissa + packed FFMA2.
JF_DEV void deq8_packed(uint32_t w0, uint32_t w1, DeqScale k, float *v) {
  const uint32_t u[2] = {w0 ^ 0x80808080u, w1 ^ 0x80808080u};
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int j = 0; j < 4; j += 2) {
      const uint32_t b0 = prmt_raw(u[h], 0x4B000000u, 0x7404u | (j << 4));
      const uint32_t b1 = prmt_raw(u[h], 0x4B000000u, 0x7404u | ((j + 1) << 4));
      ffma2_rn(v[4 * h + j], v[4 * h + j + 1], __uint_as_float(b0), __uint_as_float(b1), k.s8, k.s8, k.c, k.c);
    }
}

// 4 codes of a word -> v[0..3]
JF_DEV void deq4(uint32_t word, DeqScale k, float *v) {
  const uint32_t u = word ^ 0x80808080u;
#pragma unroll
  for (int j = 0; j < 4; ++j) v[j] = deq_code(u, j, k);
}

JF_DEV uint32_t abs_bits(float x) { return __float_as_uint(x) & 0x7fffffffu; }

// pack 4 codes into one 32-bit word (little-endian byte order = column order)
JF_DEV uint32_t pack4(int a, int b, int c, int d) {
  return (uint32_t)(a & 0xff) | ((uint32_t)(b & 0xff) << 8) | ((uint32_t)(c & 0xff) << 16) |
         ((uint32_t)(d & 0xff) << 24);
}

JF_DEV float code_at(uint32_t word, int i) {
  return (float)(int8_t)((word >> (8 * i)) & 0xffu);
}

// ── numpy float32 pairwise summation (documented in the oracle) ─────────
// Sum of v[0..n) read through an accessor, in numpy's exact order.
template <typename Get>
JF_DEV float pairwise_leaf(Get get, int base, int n) {
  if (n < 8) {
    float r = 0.0f;
    for (int i = 0; i < n; ++i) r = __fadd_rn(r, get(base + i));
    return r;
  }
  float r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = get(base + j);
  int i = 8;
  const int lim = n - (n % 8);
  for (; i < lim; i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __fadd_rn(r[j], get(base + i + j));
  }
  float res = __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                        __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __fadd_rn(res, get(base + i));
  return res;
}

// Full recursion (n > 128 splits at n2 = n/2 - (n/2)%8).  Depth is small
// (log2(n/128)); written iteratively via an explicit stack.
template <typename Get>
JF_DEV float pairwise_sum(Get get, int base, int n) {
  if (n <= 128) return pairwise_leaf(get, base, n);
  // post-order evaluation with an explicit stack of (base, n, state)
  struct Frame {
    int base, n, state;
    float left;
  };
  Frame st[24];
  int sp = 0;
  st[0] = {base, n, 0, 0.0f};
  float ret = 0.0f;
  while (true) {
    Frame &f = st[sp];
    if (f.n <= 128) {
      ret = pairwise_leaf(get, f.base, f.n);
      if (sp == 0) return ret;
      --sp;
      continue;  // ret flows to parent
    }
    int n2 = f.n / 2;
    n2 -= n2 % 8;
    if (f.state == 0) {
      f.state = 1;
      st[++sp] = {f.base, n2, 0, 0.0f};
    } else if (f.state == 1) {
      f.left = ret;
      f.state = 2;
      st[++sp] = {f.base + n2, f.n - n2, 0, 0.0f};
    } else {
      ret = __fadd_rn(f.left, ret);
      if (sp == 0) return ret;
      --sp;
    }
  }
}

// ── PTX wrappers: mbarrier, TMA, tcgen05 ───────────────────────────────
JF_DEV uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

JF_DEV void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

JF_DEV void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

JF_DEV void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

JF_DEV void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

JF_DEV bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

JF_DEV void mbar_wait(uint64_t *bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// Address-based variants (shared-window u32 addresses precomputed once).
JF_DEV void mbar_wait_u32(uint32_t addr, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "JF_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra JF_WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// Same, with a suspend-time hint: single-thread producer roles sleep in the
// barrier instead of spinning (they would otherwise steal issue slots from
// the promotion warps sharing their SM sub-partition).
JF_DEV void mbar_wait_u32_sleep(uint32_t addr, uint32_t parity, uint32_t hint_ns) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "JF_WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra JF_WAITS_%=;\n\t}" ::"r"(addr),
      "r"(parity), "r"(hint_ns)
      : "memory");
}

// Non-blocking phase test.
JF_DEV bool mbar_test_u32(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}

JF_DEV void mbar_arrive_u32(uint32_t addr) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(addr) : "memory");
}

JF_DEV void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

JF_DEV void prefetch_tmap(const CUtensorMap *map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

JF_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
JF_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// TMEM allocation (whole warp).  Writes the base address to smem *dst.
JF_DEV void tmem_alloc(uint32_t *dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

JF_DEV void tmem_dealloc(uint32_t addr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(addr), "r"(ncols)
               : "memory");
}

// tcgen05.mma kind::i8, A and B from shared memory descriptors, D (int32) in TMEM.
JF_DEV void mma_i8_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                      uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrive on an mbarrier once all previously issued tcgen05 async ops of this thread complete.
JF_DEV void mma_commit(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

JF_DEV void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
JF_DEV void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 32 lanes x 32 consecutive 32-bit columns: thread i gets TMEM lane (base_lane + i).
JF_DEV void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

// Fill 32 consecutive columns of the warp's 32 lanes with one 32-bit value
// (4 x .x8 stores: only 8 registers of the constant are live).
JF_DEV void tmem_ld_32x32b_x64(uint32_t taddr, uint32_t (&r)[64]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, "
      "%32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, "
      "%48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63}, [%64];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
        "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]),
        "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]),
        "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]),
        "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]),
        "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr));
}

JF_DEV void tmem_fill_32x32b_x32(uint32_t taddr, uint32_t v) {
#pragma unroll
  for (int k = 0; k < 4; ++k)
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(
            taddr + 8 * k),
        "r"(v)
        : "memory");
}

// ── packed FP32x2 arithmetic (sm_100 FFMA2 / FMUL2 / FADD2) ───────────
// Two IEEE fp32 operations per instruction, each correctly rounded exactly
// like its scalar __f*_rn counterpart (no contraction across the pair).
JF_DEV void ffma2_rn(float &d0, float &d1, float a0, float a1, float b0, float b1, float c0, float c1) {
  asm("{\n\t.reg .b64 a, b, c, d;\n\t"
      "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\tmov.b64 c, {%6, %7};\n\t"
      "fma.rn.f32x2 d, a, b, c;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
JF_DEV void fmul2_rn(float &d0, float &d1, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 a, b, d;\n\t"
      "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "mul.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
JF_DEV void fadd2_rn(float &d0, float &d1, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 a, b, d;\n\t"
      "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "add.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
JF_DEV void fsub2_rn(float &d0, float &d1, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 a, b, d;\n\t"
      "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "sub.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

// ── UMMA descriptors ───────────────────────────────────────────────────
// Shared-memory matrix descriptor (sm_100 "version 1"), 128B swizzle.
//   bits [0,14)  start address >> 4
//   bits [16,30) leading byte offset >> 4
//   bits [32,46) stride byte offset >> 4
//   bits [46,48) version = 1
//   bits [61,64) layout: 2 = SWIZZLE_128B
JF_DEV uint64_t smem_desc_sw128(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fffu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3fffu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3fffu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Instruction descriptor for kind::i8: s8 x s8 -> s32, M x N, operand majors.
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n, int a_mn_major, int b_mn_major) {
  return (2u << 4)                        // D format: S32
         | (1u << 7)                      // A: signed 8-bit
         | (1u << 10)                     // B: signed 8-bit
         | ((uint32_t)a_mn_major << 15)   // A major
         | ((uint32_t)b_mn_major << 16)   // B major
         | ((uint32_t)(n >> 3) << 17)     // N / 8
         | ((uint32_t)(m >> 4) << 24);    // M / 16
}

// Instruction descriptor for kind::f16: f16 x f16 -> f32, both K-major.
__host__ __device__ constexpr uint32_t idesc_f16_f32(int m, int n) {
  return (1u << 4)                        // D format: F32
         | (0u << 7)                      // A: F16
         | (0u << 10)                     // B: F16
         | ((uint32_t)(n >> 3) << 17)     // N / 8
         | ((uint32_t)(m >> 4) << 24);    // M / 16
}

// tcgen05.mma kind::f16 (f16 operands from shared memory, f32 accumulator in TMEM).
JF_DEV void mma_f16_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Generic-proxy shared-memory writes -> visible to the async proxy (tensor core, TMA).
JF_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

JF_DEV uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

// 4 int8 codes -> 2 f16x2 words, exactly (|code| <= 128 is exact in binary16):
// byte b -> half with bits 0x64|(b^0x80) = 1152 + code, minus 1152.
JF_DEV void i8x4_to_f16x4(uint32_t w, uint32_t &lo, uint32_t &hi) {
  const uint32_t u = w ^ 0x80808080u;
  const uint32_t magic = 0x64806480u;  // {1152, 1152} as f16x2
  uint32_t a = prmt(u, 0x64646464u, 0x4140u);
  uint32_t b = prmt(u, 0x64646464u, 0x4342u);
  asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(lo) : "r"(a), "r"(magic));
  asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(hi) : "r"(b), "r"(magic));
}

JF_DEV uint2 lds64(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}
JF_DEV float lds_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}
JF_DEV uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
JF_DEV void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}


// Codes of one row of a 32x32 block, 32 values v (scale sc, rc = fl(1/sc)), without
// XU-pipe ops: per 8 values y = fl(v * rc) (an FFMA2 with the opaque +0 `zero`, so it
// is a rounded product) and t = fl(y + 1.5*2^23) in packed ops; the code bytes are t's
// low bytes (t = 1.5*2^23 + rint(y) exactly, |y| < 2^22).  That equals the reference's
// clip(rint(v / sc)) when the scale is a normal binary16 value (`fast_ok`; then
// |v/sc| <= 127 * (1 + 2^-11) < 127.5 and the clip is a no-op) and no y lies within 3e-5
// of a half-integer (|y - fl(v/sc)| <= 2.3e-5, quant_code_fast's argument); otherwise
// those 8 values take quant_code_fast (FRND + F2I + IEEE division on the rare path).
JF_DEV void quant_codes32(const float *v, float sc, float rc, bool fast_ok, float zero, uint32_t (&w)[8]) {
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    float tt[8], emax = 0.0f;
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      float y0, y1, u0, u1, e0, e1;
      ffma2_rn(y0, y1, v[8 * h + j], v[8 * h + j + 1], rc, rc, zero, zero);
      fadd2_rn(tt[j], tt[j + 1], y0, y1, 12582912.0f, 12582912.0f);
      fsub2_rn(u0, u1, tt[j], tt[j + 1], 12582912.0f, 12582912.0f);
      fsub2_rn(e0, e1, y0, y1, u0, u1);
      emax = absmax3_nan(emax, e0, e1);
    }
    if (fast_ok && emax < 0.49997f) {
      w[2 * h] = prmt(prmt(__float_as_uint(tt[0]), __float_as_uint(tt[1]), 0x0040u),
                      prmt(__float_as_uint(tt[2]), __float_as_uint(tt[3]), 0x0040u), 0x5410u);
      w[2 * h + 1] = prmt(prmt(__float_as_uint(tt[4]), __float_as_uint(tt[5]), 0x0040u),
                          prmt(__float_as_uint(tt[6]), __float_as_uint(tt[7]), 0x0040u), 0x5410u);
    } else {
#pragma unroll
      for (int k = 2 * h; k < 2 * h + 2; ++k)
        w[k] = pack4(quant_code_fast(v[4 * k], sc, rc), quant_code_fast(v[4 * k + 1], sc, rc),
                     quant_code_fast(v[4 * k + 2], sc, rc), quant_code_fast(v[4 * k + 3], sc, rc));
    }
  }
}

// flags == 0 and a normal binary16 scale: quant_codes32's fast path may apply
JF_DEV bool quant_fast_ok(int flags, float sc) { return flags == 0 && sc >= 6.103515625e-05f; }

}  // namespace jf
