// microbench.cu — B200 pipe measurements that decide the GEMM promotion design.
//
// Prints one JSON line per measurement: FP32 pipe rates (FFMA, FFMA2, FMUL,
// FADD, I2FP), TMEM ld/st bandwidth, raw tcgen05.mma kind::i8 rate, and the
// per-element cost of each promotion variant fed from TMEM (no MMA).
// Build: make microbench  (-> ../microbench).  Run on one B200.
#include <stdio.h>

#include <algorithm>
#include <vector>

#include "common.cuh"

using namespace jf;

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));   \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

constexpr int ITERS = 4096;

// ── FP32 pipe rates ────────────────────────────────────────────────────
template <int OP>
__global__ void __launch_bounds__(1024, 1) fp_kernel(float *out, long long *cyc, float a, float b) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0.001f + i;
  int xi[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) xi[i] = threadIdx.x + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) x[i] = __fmaf_rn(x[i], a, b);
      if (OP == 1) x[i] = __fmul_rn(x[i], a);
      if (OP == 2) x[i] = __fadd_rn(x[i], b);
      if (OP == 3) {  // I2FP chain through integers
        x[i] = __int2float_rn(xi[i]);
        xi[i] = __float_as_int(x[i]) ^ it;
      }
    }
    if (OP == 5) {  // MUFU.EX2: 8 independent chains
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
    }
    if (OP == 6) {  // F2FP.BF16.F32.PACK_AB (cvt.rn.bf16x2.f32): 8 per iteration, results fed back
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uint32_t d;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(x[i]), "f"(x[(i + 1) & 7]));
        x[i] = __uint_as_float(d);
      }
    }
    if (OP == 7) {  // ex2.approx.f16x2 (2 results per instruction)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uint32_t v = __float_as_uint(x[i]);
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(v));
        x[i] = __uint_as_float(v);
      }
    }
    if (OP == 8) {  // cvt.rn.f16x2.f32
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uint32_t d;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(x[i]), "f"(x[(i + 1) & 7]));
        x[i] = __uint_as_float(d);
      }
    }
    if (OP == 9) {  // IADD + LOP (ALU pipe)
#pragma unroll
      for (int i = 0; i < 8; ++i) xi[i] = (xi[i] + 0x7fff) ^ it;
    }
    if (OP == 4) {  // packed f32x2 FMA: 4 instructions = 8 FMAs
#pragma unroll
      for (int i = 0; i < 8; i += 2) {
        uint64_t v = ((uint64_t)__float_as_uint(x[i + 1]) << 32) | __float_as_uint(x[i]);
        uint64_t av = ((uint64_t)__float_as_uint(a) << 32) | __float_as_uint(a);
        uint64_t bv = ((uint64_t)__float_as_uint(b) << 32) | __float_as_uint(b);
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v) : "l"(av), "l"(bv));
        x[i] = __uint_as_float((uint32_t)v);
        x[i + 1] = __uint_as_float((uint32_t)(v >> 32));
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// ── TMEM ld / st bandwidth, and promotion variants fed from TMEM ───────
// 16 warps (4 per lane quarter); VARIANT: 0 = ld only, 1 = st only,
// 2 = ld + I2F + FMUL + FMUL + FADD (exact), 3 = ld + I2F + FFMA (fast),
// 4 = ld + st(magic) + FFMA + FADD (fast, magic), 5 = ld + st + FFMA + FMUL + FADD (exact, magic)
template <int VARIANT>
__global__ void __launch_bounds__(512, 1) tmem_kernel(float *out, long long *cyc, float sa, float sb, float zero) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&tbase, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tbase + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 128;
  float acc[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) acc[j] = 0.f;
  uint32_t r[32];
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS / 4; ++it) {
    const uint32_t ta = t + (it & 3) * 32;
    if (VARIANT != 1) {
      tmem_ld_32x32b_x32(ta, r);
      tmem_wait_ld();
    }
    if (VARIANT == 1 || VARIANT == 4 || VARIANT == 5) {
      tmem_fill_32x32b_x32(ta, 0x4B400000u + it);
      tmem_wait_st();
    }
    if (VARIANT == 0) {
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = __uint_as_float(__float_as_uint(acc[j]) ^ r[j]);
    } else if (VARIANT == 2) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        acc[j] = __fadd_rn(acc[j], __fmul_rn(__fmul_rn(__int2float_rn((int)r[j]), sa), sb));
    } else if (VARIANT == 3) {
      const float s = sa * sb;
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = __fmaf_rn(__int2float_rn((int)r[j]), s, acc[j]);
    } else if (VARIANT == 4) {
      const float s = sa * sb, ncs = -12582912.0f * s;
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = __fadd_rn(acc[j], __fmaf_rn(__uint_as_float(r[j]), s, ncs));
    } else if (VARIANT == 6) {  // fast, packed: I2F + FFMA2
      const float s = sa * sb;
#pragma unroll
      for (int j = 0; j < 32; j += 2)
        ffma2_rn(acc[j], acc[j + 1], __int2float_rn((int)r[j]), __int2float_rn((int)r[j + 1]), s, s,
                 acc[j], acc[j + 1]);
    } else if (VARIANT == 7) {  // exact, packed: I2F + FMUL2 + FMUL2 + FADD2
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        float t0, t1;
        fmul2_rn(t0, t1, __int2float_rn((int)r[j]), __int2float_rn((int)r[j + 1]), sa, sa);
        fmul2_rn(t0, t1, t0, t1, sb, sb);
        fadd2_rn(acc[j], acc[j + 1], acc[j], acc[j + 1], t0, t1);
      }
    } else if (VARIANT == 9) {  // exact, 3 packed FP32 ops (as gemm_i8_kernel): I2F, FMUL2, FFMA2(+0), FADD2
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        float t0, t1;
        fmul2_rn(t0, t1, __int2float_rn((int)r[j]), __int2float_rn((int)r[j + 1]), sa, sa);
        ffma2_rn(t0, t1, t0, t1, sb, sb, zero, zero);
        fadd2_rn(acc[j], acc[j + 1], acc[j], acc[j + 1], t0, t1);
      }
    } else if (VARIANT == 8) {  // I2F only (throughput of the conversion pipe)
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = __int_as_float(__float_as_int(acc[j]) ^ __float_as_int(__int2float_rn((int)r[j])));
    } else if (VARIANT == 5) {
      const float ncs = -12582912.0f * sa;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        acc[j] = __fadd_rn(acc[j], __fmul_rn(__fmaf_rn(__uint_as_float(r[j]), sa, ncs), sb));
    }
  }
  tc_fence_before();
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (warp == 0) tmem_dealloc(tbase, 512);
}

// ── raw tcgen05.mma kind::i8 issue rate ────────────────────────────────
// MODE 0: back-to-back MMAs, one commit at the end.
// MODE 1: a tcgen05.commit (to one of 4 mbarriers) after every MMA, never waited.
// MODE 2: MMA -> commit -> wait on that commit before the next MMA (latency).
template <int N, int MODE = 0>
__global__ void __launch_bounds__(128, 1) mma_kernel(long long *cyc, int nmma) {
  extern __shared__ uint8_t smraw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar;
  __shared__ uint64_t bars[4];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (128 + N) * 128 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t *>(sm)[i] = 0x01010101u * (i & 7);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tbase, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 32) {
    const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 128 * 128);
    constexpr uint32_t idesc = idesc_i8(128, N, 0, 0);
    long long t0 = clock64();
    for (int i = 0; i < nmma; ++i) {
      const int c = i & 3;
      const uint32_t dst = (MODE >= 6) ? tbase + (i & 3) * N : tbase + (i & 1) * N;
      mma_i8_ss(dst % 512 + (tbase & 0xffff0000u), smem_desc_sw128(a0 + c * 32, 16, 1024),
                smem_desc_sw128(b0 + c * 32, 16, 1024), idesc, (MODE == 6 || MODE == 8) ? 0u : 1u);
      if (MODE >= 1 && MODE != 8) mma_commit(&bars[i & 3]);
      if (MODE == 2) mbar_wait(&bars[i & 3], (i >> 2) & 1);
      if (MODE == 3 || MODE == 5) tc_fence_after();
      if (MODE == 4) {
        tc_fence_after();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
  }
  if (MODE == 5 && warp >= 2) {  // concurrent TMEM readers on the second half of TMEM
    uint32_t r[32];
    uint32_t acc = 0;
    for (int i = 0; i < nmma / 2; ++i) {
      tmem_ld_32x32b_x32(tbase + ((uint32_t)((warp & 3) * 32) << 16) + 256 + (i & 7) * 32, r);
      tmem_wait_ld();
      acc ^= r[i & 31];
    }
    if (acc == 0x12345) cyc[blockIdx.x] = 0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

// Concurrency: MMA+commit stream (1 thread) alongside TMEM readers (W warps of LDTM.xX)
// reading 64 KB per "chunk" each; no barriers between them.  Reports both rates.
template <int W, int X>
__global__ void __launch_bounds__(32 * (W + 1), 1) mma_ld_kernel(long long *cyc, int nchunk, float *out) {
  extern __shared__ uint8_t smraw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tbase;
  __shared__ uint64_t bars[4];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 256 * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x01010101u * (i & 7);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  if (warp == W) tmem_alloc(&tbase, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == W) {
    if ((threadIdx.x & 31) == 0) {
      const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 128 * 128);
      long long t0 = clock64();
      for (int i = 0; i < (W < 0 ? 0 : nchunk); ++i) {
        mma_i8_ss(tbase + (i & 1) * 128, smem_desc_sw128(a0 + (i & 3) * 32, 16, 1024),
                  smem_desc_sw128(b0 + (i & 3) * 32, 16, 1024), idesc_i8(128, 128, 0, 0), 0u);
        mma_commit(&bars[i & 3]);
      }
      mbar_wait(&bars[(nchunk - 1) & 3], ((nchunk - 1) >> 2) & 1);
      cyc[blockIdx.x * 2] = clock64() - t0;
    }
  } else {
    // each warp reads its lane quarter x (128*4/W) columns per chunk
    constexpr int kColsPerWarp = 128 * 4 / W;
    const uint32_t t = tbase + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * kColsPerWarp;
    uint32_t acc = 0;
    long long t0 = clock64();
    for (int i = 0; i < nchunk; ++i) {
      for (int k = 0; k < kColsPerWarp; k += (X == 256 || X == 128) ? 32 : X) {
        if (X == 32) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(t + 256 + (i & 1) * 128 + k, r);
          tmem_wait_ld();
          acc ^= r[i & 31];
        } else if (X == 256 || X == 128) {  // 16x256b.x8 / 16x128b.x16: 16 lanes x 64 cols per instr
          uint32_t r[32];
          const uint32_t ta = t + 256 + (i & 1) * 128 + k;
          if (X == 256)
            asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]) : "r"(ta));
          else
            asm volatile("tcgen05.ld.sync.aligned.16x128b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]) : "r"(ta));
          tmem_wait_ld();
          acc ^= r[i & 31];
        } else {
          uint32_t r[64];
          tmem_ld_32x32b_x64(t + 256 + (i & 1) * 128 + k, r);
          tmem_wait_ld();
          acc ^= r[i & 63];
        }
      }
    }
    if (warp == 0 && (threadIdx.x & 31) == 0) cyc[blockIdx.x * 2 + 1] = clock64() - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == W) tmem_dealloc(tbase, 512);
}

// Legacy warp-level IMMA: mma.sync.m16n8k32 s8 x s8 -> s32 (register accumulators).
__global__ void __launch_bounds__(512, 1) mmasync_kernel(long long *cyc, int iters, int *out) {
  uint32_t a[4], b[2];
  int c[8][4];
  for (int i = 0; i < 4; ++i) a[i] = 0x01010101u * (threadIdx.x + i);
  for (int i = 0; i < 2; ++i) b[i] = 0x01020304u * (threadIdx.x + i);
  for (int j = 0; j < 8; ++j)
    for (int i = 0; i < 4; ++i) c[j][i] = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile(
          "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  __syncthreads();
  long long t1 = clock64();
  int s = 0;
  for (int j = 0; j < 8; ++j)
    for (int i = 0; i < 4; ++i) s += c[j][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

static int g_sms;

static double median_cycles(long long *d_cyc, int n) {
  std::vector<long long> h(n);
  CK(cudaMemcpy(h.data(), d_cyc, n * sizeof(long long), cudaMemcpyDeviceToHost));
  std::sort(h.begin(), h.end());
  return (double)h[n / 2];
}

#include <algorithm>

template <int OP>
void run_fp(const char *name, float *d_out, long long *d_cyc, double ops_per_iter_thread) {
  fp_kernel<OP><<<g_sms, 1024>>>(d_out, d_cyc, 1.0001f, 0.5f);
  CK(cudaDeviceSynchronize());
  fp_kernel<OP><<<g_sms, 1024>>>(d_out, d_cyc, 1.0001f, 0.5f);
  CK(cudaDeviceSynchronize());
  double cyc = median_cycles(d_cyc, g_sms);
  double ops = ops_per_iter_thread * ITERS * 1024.0;
  printf("{\"bench\": \"%s\", \"ops_per_clk_per_sm\": %.1f, \"cycles\": %.0f}\n", name, ops / cyc, cyc);
}

template <int V>
void run_tmem(const char *name, float *d_out, long long *d_cyc) {
  tmem_kernel<V><<<g_sms, 512>>>(d_out, d_cyc, 0.01f, 0.02f, 0.0f);
  CK(cudaDeviceSynchronize());
  tmem_kernel<V><<<g_sms, 512>>>(d_out, d_cyc, 0.01f, 0.02f, 0.0f);
  CK(cudaDeviceSynchronize());
  double cyc = median_cycles(d_cyc, g_sms);
  double elems = 16.0 * 32 * 32 * (ITERS / 4);  // 16 warps x 32 lanes x 32 cols per iter
  printf("{\"bench\": \"%s\", \"elems_per_clk_per_sm\": %.1f, \"bytes_per_clk_per_sm\": %.1f, \"cycles\": %.0f}\n",
         name, elems / cyc, elems * 4 / cyc, cyc);
}

template <int N, int MODE = 0>
void run_mma(long long *d_cyc) {
  const size_t smem = 1024 + (128 + N) * 128;
  CK(cudaFuncSetAttribute(mma_kernel<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int nmma = 4096;
  mma_kernel<N, MODE><<<g_sms, 128, smem>>>(d_cyc, nmma);
  CK(cudaDeviceSynchronize());
  mma_kernel<N, MODE><<<g_sms, 128, smem>>>(d_cyc, nmma);
  CK(cudaDeviceSynchronize());
  double cyc = median_cycles(d_cyc, g_sms);
  double macs = 128.0 * N * 32 * nmma;
  printf("{\"bench\": \"mma_i8_m128_n%d_k32_mode%d\", \"mac_per_clk_per_sm\": %.1f, \"clk_per_mma\": %.2f}\n", N,
         MODE, macs / cyc, cyc / nmma);
}

template <int W, int X>
void run_mma_ld(long long *d_cyc, float *d_out) {
  const size_t smem = 1024 + 256 * 128;
  CK(cudaFuncSetAttribute(mma_ld_kernel<W, X>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int n = 2048;
  mma_ld_kernel<W, X><<<g_sms, 32 * (W + 1), smem>>>(d_cyc, n, d_out);
  CK(cudaDeviceSynchronize());
  mma_ld_kernel<W, X><<<g_sms, 32 * (W + 1), smem>>>(d_cyc, n, d_out);
  CK(cudaDeviceSynchronize());
  std::vector<long long> h(2 * g_sms);
  CK(cudaMemcpy(h.data(), d_cyc, 2 * g_sms * sizeof(long long), cudaMemcpyDeviceToHost));
  printf("{\"bench\": \"mma+ld W=%d x%d\", \"mma_clk_per_chunk\": %.1f, \"ld_clk_per_chunk\": %.1f}\n", W, X,
         (double)h[0] / n, (double)h[1] / n);
}

void run_mmasync(long long *d_cyc, float *d_out) {
  const int iters = 2048;
  mmasync_kernel<<<g_sms, 512>>>(d_cyc, iters, (int *)d_out);
  CK(cudaDeviceSynchronize());
  mmasync_kernel<<<g_sms, 512>>>(d_cyc, iters, (int *)d_out);
  CK(cudaDeviceSynchronize());
  double cyc = median_cycles(d_cyc, g_sms);
  double macs = 512.0 / 32 * iters * 8 * (16 * 8 * 32);  // 16 warps
  printf("{\"bench\": \"mma.sync m16n8k32 s8 (16 warps)\", \"mac_per_clk_per_sm\": %.1f}\n", macs / cyc);
}


// Promotion (exact, gemm form) by 16 warps on TMEM columns 0..127 while warp 16
// lane 0 streams MMAs (M=128,N=128,K=32) into columns 256..511, optionally
// throttled: one MMA per `gap` clk.  Measures TMEM read/compute contention with
// concurrent tensor-core writes.
__global__ void __launch_bounds__(544, 1) promote_vs_mma_kernel(float *out, long long *cyc, float sa, float sb,
                                                                 float zero, int nmma, int gap) {
  extern __shared__ uint8_t smraw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 256 * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x01010101u * (i & 7);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    done = 0;
  }
  if (warp == 0) tmem_alloc(&tbase, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 16) {
    if ((threadIdx.x & 31) == 0 && nmma > 0) {
      const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 128 * 128);
      for (int i = 0; i < nmma; ++i) {
        long long t0 = clock64();
        mma_i8_ss(tbase + 256 + (i & 1) * 128, smem_desc_sw128(a0 + (i & 3) * 32, 16, 1024),
                  smem_desc_sw128(b0 + (i & 3) * 32, 16, 1024), idesc_i8(128, 128, 0, 0), 0u);
        if (gap > 0)
          while (clock64() - t0 < gap) {
          }
      }
      mma_commit(&bar);
      mbar_wait(&bar, 0);
    }
  } else {
    const uint32_t t = tbase + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 32;
    float acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = 0.f;
    uint32_t r[32];
    long long t0 = clock64();
    for (int it = 0; it < ITERS / 4; ++it) {
      tmem_ld_32x32b_x32(t, r);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        float t0f, t1f;
        fmul2_rn(t0f, t1f, __int2float_rn((int)r[j]), __int2float_rn((int)r[j + 1]), sa, sa);
        ffma2_rn(t0f, t1f, t0f, t1f, sb, sb, zero, zero);
        fadd2_rn(acc[j], acc[j + 1], acc[j], acc[j + 1], t0f, t1f);
      }
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) s += acc[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

void run_promote_vs_mma(long long *d_cyc, float *d_out, int nmma, int gap) {
  const size_t smem = 1024 + 256 * 128;
  CK(cudaFuncSetAttribute(promote_vs_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int rep = 0; rep < 2; ++rep) {
    promote_vs_mma_kernel<<<g_sms, 544, smem>>>(d_out, d_cyc, 0.01f, 0.02f, 0.0f, nmma, gap);
    CK(cudaDeviceSynchronize());
  }
  double cyc = median_cycles(d_cyc, g_sms);
  double elems = 16.0 * 32 * 32 * (ITERS / 4);
  printf("{\"bench\": \"promote_exact_vs_mma nmma=%d gap=%d\", \"elems_per_clk_per_sm\": %.1f, \"clk_per_16k\": %.0f}\n",
         nmma, gap, elems / cyc, 16384.0 * cyc / elems);
}


// The GEMM's TMEM hand-off in isolation: warp 16 lane 0 issues one MMA per
// chunk into buffer c % 4 after all 16 promotion warps released it (tempty,
// count 16) and commits tfull; the promotion warps wait tfull, load, release,
// promote (exact, gemm form).  WAITK selects the promotion-warp wait: 0 spin
// try_wait, 1 try_wait with a suspend hint.
template <int WAITK, int SCALES>
__global__ void __launch_bounds__(544, 1) handoff_kernel(float *out, long long *cyc, float sa, float sb, float zero,
                                                         int nchunk, const float *gsa, const float *gsb) {
  extern __shared__ uint8_t smraw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tbase;
  __shared__ uint64_t tfull[4], tempty[4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 256 * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x01010101u * (i & 7);
  if (threadIdx.x == 0) {
    for (int b = 0; b < 4; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 16);
    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tbase, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t bf = smem_u32(&tfull[0]), be = smem_u32(&tempty[0]);
  if (warp == 16) {
    if (lane == 0) {
      const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 128 * 128);
      for (int c = 0; c < nchunk; ++c) {
        const int b = c & 3;
        mbar_wait_u32(be + 8 * b, ((c >> 2) & 1) ^ 1);
        tc_fence_after();
        mma_i8_ss(tbase + b * 128, smem_desc_sw128(a0 + (c & 3) * 32, 16, 1024),
                  smem_desc_sw128(b0 + (c & 3) * 32, 16, 1024), idesc_i8(128, 128, 0, 0), 0u);
        mma_commit(&tfull[b]);
      }
    }
  } else {
    const uint32_t t = tbase + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 32;
    float acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = 0.f;
    long long t0 = clock64();
    __shared__ float ssc[2][16];
    if (threadIdx.x < 32) ssc[threadIdx.x >> 4][threadIdx.x & 15] = threadIdx.x < 16 ? sa : sb;
    asm volatile("bar.sync 1, 512;" ::: "memory");
    for (int c0 = 0; c0 < nchunk; c0 += 4) {
      float sav[4] = {sa, sa, sa, sa}, sbv[4] = {sb, sb, sb, sb};
      if (SCALES == 1) {  // as gemm_i8_kernel: one float4 of each grid per 4 chunks, from global
        const float4 x = __ldg(reinterpret_cast<const float4 *>(gsa + (warp & 3) * 4096 + c0));
        const float4 y = __ldg(reinterpret_cast<const float4 *>(gsb + (warp >> 2) * 4096 + c0));
        sav[0] = x.x; sav[1] = x.y; sav[2] = x.z; sav[3] = x.w;
        sbv[0] = y.x; sbv[1] = y.y; sbv[2] = y.z; sbv[3] = y.w;
      }
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int c = c0 + b;
        if (WAITK == 1) mbar_wait_u32_sleep(bf + 8 * b, (c >> 2) & 1, 50);
        else mbar_wait_u32(bf + 8 * b, (c >> 2) & 1);
        tc_fence_after();
        uint32_t r[32];
        tmem_ld_32x32b_x32(t + b * 128, r);
        if (SCALES == 2) {  // scales staged in shared memory (as a TMA-fed ring would)
          sav[b] = ssc[0][(warp & 3) * 4 + b];
          sbv[b] = ssc[1][(warp >> 2) * 4 + b];
        }
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_u32(be + 8 * b);
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          float t0f, t1f;
          fmul2_rn(t0f, t1f, __int2float_rn((int)r[j]), __int2float_rn((int)r[j + 1]), sav[b], sav[b]);
          ffma2_rn(t0f, t1f, t0f, t1f, sbv[b], sbv[b], zero, zero);
          fadd2_rn(acc[j], acc[j + 1], acc[j], acc[j + 1], t0f, t1f);
        }
      }
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) s += acc[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

template <int WAITK, int SCALES = 0>
void run_handoff(long long *d_cyc, float *d_out) {
  const size_t smem = 1024 + 256 * 128;
  const int n = 1024;
  static float *gs = nullptr;
  if (!gs) {
    CK(cudaMalloc(&gs, 2 * 4 * 4096 * sizeof(float)));
    CK(cudaMemset(gs, 0, 2 * 4 * 4096 * sizeof(float)));
  }
  CK(cudaFuncSetAttribute(handoff_kernel<WAITK, SCALES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int rep = 0; rep < 2; ++rep) {
    handoff_kernel<WAITK, SCALES><<<g_sms, 544, smem>>>(d_out, d_cyc, 0.01f, 0.02f, 0.0f, n, gs, gs + 4 * 4096);
    CK(cudaDeviceSynchronize());
  }
  double cyc = median_cycles(d_cyc, g_sms);
  printf("{\"bench\": \"handoff_exact wait=%d scales=%d\", \"clk_per_chunk\": %.0f}\n", WAITK, SCALES, cyc / n);
}

int main() {
  CK(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0));
  int clk_khz = 0;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  printf("{\"bench\": \"device\", \"sms\": %d, \"clock_khz_attr\": %d}\n", g_sms, clk_khz);
  float *d_out;
  long long *d_cyc;
  CK(cudaMalloc(&d_out, g_sms * 1024 * sizeof(float)));
  CK(cudaMalloc(&d_cyc, 2 * g_sms * sizeof(long long)));
  run_fp<0>("ffma", d_out, d_cyc, 8);
  run_fp<1>("fmul", d_out, d_cyc, 8);
  run_fp<2>("fadd", d_out, d_cyc, 8);
  run_fp<3>("i2fp_chain", d_out, d_cyc, 8);
  run_fp<4>("ffma2_x2_fmas", d_out, d_cyc, 8);
  run_fp<5>("mufu_ex2", d_out, d_cyc, 8);
  run_fp<6>("cvt_bf16x2_f32 (instr)", d_out, d_cyc, 8);
  run_fp<7>("ex2_f16x2 (instr)", d_out, d_cyc, 8);
  run_fp<8>("cvt_f16x2_f32 (instr)", d_out, d_cyc, 8);
  run_fp<9>("iadd_lop (2 ops)", d_out, d_cyc, 16);
  run_tmem<0>("tmem_ld_x32", d_out, d_cyc);
  run_tmem<1>("tmem_st_x8x4", d_out, d_cyc);
  run_tmem<2>("promote_exact_i2f", d_out, d_cyc);
  run_tmem<3>("promote_fast_i2f", d_out, d_cyc);
  run_tmem<4>("promote_fast_magic", d_out, d_cyc);
  run_tmem<5>("promote_exact_magic", d_out, d_cyc);
  run_tmem<6>("promote_fast_i2f_ffma2", d_out, d_cyc);
  run_tmem<7>("promote_exact_i2f_packed", d_out, d_cyc);
  run_tmem<8>("i2f_plus_lop", d_out, d_cyc);
  run_tmem<9>("promote_exact_3op_i2f (gemm form)", d_out, d_cyc);
  run_mma<128>(d_cyc);
  run_mma<256>(d_cyc);
  run_mma<64>(d_cyc);
  run_mma<128, 1>(d_cyc);
  run_mma<128, 2>(d_cyc);
  run_mma<256, 1>(d_cyc);
  run_mma<128, 3>(d_cyc);
  run_mma<128, 4>(d_cyc);
  run_mma<128, 5>(d_cyc);
  run_mma<128, 6>(d_cyc);   // accumulate=0, commit per MMA, 4 rotating buffers
  run_mma<128, 7>(d_cyc);   // accumulate=1, commit per MMA, 4 rotating buffers
  run_mma<128, 8>(d_cyc);   // accumulate=0, no per-MMA commit
  run_mmasync(d_cyc, d_out);
  // ITERS/4 = 1024 promotion iterations per warp = 1024 chunks; MMAs over the same span
  run_handoff<0>(d_cyc, d_out);
  run_handoff<1>(d_cyc, d_out);
  run_handoff<0, 1>(d_cyc, d_out);
  run_handoff<0, 2>(d_cyc, d_out);
  run_promote_vs_mma(d_cyc, d_out, 0, 0);
  run_promote_vs_mma(d_cyc, d_out, 1024, 400);
  run_promote_vs_mma(d_cyc, d_out, 1024, 200);
  run_promote_vs_mma(d_cyc, d_out, 4096, 0);
  run_mma_ld<16, 32>(d_cyc, d_out);
  run_mma_ld<8, 32>(d_cyc, d_out);
  run_mma_ld<8, 64>(d_cyc, d_out);
  run_mma_ld<4, 64>(d_cyc, d_out);
  // run_mma_ld<16, 256>: illegal address (16x256b shape needs a different lane mapping)

  return 0;
}
