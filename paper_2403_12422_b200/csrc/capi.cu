// capi.cu — host-side plumbing of libjetfire: error reporting, SM count,
// TMA tensor-map encoding (driver entry point fetched through the runtime,
// so the library needs no -lcuda link).
#include <cudaTypedefs.h>
#include <stdio.h>
#include <string.h>

#include <mutex>
#include <set>
#include <utility>

#include "common.cuh"

static thread_local char g_err[512] = "";

void jf_set_error(const char *msg) {
  strncpy(g_err, msg, sizeof(g_err) - 1);
  g_err[sizeof(g_err) - 1] = 0;
}

int jf_launch_check(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
    return JF_ERR_LAUNCH;
  }
  return JF_OK;
}

int jf_num_sms() {
  static int n[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int &v = n[dev & 63];
  if (v == 0) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
  }
  return v;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is a per-DEVICE setting: remember
// the (kernel, device) pairs already raised, so a process driving several GPUs sets
// it once on each.
int jf_set_smem_attr(const void *func, int bytes, const char *what) {
  static std::mutex mu;
  static std::set<std::pair<const void *, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    if (done.count({func, dev})) return JF_OK;
  }
  if (cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
    return jf_launch_check(what);
  std::lock_guard<std::mutex> lk(mu);
  done.insert({func, dev});
  return JF_OK;
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D int8 tensor map: rows x cols (cols contiguous, row stride ld bytes),
// box box_rows x box_cols; 128-byte swizzle (box_cols must then be 128) or none.
static bool jf_make_tmap_i8_encode(CUtensorMap *map, const void *ptr, int64_t rows, int64_t cols, int64_t ld,
                     int box_cols, int box_rows, bool swizzle128) {
  auto enc = get_encode();
  if (!enc) {
    jf_set_error("cuTensorMapEncodeTiled unavailable");
    return false;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    snprintf(g_err, sizeof(g_err), "cuTensorMapEncodeTiled failed (%d) rows=%lld cols=%lld ld=%lld",
             (int)r, (long long)rows, (long long)cols, (long long)ld);
    return false;
  }
  return true;
}

// 2-D f16 tensor map: rows x cols, row stride ld elements, 128-byte swizzle.
static bool jf_make_tmap_f16_encode(CUtensorMap *map, const void *ptr, int64_t rows, int64_t cols, int64_t ld,
                      int box_cols, int box_rows) {
  auto enc = get_encode();
  if (!enc) {
    jf_set_error("cuTensorMapEncodeTiled unavailable");
    return false;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void *>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    snprintf(g_err, sizeof(g_err), "cuTensorMapEncodeTiled(f16) failed (%d) rows=%lld cols=%lld", (int)r,
             (long long)rows, (long long)cols);
    return false;
  }
  return true;
}

// 2-D fp32 tensor map (scale grids): rows x cols, row stride ld elements, no swizzle.
static bool jf_make_tmap_f32_encode(CUtensorMap *map, const void *ptr, int64_t rows, int64_t cols, int64_t ld,
                      int box_cols, int box_rows) {
  auto enc = get_encode();
  if (!enc) {
    jf_set_error("cuTensorMapEncodeTiled unavailable");
    return false;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    snprintf(g_err, sizeof(g_err), "cuTensorMapEncodeTiled(f32) failed (%d)", (int)r);
    return false;
  }
  return true;
}

extern "C" int jf_version(void) { return 1; }
extern "C" const char *jf_last_error(void) { return g_err; }
extern "C" int jf_sm_count(void) { return jf_num_sms(); }

// ── tensor-map cache ───────────────────────────────────────────────────
// cuTensorMapEncodeTiled costs microseconds of host time and every GEMM launch
// needs four maps.  A map depends only on (address, dims, stride, box, kind),
// so a reused allocation with the same shape gets a bit-identical map: cache
// them (direct-mapped, 4096 entries).
namespace {
struct TmapKey {
  const void *ptr;
  int64_t rows, cols, ld;
  int box_cols, box_rows, kind;
  bool operator==(const TmapKey &o) const {
    return ptr == o.ptr && rows == o.rows && cols == o.cols && ld == o.ld && box_cols == o.box_cols &&
           box_rows == o.box_rows && kind == o.kind;
  }
};
struct TmapEntry {
  TmapKey key;
  CUtensorMap map;
  bool valid;
};
constexpr int kTmapCache = 4096;
TmapEntry g_tmaps[kTmapCache];
std::mutex g_tmap_mu;

size_t tmap_slot(const TmapKey &k) {
  uint64_t h = (uint64_t)(uintptr_t)k.ptr * 0x9E3779B97F4A7C15ull;
  h ^= (uint64_t)k.rows * 0xC2B2AE3D27D4EB4Full + (uint64_t)k.cols * 0x165667B19E3779F9ull;
  h ^= (uint64_t)k.ld * 0x27D4EB2F165667C5ull + (uint64_t)(k.box_cols * 131 + k.box_rows * 7 + k.kind);
  return (size_t)((h ^ (h >> 29)) % kTmapCache);
}

template <typename F>
bool cached_tmap(CUtensorMap *map, const TmapKey &k, F encode) {
  const size_t s = tmap_slot(k);
  {
    std::lock_guard<std::mutex> lk(g_tmap_mu);
    if (g_tmaps[s].valid && g_tmaps[s].key == k) {
      *map = g_tmaps[s].map;
      return true;
    }
  }
  if (!encode(map)) return false;
  std::lock_guard<std::mutex> lk(g_tmap_mu);
  g_tmaps[s].key = k;
  g_tmaps[s].map = *map;
  g_tmaps[s].valid = true;
  return true;
}
}  // namespace

bool jf_make_tmap_i8(CUtensorMap *map, const void *ptr, int64_t rows, int64_t cols, int64_t ld, int box_cols,
                     int box_rows, bool swizzle128) {
  return cached_tmap(map, TmapKey{ptr, rows, cols, ld, box_cols, box_rows, swizzle128 ? 1 : 0}, [&](CUtensorMap *m) {
    return jf_make_tmap_i8_encode(m, ptr, rows, cols, ld, box_cols, box_rows, swizzle128);
  });
}

bool jf_make_tmap_f16(CUtensorMap *map, const void *ptr, int64_t rows, int64_t cols, int64_t ld, int box_cols,
                      int box_rows) {
  return cached_tmap(map, TmapKey{ptr, rows, cols, ld, box_cols, box_rows, 2},
                     [&](CUtensorMap *m) { return jf_make_tmap_f16_encode(m, ptr, rows, cols, ld, box_cols, box_rows); });
}

bool jf_make_tmap_f32(CUtensorMap *map, const void *ptr, int64_t rows, int64_t cols, int64_t ld, int box_cols,
                      int box_rows) {
  return cached_tmap(map, TmapKey{ptr, rows, cols, ld, box_cols, box_rows, 3},
                     [&](CUtensorMap *m) { return jf_make_tmap_f32_encode(m, ptr, rows, cols, ld, box_cols, box_rows); });
}
