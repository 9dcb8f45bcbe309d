#include "rb_common.h"
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <set>
#include <unordered_map>

namespace rb {

static thread_local char g_err[512] = {0};

int set_error(const char* msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return RB_ERR_ARG;
}

int set_cuda_error(const char* where, cudaError_t e) {
  snprintf(g_err, sizeof(g_err), "%s: %s (%d)", where, cudaGetErrorString(e), (int)e);
  return RB_ERR_CUDA;
}

int set_cu_error(const char* where, CUresult r) {
  snprintf(g_err, sizeof(g_err), "%s: CUresult %d", where, (int)r);
  return RB_ERR_DRIVER;
}

const char* last_error() { return g_err; }

void* driver_symbol(const char* name) {
  static std::mutex mu;
  static std::unordered_map<std::string, void*> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(name);
  if (it != cache.end()) return it->second;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess) fn = nullptr;
  cache[name] = fn;
  return fn;
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct TmapKey {
  uint64_t base, inner, outer, ld;
  uint32_t bi, bo;
  bool operator==(const TmapKey& o) const {
    return base == o.base && inner == o.inner && outer == o.outer && ld == o.ld && bi == o.bi && bo == o.bo;
  }
};
struct TmapKeyHash {
  size_t operator()(const TmapKey& k) const {
    uint64_t h = k.base * 0x9E3779B97F4A7C15ull;
    h ^= (k.inner + 0x632BE59BD9B4E019ull + (h << 6) + (h >> 2));
    h ^= (k.outer + 0x8CB92BA72F3D8DD7ull + (h << 6) + (h >> 2));
    h ^= (k.ld + ((uint64_t)k.bi << 32 | k.bo) + (h << 6) + (h >> 2));
    return (size_t)h;
  }
};

// Encoding a tensor map costs microseconds of host time; weights and the
// executor's activation buffers never move, so maps are cached by their full
// key (address, extents, stride, box). A map depends on nothing else, so a
// cached entry is valid for any buffer that matches the key.
int make_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
                      uint32_t box_inner, uint32_t box_outer) {
  static std::mutex mu;
  static std::unordered_map<TmapKey, CUtensorMap, TmapKeyHash> cache;
  TmapKey key{reinterpret_cast<uint64_t>(base), inner, outer, ld, box_inner, box_outer};
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *map = it->second;
      return 0;
    }
  }
  static PFN_encodeTiled enc = nullptr;
  if (!enc) {
    enc = reinterpret_cast<PFN_encodeTiled>(driver_symbol("cuTensorMapEncodeTiled"));
    if (!enc) return set_error("cuTensorMapEncodeTiled unavailable");
  }
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_cu_error("cuTensorMapEncodeTiled", r);
  std::lock_guard<std::mutex> lk(mu);
  if (cache.size() > 65536) cache.clear();
  cache.emplace(key, *map);
  return 0;
}

static bool g_pdl = true;
bool pdl_enabled() { return g_pdl; }
void set_pdl(bool on) { g_pdl = on; }

}  // namespace rb

namespace rb {
// Paged KV cache layer [nb][2 (K,V)][Hkv][16][128] bf16 as a 5D tensor for one-op-per-page
// loads: d0 = 64 dims (128 B, swizzled), d1 = 16 tokens (256 B), d2 = 2 dim halves (128 B),
// d3 = K/V (Hkv x 4 KB), d4 = 4 KB page-head rows ((page * 2 + kv) * Hkv + head). A box
// {64, 16, 2, 2, 1} lands as [K lo | K hi | V lo | V hi] x 16 rows x 128 B, the same smem
// image as four {64, 16} boxes of the 2D view.
int make_tmap_kv5d_bf16(CUtensorMap* map, const void* cache_layer, uint64_t num_blocks, int hkv) {
  static std::mutex mu;
  static std::unordered_map<TmapKey, CUtensorMap, TmapKeyHash> cache;
  TmapKey key{reinterpret_cast<uint64_t>(cache_layer), num_blocks, (uint64_t)hkv, 5, 64, 16};
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *map = it->second;
      return 0;
    }
  }
  static PFN_encodeTiled enc = nullptr;
  if (!enc) {
    enc = reinterpret_cast<PFN_encodeTiled>(driver_symbol("cuTensorMapEncodeTiled"));
    if (!enc) return set_error("cuTensorMapEncodeTiled unavailable");
  }
  cuuint64_t dims[5] = {64, 16, 2, 2, (cuuint64_t)num_blocks * 2 * hkv};
  cuuint64_t strides[4] = {256, 128, (cuuint64_t)hkv * 4096, 4096};
  cuuint32_t box[5] = {64, 16, 2, 2, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(cache_layer), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_cu_error("cuTensorMapEncodeTiled(kv5d)", r);
  std::lock_guard<std::mutex> lk(mu);
  cache.emplace(key, *map);
  return 0;
}
}  // namespace rb

namespace rb {
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel): the attribute is
// per device, so a process that launches on several GPUs sets it on each.
cudaError_t set_smem_attr_once(const void* fn, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({dev, fn})) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.insert({dev, fn});
  return e;
}
}  // namespace rb
