// fq_tma.cu — host-side creation of TMA tensor maps (driver entry point fetched at run time, so
// libfq.so does not link libcuda and still loads on GPU-less machines).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstring>
#include <mutex>

#include "fq_internal.h"

namespace fq {

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// Descriptor cache: encoding a tensor map costs host time on every GEMM call, while the
// descriptors of a call sequence are almost always the same (weights, scales and the workspace
// regions are long-lived; activations are often reused buffers).  A small direct-mapped cache keyed
// by every encoding argument returns the previously encoded 128-byte descriptor.
namespace {
struct TmapKey {
  const void* base;
  uint64_t inner, outer, stride;
  uint32_t box_inner, box_outer;
  int elem_bytes, swizzle;
  bool operator==(const TmapKey& o) const {
    return base == o.base && inner == o.inner && outer == o.outer && stride == o.stride &&
           box_inner == o.box_inner && box_outer == o.box_outer && elem_bytes == o.elem_bytes &&
           swizzle == o.swizzle;
  }
};
struct TmapEntry {
  TmapKey key;
  alignas(64) CUtensorMap map;
  bool valid;
};
constexpr int kTmapCache = 256;
TmapEntry g_tmap_cache[kTmapCache];
std::mutex g_tmap_mu;
size_t tmap_hash(const TmapKey& k) {
  uint64_t h = reinterpret_cast<uintptr_t>(k.base) * 0x9E3779B97F4A7C15ull;
  h ^= (k.inner * 31 + k.outer) * 0xC2B2AE3D27D4EB4Full;
  h ^= (k.stride + ((uint64_t)k.box_inner << 32) + k.box_outer) * 0x165667B19E3779F9ull;
  h ^= (uint64_t)(k.elem_bytes * 131 + k.swizzle);
  return (size_t)(h ^ (h >> 29)) % kTmapCache;
}
}  // namespace

static bool encode_tmap_2d(void* tmap, const void* base, int elem_bytes, uint64_t inner, uint64_t outer,
                           uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, int swizzle_bytes);

bool make_tmap_2d(void* tmap, const void* base, int elem_bytes, uint64_t inner, uint64_t outer,
                  uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, int swizzle_bytes) {
  const TmapKey key{base, inner, outer, row_stride_bytes, box_inner, box_outer, elem_bytes, swizzle_bytes};
  const size_t slot = tmap_hash(key);
  {
    std::lock_guard<std::mutex> lk(g_tmap_mu);
    const TmapEntry& e = g_tmap_cache[slot];
    if (e.valid && e.key == key) {
      std::memcpy(tmap, &e.map, sizeof(CUtensorMap));
      return true;
    }
  }
  if (!encode_tmap_2d(tmap, base, elem_bytes, inner, outer, row_stride_bytes, box_inner, box_outer, swizzle_bytes))
    return false;
  std::lock_guard<std::mutex> lk(g_tmap_mu);
  TmapEntry& e = g_tmap_cache[slot];
  e.key = key;
  std::memcpy(&e.map, tmap, sizeof(CUtensorMap));
  e.valid = true;
  return true;
}

static bool encode_tmap_2d(void* tmap, const void* base, int elem_bytes, uint64_t inner, uint64_t outer,
                           uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, int swizzle_bytes) {
  auto enc = get_encode();
  if (!enc) return false;
  CUtensorMapDataType dt = elem_bytes == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                         : elem_bytes == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                           : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(reinterpret_cast<CUtensorMap*>(tmap), dt, 2, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                   : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                   : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                         : CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace fq
