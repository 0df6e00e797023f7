// fq_common.cuh — device helpers shared by the sm_100a kernels of libfq (product path only).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fq.h"

namespace fq {

// ---- dtype traits -------------------------------------------------------------------------------
template <typename T> struct Dt;
template <> struct Dt<__nv_bfloat16> {
  static constexpr int id = FQ_BF16;
  __device__ static float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
  __device__ static __nv_bfloat16 from_f(float v) { return __float2bfloat16_rn(v); }
  __device__ static __nv_bfloat16 from_d(double v) { return __double2bfloat16(v); }
  // int4 -> (128 + (n ^ 8)) magic: exponent of 128, mantissa LSB weight 1.
  static constexpr uint32_t kMagic4 = 0x43084308u;  // (x & 0x000F000F) ^ this -> 0x43 | (n^8)
  static constexpr uint32_t kBias4 = 0x43084308u;   // bf16x2 (136, 136)
};
template <> struct Dt<__half> {
  static constexpr int id = FQ_FP16;
  __device__ static float to_f(__half v) { return __half2float(v); }
  __device__ static __half from_f(float v) { return __float2half_rn(v); }
  __device__ static __half from_d(double v) { return __double2half(v); }
  static constexpr uint32_t kMagic4 = 0x64086408u;  // fp16 1024 + (n^8)
  static constexpr uint32_t kBias4 = 0x64086408u;   // fp16x2 (1032, 1032)
};
template <> struct Dt<float> {
  static constexpr int id = FQ_FP32;
  __device__ static float to_f(float v) { return v; }
};

__device__ __forceinline__ bool is_finite_f(float x) { return isfinite(x); }

// ---- PTX helpers ----------------------------------------------------------------------------------
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ldg_keep(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t lop3_and_xor(uint32_t a, uint32_t b, uint32_t c) {
  // (a & b) ^ c
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0x6A;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

}  // namespace fq
