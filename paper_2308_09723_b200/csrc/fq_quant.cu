// fq_quant.cu — kernels A1 (adaptive range pyramid + level flags) and A3 (scale, quantize, pack).
//
// A3 follows App. A: s = 2*max|A_group|/(2^b-1), Q = integer(A/s), with groups of
// `group` contiguous elements along K of each paper column (§4.1), scales stored in the
// activation dtype.  Arithmetic contract (bit-exact with the oracle):
//   * amax is exact;  s = RNE_dtype((double)(2*amax) / (2^b-1)) — the double quotient can never sit
//     on a bf16/fp16 tie, so this equals one rounding of the exact rational (R4);
//   * q = clamp(round_half_away(x / s)): for 16-bit W under a normal scale, x * rcp(s) nudged 2^-15
//     away from zero and rounded to nearest (exact: the estimate is within 2^-20 of x / s, off-tie
//     quotients are >= 2^-14 from a half-integer); fp32 W and subnormal scales: the half-integer
//     test |x| - (floor(y) + 1/2) s >= 0 evaluated exactly by one fma; clamp to [-2^(b-1), 2^(b-1)-1].
// A1 follows P:147-149 §3.3 under reading R6: level L fires iff some child group range is below
// alpha * its parent's range, compared exactly as 1000*child < alpha_milli*parent in fp64.
//
// Layout: power-of-two groups of 32 .. 1024 run quantize_warp_kernel -- one warp per 1024-element
// unit of a column, a group = a run of lanes, no shared memory or block barrier.  Other groups run
// quantize_kernel: one CTA per K-slice of a column, each thread holding <= 8 chunks of 8 elements
// in registers; pass 1 writes one max|.| per chunk to shared memory, pass 2 reduces chunks to
// groups and writes the scales, pass 3 turns the register-resident chunks into codes.  Both read W
// from HBM once and write codes/scales once (the algorithmic minimum).
#include <algorithm>

#include "fq_common.cuh"
#include "fq_internal.h"

namespace fq {

// One 8-element chunk of a weight row kept in its raw storage format (16 B bf16/fp16, 32 B fp32).
template <typename TIn>
struct Chunk8 {
  static constexpr int NV = sizeof(TIn) / 2;  // uint4 words
  uint4 r[NV];
  __device__ __forceinline__ void load(const TIn* p) {
#pragma unroll
    for (int i = 0; i < NV; ++i) r[i] = __ldg(reinterpret_cast<const uint4*>(p) + i);
  }
  __device__ __forceinline__ void lds(uint32_t addr) {
#pragma unroll
    for (int i = 0; i < NV; ++i) r[i] = lds128(addr + 16 * i);
  }
  __device__ __forceinline__ void decode(float (&v)[8]) const;
  __device__ __forceinline__ float amax() const;
};
template <>
__device__ __forceinline__ void Chunk8<__nv_bfloat16>::decode(float (&v)[8]) const {
  const uint32_t w[4] = {r[0].x, r[0].y, r[0].z, r[0].w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[2 * i] = __uint_as_float(w[i] << 16);
    v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}
template <>
__device__ __forceinline__ void Chunk8<__half>::decode(float (&v)[8]) const {
  const __half2* h = reinterpret_cast<const __half2*>(&r[0]);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __half22float2(h[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}
template <>
__device__ __forceinline__ void Chunk8<float>::decode(float (&v)[8]) const {
  v[0] = __uint_as_float(r[0].x); v[1] = __uint_as_float(r[0].y);
  v[2] = __uint_as_float(r[0].z); v[3] = __uint_as_float(r[0].w);
  v[4] = __uint_as_float(r[1].x); v[5] = __uint_as_float(r[1].y);
  v[6] = __uint_as_float(r[1].z); v[7] = __uint_as_float(r[1].w);
}

// max|x| of a chunk of 16-bit values straight from the bit patterns: with the sign bit cleared,
// finite values order like unsigned integers and every Inf/NaN pattern lies above all of them, so
// two packed 16-bit unsigned max operations per pair replace the per-element decode + FMNMX.
// Returns +inf if any element is non-finite (the group is then flagged).
template <>
__device__ __forceinline__ float Chunk8<__nv_bfloat16>::amax() const {
  const uint32_t m = __vmaxu2(__vmaxu2(r[0].x & 0x7FFF7FFFu, r[0].y & 0x7FFF7FFFu),
                              __vmaxu2(r[0].z & 0x7FFF7FFFu, r[0].w & 0x7FFF7FFFu));
  const uint32_t h = max(m & 0xFFFFu, m >> 16);
  return h >= 0x7F80u ? __int_as_float(0x7f800000) : __uint_as_float(h << 16);
}
template <>
__device__ __forceinline__ float Chunk8<__half>::amax() const {
  const uint32_t m = __vmaxu2(__vmaxu2(r[0].x & 0x7FFF7FFFu, r[0].y & 0x7FFF7FFFu),
                              __vmaxu2(r[0].z & 0x7FFF7FFFu, r[0].w & 0x7FFF7FFFu));
  const uint32_t h = max(m & 0xFFFFu, m >> 16);
  return h >= 0x7C00u ? __int_as_float(0x7f800000) : __half2float(__ushort_as_half((unsigned short)h));
}

// max|x| over a chunk; +inf if any element is non-finite (the group is then flagged).
__device__ __forceinline__ float chunk_amax(const float (&v)[8]) {
  float m = 0.f;
  bool fin = true;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    fin &= isfinite(v[i]);
    m = fmaxf(m, fabsf(v[i]));
  }
  return fin ? m : __int_as_float(0x7f800000);
}

template <>
__device__ __forceinline__ float Chunk8<float>::amax() const {
  float v[8];
  decode(v);
  return chunk_amax(v);
}

constexpr int kQThreads = 256;

// ------------------------------------------------------------------------------------- A3
constexpr int kQCpt = 8;      // chunks per thread cached in registers by the quantizer
constexpr int kQSlice = 12288;  // target K-slice per CTA (192 threads at kQCpt = 8)

// Pass 2 of A3 for one group: the scale from the group's max|x| (App. A; R4).  Returns
// the status bits (1: non-finite weights, 2: scale overflows the scale dtype); s = 0 zeroes the codes.
template <typename TS, int BITS>
__device__ __forceinline__ int group_scale(float amax, float& s, TS& s_t) {
  s = 0.f;
  if (!isfinite(amax)) {
    s_t = Dt<TS>::from_f(0.f);
    return 1;
  }
  s_t = Dt<TS>::from_d(2.0 * (double)amax / (double)((1 << BITS) - 1));
  s = Dt<TS>::to_f(s_t);
  if (!isfinite(s)) {
    s = 0.f;
    s_t = Dt<TS>::from_f(0.f);
    return 2;
  }
  return 0;
}

// Smallest normal value of the scale dtype: below it the scale carries fewer significant bits, so
// |x| / s may leave [-2^(b-1) - 1/2, 2^(b-1) + 1/2] and the fast path's one-sided clamp no longer
// suffices (fp16 scales of groups with amax < ~2^-14 (2^b - 1) / 2).
template <typename TS>
__device__ __forceinline__ float scale_min_normal() {
  return Dt<TS>::id == FQ_FP16 ? 6.103515625e-05f /* 2^-14 */ : 1.17549435e-38f /* 2^-126 */;
}

// Pass 3 of A3 for one 8-element chunk: the codes of v[0..8) under scale s (rs = rcp(s), 0 when
// s == 0), packed as stored -- int4: 32 bits (.x), int8: 64 bits, int3: 24 bits, int2: 16 bits.
// fast: 16-bit W under a normal scale (the caller's per-group choice); else the exact test below.
template <typename TIn, int BITS>
__device__ __forceinline__ uint2 pack_chunk(const float (&v)[8], float s, float rs, bool fast) {
  constexpr int lo = -(1 << (BITS - 1)), hi = (1 << (BITS - 1)) - 1;
  // offset-binary code u = q + 2^(b-1) in [0, 2^b - 1]; the stored two's complement field is
  // u ^ 2^(b-1).
  uint32_t u[8];
  if (Dt<TIn>::id != FQ_FP32 && fast) {
    // 16-bit W, signed magic-number rounding: t = fma(x, rcp(s), 1.5 * 2^23 + 2^(b-1)) holds
    // u' = rn_even(x / s) + 2^(b-1) in its low mantissa bits (the magic is even, the sum stays in
    // [2^23, 2^24)), so the raw bits ARE 0x4B400000 + u'.  |x| <= amax keeps x / s within
    // (-2^(b-1) - 1/2, 2^(b-1) + 1/2), so only the top needs a clamp.
    constexpr float kMagic = 12582912.f + (float)(1 << (BITS - 1));
    constexpr int32_t kBase = 0x4B400000;
    int32_t tb[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      // y = x * rcp(s) nudged 2^-15 away from zero: |x * rcp(s) - x / s| <= 8.5 * 2^-23 < 2^-20, and
      // an off-tie quotient is >= 2^-14 from every half-integer (x, s with <= 11 significant bits),
      // so the nudge carries exact ties past the half-integer (round half AWAY) and leaves every other
      // quotient on its side; the magic add then rounds to the nearest integer.  Exhaustively checked
      // against the exact rational rounding on every finite bf16 pattern (tests/test_gpu_quant.py).
      const float nudge = __uint_as_float((__float_as_uint(v[i]) & 0x80000000u) | 0x38000000u);  // +-2^-15
      const float t = fmaf(v[i], rs, nudge) + kMagic;
      tb[i] = min(__float_as_int(t), kBase + (1 << BITS) - 1);
    }
    // pack the raw bit patterns: every field carries kBase, whose packed sum is one constant
    if (BITS == 4) {
      uint32_t w = (uint32_t)tb[7];
#pragma unroll
      for (int i = 6; i >= 0; --i) w = w * 16u + (uint32_t)tb[i];
      constexpr uint32_t kBias = (uint32_t)kBase * 0x11111111u;
      return make_uint2((w - kBias) ^ 0x88888888u, 0u);
    }
    if (BITS == 8) {
      constexpr uint32_t kBias = (uint32_t)kBase * 0x01010101u;
      uint2 w;
      w.x = ((uint32_t)tb[3] * 256u + (uint32_t)tb[2]) * 256u * 256u + (uint32_t)tb[1] * 256u + (uint32_t)tb[0];
      w.y = ((uint32_t)tb[7] * 256u + (uint32_t)tb[6]) * 256u * 256u + (uint32_t)tb[5] * 256u + (uint32_t)tb[4];
      w.x = (w.x - kBias) ^ 0x80808080u;
      w.y = (w.y - kBias) ^ 0x80808080u;
      return w;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) u[i] = (uint32_t)(tb[i] - kBase);
  } else {
    // fp32 W (24-bit x: no tie-distance guarantee) and subnormal scales: round_half_away(|x| / s)
    // decided exactly.  c = floor(y) for an estimate y within 1/2 of |x| / s; |x| / s >= c + 1/2
    // iff |x| - (c + 1/2) s >= 0, and fma evaluates that difference exactly before its one rounding,
    // which keeps the sign (its exact value is a multiple of 2^-149, so it never rounds to 0).
    // Scales below 2^-100 are first rescaled with x by 2^64 (exact) so rcp(s) stays finite.
    const float k2 = s < 7.88860905e-31f /* 2^-100 */ ? 1.8446744e19f /* 2^64 */ : 1.f;
    const float ss = s * k2, rr = s == 0.f ? 0.f : __frcp_rn(ss);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float a = fabsf(v[i]) * k2;
      const float c = floorf(a * rr);
      float m = fmaf(-(c + 0.5f), ss, a) >= 0.f ? c + 1.f : c;
      if (s == 0.f) m = 0.f;
      const bool neg = v[i] < 0.f;
      m = fminf(m, neg ? (float)-lo : (float)hi);
      u[i] = (uint32_t)(int)((neg ? -m : m) + (float)-lo);
    }
    if (BITS == 4) {
      uint32_t w = u[7];
#pragma unroll
      for (int i = 6; i >= 0; --i) w = w * 16u + u[i];
      return make_uint2(w ^ 0x88888888u, 0u);
    }
    if (BITS == 8) {
      uint2 w;
      w.x = ((u[3] * 256u + u[2]) * 256u + u[1]) * 256u + u[0];
      w.y = ((u[7] * 256u + u[6]) * 256u + u[5]) * 256u + u[4];
      return make_uint2(w.x ^ 0x80808080u, w.y ^ 0x80808080u);
    }
  }
  // int3 / int2 (reading R19): the chunk's b-bit two's-complement fields of the
  // column's little-endian bit stream
  uint32_t w = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) w |= ((u[i] ^ (1u << (BITS - 1))) & ((1u << BITS) - 1)) << (BITS * i);
  return make_uint2(w, 0u);
}

// Pass 3 of A3 for one chunk, stored as chunk `chunk` of column n's packed codes.
template <typename TIn, int BITS>
__device__ __forceinline__ void emit_chunk(const float (&v)[8], float s, float rs, bool fast,
                                           uint8_t* __restrict__ codes, int n, int K, int chunk) {
  const uint2 w = pack_chunk<TIn, BITS>(v, s, rs, fast);
  if (BITS == 4) {
    reinterpret_cast<uint32_t*>(codes + (size_t)n * (K / 2))[chunk] = w.x;
  } else if (BITS == 8) {
    reinterpret_cast<uint2*>(codes + (size_t)n * K)[chunk] = w;
  } else if (BITS == 2) {
    reinterpret_cast<uint16_t*>(codes + (size_t)n * (K / 4))[chunk] = (uint16_t)w.x;
  } else {
    uint8_t* b = codes + (size_t)n * (K / 8 * 3) + (size_t)chunk * 3;
    b[0] = (uint8_t)w.x;
    b[1] = (uint8_t)(w.x >> 8);
    b[2] = (uint8_t)(w.x >> 16);
  }
}

template <typename TIn, typename TS, int BITS, int CPT = kQCpt>
__global__ void __launch_bounds__(sizeof(TIn) == 4 ? 512 : 1024) quantize_kernel(const TIn* __restrict__ W, int K,
                                                             int KS, int N, int group,
                                                             uint8_t* __restrict__ codes,
                                                             TS* __restrict__ scales,
                                                             int32_t* __restrict__ status,
                                                             const float* __restrict__ amax_tab,
                                                             int tab_r0, int tab_span) {
  extern __shared__ float smem[];
  // CTA = one K-slice of KS elements (a multiple of the group) of one paper column: long columns
  // are split so that every CTA stays small enough for several to share an SM.
  const int nsl = K / KS;
  const int n = blockIdx.x / nsl, sl = blockIdx.x - n * nsl;
  const int nchunk = KS >> 3;
  const int G = KS / group;
  const int cpg = group >> 3;  // chunks per group
  float* pm = smem;            // [nchunk]
  float* sc = smem + nchunk;   // [G] scale as float (0 => codes 0)
  float* sr = sc + G;          // [G] rcp(scale) (0 when the scale is 0)
  __shared__ int s_status;
  const TIn* row = W + (size_t)n * K + (size_t)sl * KS;
  if (threadIdx.x == 0) s_status = 0;

  // pass 1: chunk maxima; the raw chunks stay in registers for pass 3 (CPT chunks per thread,
  // the launcher sizes the CTA so that K <= 8 * CPT * blockDim.x) — W is read from HBM once.
  const int T = blockDim.x;
  Chunk8<TIn> raw[CPT];
  // all loads first (CPT x 16 B in flight per thread), then the maxima
#pragma unroll
  for (int i = 0; i < CPT; ++i) {
    const int c = threadIdx.x + i * T;
    if (c < nchunk) raw[i].load(row + (size_t)c * 8);
  }
#pragma unroll
  for (int i = 0; i < CPT; ++i) {
    const int c = threadIdx.x + i * T;
    if (c < nchunk) pm[c] = raw[i].amax();
  }
  __syncthreads();

  // pass 2: group maxima -> scales
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto finish_group = [&](int j, float amax) {
    float s;
    TS s_t;
    const int st = group_scale<TS, BITS>(amax, s, s_t);
    sc[j] = s;
    sr[j] = s == 0.f ? 0.f : __frcp_rn(s);
    scales[(size_t)(sl * G + j) * N + n] = s_t;
    if (st) atomicOr(&s_status, st);
  };
  if (amax_tab) {
    // row-parallel shard of a group that spans several K-shards (TP, group > K/world): the group
    // amax is the max of the shards' column maxima (table [world][N] after the MAX all-reduce);
    // the shard holds one group (G == 1).
    if (threadIdx.x == 0) {
      float m = 0.f;
      for (int r = tab_r0; r < tab_r0 + tab_span; ++r) m = fmaxf(m, amax_tab[(size_t)r * N + n]);
      finish_group(0, m);
    }
  } else if (cpg <= 32) {
    for (int j = threadIdx.x; j < G; j += T) {
      float m = 0.f;
      for (int i = 0; i < cpg; ++i) m = fmaxf(m, pm[j * cpg + i]);  // fmaxf keeps +inf
      finish_group(j, m);
    }
  } else {
    for (int j = warp; j < G; j += T / 32) {
      float m = 0.f;
      for (int i = lane; i < cpg; i += 32) m = fmaxf(m, pm[j * cpg + i]);
#pragma unroll
      for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) finish_group(j, m);
    }
  }
  __syncthreads();

  // pass 3: codes
  const uint32_t cpg_magic = 0xFFFFFFFFu / (uint32_t)cpg + 1u;  // ceil(2^32 / cpg), cpg >= 2
#pragma unroll
  for (int ci = 0; ci < CPT; ++ci) {
    const int c = threadIdx.x + ci * T;
    if (c >= nchunk) break;
    float v[8];
    raw[ci].decode(v);
    const int j = (int)__umulhi((uint32_t)c, cpg_magic);  // c / cpg, exact for c < 2^32 / cpg
    emit_chunk<TIn, BITS>(v, sc[j], sr[j], sc[j] >= scale_min_normal<TS>(), codes, n, K, sl * nchunk + c);
  }
  __syncthreads();
  if (threadIdx.x == 0 && s_status && status) atomicOr(status, s_status);
}

// A3, one warp per 1024-element unit of a column (the product kernel for power-of-two groups of
// 32 .. 1024): lane l holds elements [32 l, 32 l + 32) of the unit -- four chunks of ONE group --
// so a group is a run of group/32 lanes and its max a butterfly of log2(group/32) shuffles.  Every
// lane then derives its group's scale (the same instructions warp-wide), quantizes its 32 elements
// from registers and writes them with one (int4) / two (int8) 16-byte stores.  No shared memory and
// no block barrier: each warp keeps kQwUnits units (kQwUnits x 64 B per lane) of loads in flight.
// The per-column kernel above serialises load -> reduce -> emit inside each CTA (0.54 of HBM on
// OPT-175B FC1, profiles/r02/quantize_adapt_ncu.txt).
constexpr int kQwThreads = 256;

template <typename TIn, typename TS, int BITS>
__global__ void __launch_bounds__(kQwThreads) quantize_warp_kernel(const TIn* __restrict__ W, int K, int N,
                                                                   int glog, uint8_t* __restrict__ codes,
                                                                   TS* __restrict__ scales,
                                                                   int32_t* __restrict__ status) {
  constexpr int R = sizeof(TIn) == 4 ? 1 : 2;  // units in flight per warp (64 B of W per lane each)
  const int lane = threadIdx.x & 31;
  const int lpg = 1 << (glog - 5);  // lanes per group
  const int upc = (K + 1023) >> 10;  // units per column (the last may be partial: whole groups)
  const long units = (long)N * upc;
  const long nw = (long)gridDim.x * (kQwThreads / 32);
  int st = 0;
  for (long u0 = (long)blockIdx.x * (kQwThreads / 32) + (threadIdx.x >> 5); u0 < units; u0 += nw * R) {
    Chunk8<TIn> raw[R][4];
    int nn[R], kk[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const long u = u0 + r * nw;
      nn[r] = (int)(u / upc);
      kk[r] = (int)(u - (long)nn[r] * upc) * 1024 + lane * 32;
      if (u < units && kk[r] < K) {
        const TIn* p = W + (size_t)nn[r] * K + kk[r];
#pragma unroll
        for (int c = 0; c < 4; ++c) raw[r][c].load(p + 8 * c);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (u0 + r * nw >= units) break;  // warp-uniform
      const bool ok = kk[r] < K;        // a group lies wholly inside or outside K
      float m = 0.f;
      if (ok) {
#pragma unroll
        for (int c = 0; c < 4; ++c) m = fmaxf(m, raw[r][c].amax());  // +inf marks a non-finite element
      }
      for (int o = 1; o < lpg; o <<= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (!ok) continue;
      float s;
      TS s_t;
      st |= group_scale<TS, BITS>(m, s, s_t);
      const float rs = s == 0.f ? 0.f : __frcp_rn(s);
      const bool fast = s >= scale_min_normal<TS>();
      const int n = nn[r], k = kk[r];
      if ((lane & (lpg - 1)) == 0) scales[(size_t)(k >> glog) * N + n] = s_t;
      uint2 w[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float v[8];
        raw[r][c].decode(v);
        w[c] = pack_chunk<TIn, BITS>(v, s, rs, fast);
      }
      if (BITS == 4) {
        *reinterpret_cast<uint4*>(codes + (size_t)n * (K / 2) + k / 2) = make_uint4(w[0].x, w[1].x, w[2].x, w[3].x);
      } else if (BITS == 8) {
        uint4* d = reinterpret_cast<uint4*>(codes + (size_t)n * K + k);
        d[0] = make_uint4(w[0].x, w[0].y, w[1].x, w[1].y);
        d[1] = make_uint4(w[2].x, w[2].y, w[3].x, w[3].y);
      } else if (BITS == 2) {
        *reinterpret_cast<uint2*>(codes + (size_t)n * (K / 4) + k / 4) =
            make_uint2(w[0].x | (w[1].x << 16), w[2].x | (w[3].x << 16));
      } else {  // four 24-bit fields = three words
        uint32_t* d = reinterpret_cast<uint32_t*>(codes + (size_t)n * (K / 8 * 3) + k / 8 * 3);
        d[0] = w[0].x | (w[1].x << 24);
        d[1] = (w[1].x >> 8) | (w[2].x << 16);
        d[2] = (w[2].x >> 16) | (w[3].x << 8);
      }
    }
  }
  if (st && status) atomicOr(status, st);
}

// ------------------------------------------------------------------------------------- A1
// Per column: chunk maxima -> finest-level group maxima -> pairwise up the ladder (each level is
// an exact halving of the one above, so parent(j) = j/2) -> OR of the level flags.
constexpr int kMaxLevels = 16;

template <typename TIn>
__global__ void __launch_bounds__(kQThreads) adapt_flags_kernel(const TIn* __restrict__ W, int K,
                                                                int N, int nlev, int gfin,
                                                                uint32_t alpha_milli,
                                                                int32_t* __restrict__ flags, int flag_ofs,
                                                                float* __restrict__ colmax,
                                                                int32_t* __restrict__ status) {
  extern __shared__ float smem[];
  const int nchunk = K >> 3;
  const int Gf = K / gfin;
  float* pm = smem;               // [nchunk]
  float* lev = smem + nchunk;     // levels finest..0 packed: offsets below
  __shared__ int s_flag[kMaxLevels];
  __shared__ int s_status;
  if (threadIdx.x < kMaxLevels) s_flag[threadIdx.x] = 0;
  if (threadIdx.x == 0) s_status = 0;
  const int n = blockIdx.x;
  const TIn* row = W + (size_t)n * K;
#pragma unroll 4
  for (int c = threadIdx.x; c < nchunk; c += kQThreads) {
    Chunk8<TIn> ch;
    ch.load(row + (size_t)c * 8);
    pm[c] = ch.amax();
  }
  __syncthreads();
  // finest level L = nlev-1 stored at lev[0 .. Gf)
  const int cpg = gfin >> 3;
  for (int j = threadIdx.x; j < Gf; j += kQThreads) {
    float m = 0.f;
    for (int i = 0; i < cpg; ++i) m = fmaxf(m, pm[j * cpg + i]);
    lev[j] = m;
  }
  __syncthreads();
  // coarser levels: level L has Gf >> (nlev-1-L) groups; offset off(L) accumulates.
  int off_child = 0, cnt_child = Gf;
  for (int L = nlev - 2; L >= 0; --L) {
    const int off_par = off_child + cnt_child, cnt_par = cnt_child >> 1;
    for (int j = threadIdx.x; j < cnt_par; j += kQThreads)
      lev[off_par + j] = fmaxf(lev[off_child + 2 * j], lev[off_child + 2 * j + 1]);
    __syncthreads();
    // flag for child level L+1 against parent level L
    bool fire = false;
    for (int j = threadIdx.x; j < cnt_child; j += kQThreads) {
      const double ch = lev[off_child + j], pa = lev[off_par + (j >> 1)];
      fire |= (1000.0 * ch < (double)alpha_milli * pa);
    }
    if (__syncthreads_or(fire) && threadIdx.x == 0) s_flag[L + 1] = 1;
    off_child = off_par;
    cnt_child = cnt_par;
  }
  if (threadIdx.x == 0 && !isfinite(lev[off_child])) s_status = 1;
  if (threadIdx.x == 0 && colmax) colmax[n] = lev[off_child];  // level 0: max|W[n, :]| (+inf: non-finite)
  __syncthreads();
  if (flags && threadIdx.x >= 1 && threadIdx.x < nlev && s_flag[threadIdx.x])
    atomicOr(&flags[flag_ofs + threadIdx.x - 1], 1);
  if (threadIdx.x == 0 && s_status && status) atomicOr(status, 1);
}

// Warp-per-column variant (K <= 65536): one warp owns a column and its private shared-memory pyramid,
// so the levels need only __syncwarp -- the block-wide version's __syncthreads per level and its
// mostly idle threads at the coarse levels made it issue-bound (13.8 instructions per weight).
template <typename TIn, int WPC>
__global__ void __launch_bounds__(32 * WPC) adapt_flags_warp_kernel(const TIn* __restrict__ W, int K, int N, int nlev,
                                                                     int gfin, uint32_t alpha_milli,
                                                                     int32_t* __restrict__ flags, int flag_ofs,
                                                                     float* __restrict__ colmax,
                                                                     int32_t* __restrict__ status) {
  extern __shared__ float smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = blockIdx.x * WPC + warp;
  if (n >= N) return;  // whole warps leave (no block-level barrier below)
  const int nchunk = K >> 3;
  const int Gf = K / gfin;
  float* pm = smem + (size_t)warp * (nchunk + 2 * Gf);  // [nchunk] chunk maxima
  float* lev = pm + nchunk;                              // levels finest .. 0, packed
  const TIn* row = W + (size_t)n * K;
#pragma unroll 8
  for (int c = lane; c < nchunk; c += 32) {
    Chunk8<TIn> ch;
    ch.load(row + (size_t)c * 8);
    pm[c] = ch.amax();
  }
  __syncwarp();
  const int cpg = gfin >> 3;
  for (int j = lane; j < Gf; j += 32) {
    float m = 0.f;
    for (int i = 0; i < cpg; ++i) m = fmaxf(m, pm[j * cpg + i]);
    lev[j] = m;
  }
  __syncwarp();
  uint32_t fired = 0;  // bit L: level L fires (some child group below alpha x its parent)
  int off_child = 0, cnt_child = Gf;
  for (int L = nlev - 2; L >= 0; --L) {
    const int off_par = off_child + cnt_child, cnt_par = cnt_child >> 1;
    bool fire = false;
    for (int j = lane; j < cnt_par; j += 32) {
      const float a = lev[off_child + 2 * j], b = lev[off_child + 2 * j + 1];
      const float pa = fmaxf(a, b);
      lev[off_par + j] = pa;
      const double ap = (double)alpha_milli * pa;
      fire |= (1000.0 * (double)a < ap) | (1000.0 * (double)b < ap);
    }
    if (__any_sync(0xffffffffu, fire)) fired |= 1u << (L + 1);
    __syncwarp();
    off_child = off_par;
    cnt_child = cnt_par;
  }
  if (lane == 0) {
    const float top = lev[off_child];  // level 0: max|W[n, :]| (+inf: non-finite)
    if (colmax) colmax[n] = top;
    if (!isfinite(top) && status) atomicOr(status, 1);
    if (flags)
      for (int L = 1; L < nlev; ++L)
        if (fired & (1u << L)) atomicOr(&flags[flag_ofs + L - 1], 1);
  }
}

// ------------------------------------------------------------------------------------- launchers
struct AmaxTab {
  const float* tab;
  int r0, span;
};

template <typename TIn, typename TS, int BITS, int CPT>
static cudaError_t launch_quant_c(const void* W, int K, int N, int group, void* codes, void* scales,
                                  int32_t* status, cudaStream_t st, int slice, AmaxTab at) {
  // K-slice per CTA: the fewest slices that bring it to <= kQSlice elements (slices are whole
  // groups; a group longer than that, e.g. one scale per column, keeps the whole column).
  const int G = K / group;
  int nsl = G;
  for (int d = 1; d <= G; ++d)
    if (G % d == 0 && K / d <= slice) { nsl = d; break; }
  const int KS = K / nsl;
  const size_t smem = (size_t)(KS / 8 + 2 * (KS / group)) * sizeof(float);
  auto kern = quantize_kernel<TIn, TS, BITS, CPT>;
  if (smem > 48 * 1024) {  // sized for the largest group the API accepts (65536 elements)
    cudaError_t e = ensure_smem_attr<quantize_kernel<TIn, TS, BITS, CPT>>((65536 / 8 + 2) * (int)sizeof(float));
    if (e != cudaSuccess) return e;
  }
  // threads: enough that every 8-element chunk is cached in registers (<= kQCpt per thread)
  const int nchunk = KS / 8;
  int threads = ((nchunk + CPT - 1) / CPT + 31) / 32 * 32;
  threads = threads < 128 ? 128 : threads;
  if (threads > (sizeof(TIn) == 4 ? 512 : 1024)) return cudaErrorInvalidValue;  // rejected by the API
  kern<<<(unsigned)N * nsl, threads, smem, st>>>((const TIn*)W, K, KS, N, group, (uint8_t*)codes, (TS*)scales,
                                                 status, at.tab, at.r0, at.span);
  return cudaGetLastError();
}

template <typename TIn, typename TS, int BITS>
static cudaError_t launch_quant(const void* W, int K, int N, int group, void* codes, void* scales,
                                int32_t* status, cudaStream_t st, AmaxTab at) {
#ifndef FQ_QUANT_WARP
#define FQ_QUANT_WARP 1
#endif
  if (FQ_QUANT_WARP && !at.tab && group >= 32 && group <= 1024 && (group & (group - 1)) == 0) {
    auto kern = quantize_warp_kernel<TIn, TS, BITS>;
    static int bps = 0;  // resident CTAs per SM (per instantiation)
    if (!bps) {
      cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, kQwThreads, 0);
      if (e != cudaSuccess) return e;
      bps = std::max(bps, 1);
    }
    const long units = (long)N * ((K + 1023) / 1024);
    const long grid = std::min<long>((units + kQwThreads / 32 - 1) / (kQwThreads / 32), (long)bps * num_sms());
    kern<<<(unsigned)grid, kQwThreads, 0, st>>>((const TIn*)W, K, N, __builtin_ctz(group), (uint8_t*)codes,
                                                (TS*)scales, status);
    return cudaGetLastError();
  }
  // per-column kernel: row-parallel shards of groups spanning several shards (amax table), groups
  // of 16, above 1024 or not a power of two.  Measured on B200 (OPT FC1/FC2): 8 chunks per thread and
  // 12288-element slices beat 4 chunks and 4096 / 6144 / 24576-element slices
  return launch_quant_c<TIn, TS, BITS, kQCpt>(W, K, N, group, codes, scales, status, st, kQSlice, at);
}

template <typename TIn, typename TS>
static cudaError_t launch_quant_b(int bits, const void* W, int K, int N, int group, void* codes,
                                  void* scales, int32_t* status, cudaStream_t st, AmaxTab at) {
  switch (bits) {
    case 2: return launch_quant<TIn, TS, 2>(W, K, N, group, codes, scales, status, st, at);
    case 3: return launch_quant<TIn, TS, 3>(W, K, N, group, codes, scales, status, st, at);
    case 4: return launch_quant<TIn, TS, 4>(W, K, N, group, codes, scales, status, st, at);
    default: return launch_quant<TIn, TS, 8>(W, K, N, group, codes, scales, status, st, at);
  }
}

template <typename TIn>
static cudaError_t launch_quant_s(int sdt, int bits, const void* W, int K, int N, int group,
                                  void* codes, void* scales, int32_t* status, cudaStream_t st, AmaxTab at) {
  return sdt == FQ_BF16
             ? launch_quant_b<TIn, __nv_bfloat16>(bits, W, K, N, group, codes, scales, status, st, at)
             : launch_quant_b<TIn, __half>(bits, W, K, N, group, codes, scales, status, st, at);
}

cudaError_t run_quantize(int wdt, int sdt, int bits, const void* W, int K, int N, int group,
                         void* codes, void* scales, int32_t* status, cudaStream_t st,
                         const float* amax_tab, int tab_r0, int tab_span) {
  const AmaxTab at{amax_tab, tab_r0, tab_span};
  switch (wdt) {
    case FQ_BF16: return launch_quant_s<__nv_bfloat16>(sdt, bits, W, K, N, group, codes, scales, status, st, at);
    case FQ_FP16: return launch_quant_s<__half>(sdt, bits, W, K, N, group, codes, scales, status, st, at);
    default: return launch_quant_s<float>(sdt, bits, W, K, N, group, codes, scales, status, st, at);
  }
}

template <typename TIn>
static cudaError_t launch_adapt(const void* W, int K, int N, int nlev, int gfin, uint32_t alpha,
                                int32_t* flags, int flag_ofs, float* colmax, int32_t* status, cudaStream_t st) {
  const int Gf = K / gfin;
  const size_t per_warp = (size_t)(K / 8 + 2 * Gf) * sizeof(float);
  // warp-per-column for columns whose pyramid fits 12 KB (K <= ~16384: two 8-warp CTAs per SM);
  // long columns (e.g. OPT FC2, K = 49152) keep the block-wide kernel, which already streams them
  // near HBM speed
  if (per_warp <= 12 * 1024) {
    auto kw = adapt_flags_warp_kernel<TIn, 8>;
    cudaError_t e = ensure_smem_attr<adapt_flags_warp_kernel<TIn, 8>>(8 * 12 * 1024);
    if (e != cudaSuccess) return e;
    kw<<<(N + 7) / 8, 256, 8 * per_warp, st>>>((const TIn*)W, K, N, nlev, gfin, alpha, flags, flag_ofs, colmax,
                                               status);
    return cudaGetLastError();
  }
  const size_t smem = (size_t)(K / 8 + 2 * Gf) * sizeof(float);
  auto kern = adapt_flags_kernel<TIn>;
  if (smem > 48 * 1024) {  // sized for the largest K the API accepts (2^20, finest group >= 16)
    const size_t smax = (size_t)((1 << 20) / 8 + 2 * ((1 << 20) / 16)) * sizeof(float);
    cudaError_t e = ensure_smem_attr<adapt_flags_kernel<TIn>>((int)std::min<size_t>(smax, 227 * 1024));
    if (e != cudaSuccess) return e;
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
  }
  kern<<<N, kQThreads, smem, st>>>((const TIn*)W, K, N, nlev, gfin, alpha, flags, flag_ofs, colmax, status);
  return cudaGetLastError();
}

cudaError_t run_adapt_flags(int wdt, const void* W, int K, int N, int nlev, int gfin,
                            uint32_t alpha, int32_t* flags, int flag_ofs, float* colmax, int32_t* status,
                            cudaStream_t st) {
  switch (wdt) {
    case FQ_BF16: return launch_adapt<__nv_bfloat16>(W, K, N, nlev, gfin, alpha, flags, flag_ofs, colmax, status, st);
    case FQ_FP16: return launch_adapt<__half>(W, K, N, nlev, gfin, alpha, flags, flag_ofs, colmax, status, st);
    default: return launch_adapt<float>(W, K, N, nlev, gfin, alpha, flags, flag_ofs, colmax, status, st);
  }
}

// ------------------------------------------------------------------------------------- A1 (TP)
// Coarse levels of a K-sharded matrix (row-parallel TP, world = 2^c equal K-slices): level L
// (1 <= L <= c, group K / 2^L) has group j covering shards [j * world / 2^L, (j+1) * world / 2^L),
// so its range is the max of those shards' column maxima.  Same test as A1:
// 1000 * amax_L(n, j) < alpha_milli * amax_{L-1}(n, j / 2), exact in fp64.
__global__ void __launch_bounds__(256) adapt_cross_kernel(const float* __restrict__ colmax, int world, int N,
                                                           int ncross, uint32_t alpha_milli,
                                                           int32_t* __restrict__ flags) {
  __shared__ int s_fire[8];
  if (threadIdx.x < 8) s_fire[threadIdx.x] = 0;
  __syncthreads();
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n < N) {
    float tab[64];  // world <= 64 (checked by the API)
    for (int r = 0; r < world; ++r) tab[r] = colmax[(size_t)r * N + n];
    // level 0 -> 1 -> ... -> ncross: halve the span of shards per group
    for (int L = 1; L <= ncross; ++L) {
      const int span = world >> L;  // shards per child group
      bool fire = false;
      for (int j = 0; j < (1 << L); ++j) {
        float ch = 0.f, pa = 0.f;
        for (int r = j * span; r < (j + 1) * span; ++r) ch = fmaxf(ch, tab[r]);
        for (int r = (j >> 1) * 2 * span; r < ((j >> 1) + 1) * 2 * span; ++r) pa = fmaxf(pa, tab[r]);
        fire |= (1000.0 * (double)ch < (double)alpha_milli * (double)pa);
      }
      if (fire) s_fire[L - 1] = 1;
    }
  }
  __syncthreads();
  if (threadIdx.x < ncross && s_fire[threadIdx.x]) atomicOr(&flags[threadIdx.x], 1);
}

cudaError_t run_adapt_cross(const float* colmax, int world, int N, int nlev_cross, uint32_t alpha,
                            int32_t* flags, cudaStream_t st) {
  adapt_cross_kernel<<<(N + 255) / 256, 256, 0, st>>>(colmax, world, N, nlev_cross, alpha, flags);
  return cudaGetLastError();
}

}  // namespace fq
