// fq_gemv.cu — kernels A4 (decode GEMM, weights streamed from HBM, dequantized in registers,
// multiplied on the tensor cores with mma.sync in swap-AB form) and A5 (deterministic split-K
// fixup, fused: the last-arriving CTA of a tile reduces the partials in split order).
//
// Computes C[m,n] = sum_k A[m,k] * q[n,k] * s[k/g, n]  (§4.1: "dequantize the weights to
// match the data type of the activation and perform floating-point tensor core math").  Decode is
// "bottlenecked by memory bandwidth ... weights typically dominate the memory traffic": the
// design goal is to stream each packed weight byte exactly once at HBM speed.
//
// Mapping (swap-AB): the MMA's M=16 rows are 16 output columns n, its N=8 are tokens, K=16.
//   lane = 4*gq + t.  Thread (gq,t) owns rows n0+gq and n0+gq+8 and, inside a K chunk, the
//   contiguous K segment [kc + t*SEG, kc + (t+1)*SEG) of both rows, loaded with one 16-byte
//   streaming load per row (SEG = 32 for int4, 16 for int8).  The four lanes of a quad read 64
//   contiguous bytes of a row.
//   int4: LOP3 of a 32-bit word w (nibbles n0..n7 = k..k+7) with mask 0x000F000F yields the bf16x2
//   pair (k, k+4) as 128+(n^8) [fp16: 1024+(n^8)]; one subtract gives the exact signed code.  The
//   MMA k-slots are therefore filled with the permutation (0,4),(1,5),(2,6),(3,7) of each 8-k word;
//   the activations are loaded in natural order and permuted identically with PRMT (the sum over k
//   is invariant under a common permutation of both operands).
//   int8: bytes -> fp32 magic (bf16) or fp16 magic, natural (k, k+1) pairs.
// Scales: if group % KCHUNK == 0 every MMA of a chunk lies in one group; the chunk is accumulated
//   in a fresh fp32 fragment and folded into the accumulator with one FFMA by s[j, n] (exact codes,
//   fp32 scale application).  Otherwise (group 16..112, 48, 96, ...) the codes are scaled in the
//   activation dtype before the MMA (the paper's "dequantize to the activation dtype").
// Split-K: grid.y splits K; partials go to ws[S][M][N] fp32 and the last CTA of each output tile
//   (arrival counter, self-resetting) sums them in split order -> deterministic results.
#include <algorithm>
#include <cstdlib>
#include <cstdio>

#include "fq_common.cuh"
#include "fq_internal.h"

namespace fq {

constexpr int kGemvThreads = 256;  // 8 warps; each warp owns 16*RT output columns

struct GemvParams {
  const void* A;
  const uint8_t* codes;
  const void* scales;
  void* C;
  float* ws;       // [S][M][N] partials
  int* counters;   // [gridDim.z][gridDim.x]
  int M, K, N, group, klen, cdt;
};

template <typename T>
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1, const float (&c)[4]);
template <>
__device__ __forceinline__ void mma16816<__nv_bfloat16>(float (&d)[4], const uint32_t (&a)[4],
                                                        uint32_t b0, uint32_t b1,
                                                        const float (&c)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%10,%11,%12,%13};"
      : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(c[0]), "f"(c[1]),
        "f"(c[2]), "f"(c[3]));
}
template <>
__device__ __forceinline__ void mma16816<__half>(float (&d)[4], const uint32_t (&a)[4],
                                                 uint32_t b0, uint32_t b1, const float (&c)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%10,%11,%12,%13};"
      : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(c[0]), "f"(c[1]),
        "f"(c[2]), "f"(c[3]));
}

template <typename T>
__device__ __forceinline__ uint32_t sub2(uint32_t a, uint32_t b);
template <>
__device__ __forceinline__ uint32_t sub2<__nv_bfloat16>(uint32_t a, uint32_t b) {
  __nv_bfloat162 r = __hsub2(*reinterpret_cast<__nv_bfloat162*>(&a), *reinterpret_cast<__nv_bfloat162*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}
template <>
__device__ __forceinline__ uint32_t sub2<__half>(uint32_t a, uint32_t b) {
  __half2 r = __hsub2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}
template <typename T>
__device__ __forceinline__ uint32_t mul2(uint32_t a, uint32_t b);
template <>
__device__ __forceinline__ uint32_t mul2<__nv_bfloat16>(uint32_t a, uint32_t b) {
  __nv_bfloat162 r = __hmul2(*reinterpret_cast<__nv_bfloat162*>(&a), *reinterpret_cast<__nv_bfloat162*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}
template <>
__device__ __forceinline__ uint32_t mul2<__half>(uint32_t a, uint32_t b) {
  __half2 r = __hmul2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}

// int4 word (k..k+7) -> 4 packed pairs (k,k+4),(k+1,k+5),(k+2,k+6),(k+3,k+7), exact codes.
template <typename T>
__device__ __forceinline__ void i4_pairs(uint32_t w, uint32_t (&q)[4]) {
  constexpr uint32_t mask = 0x000F000Fu;
  q[0] = sub2<T>(lop3_and_xor(w, mask, Dt<T>::kMagic4), Dt<T>::kBias4);
  q[1] = sub2<T>(lop3_and_xor(w >> 4, mask, Dt<T>::kMagic4), Dt<T>::kBias4);
  q[2] = sub2<T>(lop3_and_xor(w >> 8, mask, Dt<T>::kMagic4), Dt<T>::kBias4);
  q[3] = sub2<T>(lop3_and_xor(w >> 12, mask, Dt<T>::kMagic4), Dt<T>::kBias4);
}

// int8 word (k..k+3) -> 2 natural pairs (k,k+1),(k+2,k+3), exact codes.
template <typename T>
__device__ __forceinline__ void i8_pairs(uint32_t w, uint32_t (&q)[2]);
template <>
__device__ __forceinline__ void i8_pairs<__half>(uint32_t w, uint32_t (&q)[2]) {
  const uint32_t u = w ^ 0x80808080u;  // offset binary: u = q + 128
  q[0] = sub2<__half>(prmt(u, 0x64646464u, 0x4140u), 0x64806480u);  // (1024+u) - 1152
  q[1] = sub2<__half>(prmt(u, 0x64646464u, 0x4342u), 0x64806480u);
}
template <>
__device__ __forceinline__ void i8_pairs<__nv_bfloat16>(uint32_t w, uint32_t (&q)[2]) {
  const uint32_t u = w ^ 0x80808080u;
  float f[4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    f[i] = __uint_as_float(prmt(u, 0x4B000000u, 0x7440u + i)) - 8388736.0f;  // 2^23 + 128
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(f[2 * i + 1]), "f"(f[2 * i]));
    q[i] = r;
  }
}

template <typename T>
__device__ __forceinline__ uint32_t splat_scale(const T* scales, size_t idx) {
  const unsigned short s = __ldg(reinterpret_cast<const unsigned short*>(scales) + idx);
  return (uint32_t)s | ((uint32_t)s << 16);
}
template <typename T>
__device__ __forceinline__ float load_scale_f(const T* scales, size_t idx) {
  return Dt<T>::to_f(__ldg(scales + idx));
}

template <typename T, int BITS, int MT, bool SACC, int RT>
__global__ void __launch_bounds__(kGemvThreads, 2) gemv_kernel(const GemvParams p) {
  constexpr int SEG = (BITS == 4) ? 32 : 16;   // K elements per thread per row per chunk
  constexpr int KCH = 4 * SEG;                 // K per chunk (quad)
  constexpr int WORDS = 4;                     // 32-bit words per 16-byte load
  constexpr int KPW = SEG / WORDS;             // K per word: 8 (int4) / 4 (int8)
  const T* __restrict__ A = reinterpret_cast<const T*>(p.A);
  const T* __restrict__ S = reinterpret_cast<const T*>(p.scales);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, t = lane & 3;
  const int N = p.N, K = p.K, M = p.M;
  const size_t row_bytes = (size_t)K * BITS / 8;
  const int rowbase = blockIdx.x * (128 * RT) + warp * 16 * RT;
  const int kbeg = blockIdx.y * p.klen;
  const int kend = min(K, kbeg + p.klen);
  const int tok0 = blockIdx.z * 16;

  // row pointers (clamped for the ragged N tail; stores are masked)
  const uint8_t* wrow[RT][2];
#pragma unroll
  for (int r = 0; r < RT; ++r)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int n = min(rowbase + r * 16 + h * 8 + gq, N - 1);
      wrow[r][h] = p.codes + (size_t)n * row_bytes;
    }
  const T* arow[MT];
  bool tok_ok[MT];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int tok = tok0 + mt * 8 + gq;
    tok_ok[mt] = tok < M;
    arow[mt] = A + (size_t)min(tok, M - 1) * K;
  }

  float acc[RT][MT][4];
#pragma unroll
  for (int r = 0; r < RT; ++r)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[r][mt][i] = 0.f;

  auto load_w = [&](uint4 (&wr)[RT][2], int kc) {
    const int k = kc + t * SEG;
    const bool ok = k < kend;
#pragma unroll
    for (int r = 0; r < RT; ++r)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        wr[r][h] = ok ? ldg_stream(wrow[r][h] + (size_t)k * BITS / 8) : make_uint4(0, 0, 0, 0);
  };

  uint4 wcur[RT][2], wnxt[RT][2];
  load_w(wcur, kbeg);
  for (int kc = kbeg; kc < kend; kc += KCH) {
    if (kc + KCH < kend) load_w(wnxt, kc + KCH);
    const int k = kc + t * SEG;
    const bool kok = k < kend;
    // activation fragments for this thread's K segment: per word 2 regs (b0,b1) per step
    uint32_t bfr[MT][WORDS][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const bool ok = kok && tok_ok[mt];
      if (BITS == 4) {
#pragma unroll
        for (int w = 0; w < WORDS; ++w) {
          const uint4 r = ok ? ldg_keep(arow[mt] + k + w * 8) : make_uint4(0, 0, 0, 0);
          bfr[mt][w][0] = prmt(r.x, r.z, 0x5410u);  // (o0,o4)
          bfr[mt][w][1] = prmt(r.x, r.z, 0x7632u);  // (o1,o5)
          bfr[mt][w][2] = prmt(r.y, r.w, 0x5410u);  // (o2,o6)
          bfr[mt][w][3] = prmt(r.y, r.w, 0x7632u);  // (o3,o7)
        }
      } else {
#pragma unroll
        for (int w2 = 0; w2 < 2; ++w2) {
          const uint4 r = ok ? ldg_keep(arow[mt] + k + w2 * 8) : make_uint4(0, 0, 0, 0);
          bfr[mt][2 * w2][0] = r.x; bfr[mt][2 * w2][1] = r.y;
          bfr[mt][2 * w2 + 1][0] = r.z; bfr[mt][2 * w2 + 1][1] = r.w;
        }
      }
    }
    float part[RT][MT][4];
    if (SACC) {
#pragma unroll
      for (int r = 0; r < RT; ++r)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int i = 0; i < 4; ++i) part[r][mt][i] = 0.f;
    }
#pragma unroll
    for (int r = 0; r < RT; ++r) {
      const uint32_t wg[4] = {wcur[r][0].x, wcur[r][0].y, wcur[r][0].z, wcur[r][0].w};
      const uint32_t wh[4] = {wcur[r][1].x, wcur[r][1].y, wcur[r][1].z, wcur[r][1].w};
#pragma unroll
      for (int w = 0; w < WORDS; ++w) {
        uint32_t sg = 0, sh = 0;
        if (!SACC) {
          const int j = (k + w * KPW) / p.group;
          const int ng = min(rowbase + r * 16 + gq, N - 1), nh = min(ng + 8, N - 1);
          sg = splat_scale<T>(S, (size_t)j * N + ng);
          sh = splat_scale<T>(S, (size_t)j * N + nh);
        }
        if (BITS == 4) {
          uint32_t qg[4], qh[4];
          i4_pairs<T>(wg[w], qg);
          i4_pairs<T>(wh[w], qh);
          if (!SACC) {
#pragma unroll
            for (int i = 0; i < 4; ++i) { qg[i] = mul2<T>(qg[i], sg); qh[i] = mul2<T>(qh[i], sh); }
          }
#pragma unroll
          for (int pp = 0; pp < 2; ++pp) {
            const uint32_t a[4] = {qg[2 * pp], qh[2 * pp], qg[2 * pp + 1], qh[2 * pp + 1]};
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
              if (SACC)
                mma16816<T>(part[r][mt], a, bfr[mt][w][2 * pp], bfr[mt][w][2 * pp + 1], part[r][mt]);
              else
                mma16816<T>(acc[r][mt], a, bfr[mt][w][2 * pp], bfr[mt][w][2 * pp + 1], acc[r][mt]);
            }
          }
        } else {
          uint32_t qg[2], qh[2];
          i8_pairs<T>(wg[w], qg);
          i8_pairs<T>(wh[w], qh);
          if (!SACC) {
#pragma unroll
            for (int i = 0; i < 2; ++i) { qg[i] = mul2<T>(qg[i], sg); qh[i] = mul2<T>(qh[i], sh); }
          }
          const uint32_t a[4] = {qg[0], qh[0], qg[1], qh[1]};
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            if (SACC)
              mma16816<T>(part[r][mt], a, bfr[mt][w][0], bfr[mt][w][1], part[r][mt]);
            else
              mma16816<T>(acc[r][mt], a, bfr[mt][w][0], bfr[mt][w][1], acc[r][mt]);
          }
        }
      }
    }
    if (SACC) {
      const int j = kc / p.group;
#pragma unroll
      for (int r = 0; r < RT; ++r) {
        const int ng = min(rowbase + r * 16 + gq, N - 1), nh = min(ng + 8, N - 1);
        const float s_g = load_scale_f<T>(S, (size_t)j * N + ng);
        const float s_h = load_scale_f<T>(S, (size_t)j * N + nh);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          acc[r][mt][0] = fmaf(s_g, part[r][mt][0], acc[r][mt][0]);
          acc[r][mt][1] = fmaf(s_g, part[r][mt][1], acc[r][mt][1]);
          acc[r][mt][2] = fmaf(s_h, part[r][mt][2], acc[r][mt][2]);
          acc[r][mt][3] = fmaf(s_h, part[r][mt][3], acc[r][mt][3]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < RT; ++r)
#pragma unroll
      for (int h = 0; h < 2; ++h) wcur[r][h] = wnxt[r][h];
  }

  // ---------------------------------------------------------------- epilogue (+ fused A5 fixup)
  auto store_out = [&](int tok, int n, float v) {
    const size_t o = (size_t)tok * N + n;
    if (p.cdt == FQ_FP32) reinterpret_cast<float*>(p.C)[o] = v;
    else reinterpret_cast<T*>(p.C)[o] = Dt<T>::from_f(v);
  };
  const int S_ = gridDim.y;
  if (S_ == 1) {
#pragma unroll
    for (int r = 0; r < RT; ++r)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int n = rowbase + r * 16 + gq + (i >> 1) * 8;
          const int tok = tok0 + mt * 8 + 2 * t + (i & 1);
          if (n < N && tok < M) store_out(tok, n, acc[r][mt][i]);
        }
    return;
  }
  float* part_out = p.ws + (size_t)blockIdx.y * M * N;
#pragma unroll
  for (int r = 0; r < RT; ++r)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int n = rowbase + r * 16 + gq + (i >> 1) * 8;
        const int tok = tok0 + mt * 8 + 2 * t + (i & 1);
        if (n < N && tok < M) __stcg(part_out + (size_t)tok * N + n, acc[r][mt][i]);
      }
  __threadfence();
  __shared__ int s_last;
  __syncthreads();
  int* ctr = p.counters + blockIdx.z * gridDim.x + blockIdx.x;
  if (threadIdx.x == 0) {
    const int prev = atomicAdd(ctr, 1);
    s_last = (prev == S_ - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
#pragma unroll
  for (int r = 0; r < RT; ++r)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int n = rowbase + r * 16 + gq + (i >> 1) * 8;
        const int tok = tok0 + mt * 8 + 2 * t + (i & 1);
        if (n < N && tok < M) {
          float v = 0.f;
          for (int s = 0; s < S_; ++s) v += __ldcg(p.ws + ((size_t)s * M + tok) * N + n);
          store_out(tok, n, v);
        }
      }
  if (threadIdx.x == 0) *ctr = 0;  // self-reset for the next call / graph replay
}

// ------------------------------------------------------------------------------------- host side
static int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

GemvPlan plan_gemv(int M, int K, int N, int bits, int group, int nsm) {
  GemvPlan p{};
  p.kchunk = bits == 4 ? 128 : 64;
  p.mt = M <= 8 ? 1 : 2;
  p.ktiles = (M + 15) / 16;
  p.rt = env_int("FQ_GEMV_RT", N >= 128 * 2 * 64 ? 2 : 1);
  if (p.rt != 1 && p.rt != 2) p.rt = 2;
  p.rows_per_cta = 128 * p.rt;
  const int gx = (N + p.rows_per_cta - 1) / p.rows_per_cta;
  const int nchunks = (K + p.kchunk - 1) / p.kchunk;
  const int slots = 2 * nsm;  // 2 CTAs per SM (launch bounds)
  int best_s = 1;
  double best = -1.0;
  const int smax = std::min(nchunks, 64);
  for (int s = 1; s <= smax; ++s) {
    const int klen = ((nchunks + s - 1) / s) * p.kchunk;
    const int s_eff = (K + klen - 1) / klen;
    if (s_eff != s) continue;
    const double ctas = (double)gx * s * p.ktiles;
    const double waves = ctas / slots;
    const double eff = waves / std::ceil(waves);
    // prefer full waves; among near-equal efficiencies prefer fewer splits (partial traffic)
    const double score = eff - 0.004 * s - (waves < 0.9 ? 1.0 : 0.0) * (1.0 - waves);
    if (score > best + 1e-9) { best = score; best_s = s; }
  }
  int s = env_int("FQ_GEMV_SPLITS", best_s);
  s = std::max(1, std::min(s, nchunks));
  p.klen = ((nchunks + s - 1) / s) * p.kchunk;
  p.splits = (K + p.klen - 1) / p.klen;
  return p;
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

size_t gemv_workspace_bytes(const GemvPlan& p, int M, int N) {
  if (p.splits <= 1) return 256;
  const int gx = (N + p.rows_per_cta - 1) / p.rows_per_cta;
  return align256((size_t)p.splits * M * N * sizeof(float)) + align256((size_t)gx * p.ktiles * sizeof(int));
}

template <typename T, int BITS, int MT, bool SACC, int RT>
static cudaError_t launch_gemv(const GemvPlan& pl, const GemvParams& prm, cudaStream_t st) {
  const int gx = (prm.N + pl.rows_per_cta - 1) / pl.rows_per_cta;
  dim3 grid(gx, pl.splits, pl.ktiles);
  gemv_kernel<T, BITS, MT, SACC, RT><<<grid, kGemvThreads, 0, st>>>(prm);
  return cudaGetLastError();
}

template <typename T, int BITS, int MT, bool SACC>
static cudaError_t dispatch_rt(const GemvPlan& pl, const GemvParams& prm, cudaStream_t st) {
  return pl.rt == 1 ? launch_gemv<T, BITS, MT, SACC, 1>(pl, prm, st)
                    : launch_gemv<T, BITS, MT, SACC, 2>(pl, prm, st);
}
template <typename T, int BITS, int MT>
static cudaError_t dispatch_sacc(bool sacc, const GemvPlan& pl, const GemvParams& prm, cudaStream_t st) {
  return sacc ? dispatch_rt<T, BITS, MT, true>(pl, prm, st) : dispatch_rt<T, BITS, MT, false>(pl, prm, st);
}
template <typename T, int BITS>
static cudaError_t dispatch_mt(bool sacc, const GemvPlan& pl, const GemvParams& prm, cudaStream_t st) {
  return pl.mt == 1 ? dispatch_sacc<T, BITS, 1>(sacc, pl, prm, st) : dispatch_sacc<T, BITS, 2>(sacc, pl, prm, st);
}
template <typename T>
static cudaError_t dispatch_bits(int bits, bool sacc, const GemvPlan& pl, const GemvParams& prm,
                                 cudaStream_t st) {
  return bits == 4 ? dispatch_mt<T, 4>(sacc, pl, prm, st) : dispatch_mt<T, 8>(sacc, pl, prm, st);
}

cudaError_t run_gemv(const GemvPlan& pl, int adt, int cdt, int bits, const void* A, int M, int K,
                     int N, const void* codes, const void* scales, int group, void* C, void* ws,
                     cudaStream_t st) {
  GemvParams prm{};
  prm.A = A;
  prm.codes = reinterpret_cast<const uint8_t*>(codes);
  prm.scales = scales;
  prm.C = C;
  prm.M = M; prm.K = K; prm.N = N; prm.group = group; prm.cdt = cdt;
  prm.klen = pl.klen;
  prm.ws = reinterpret_cast<float*>(ws);
  const size_t part = align256((size_t)pl.splits * M * N * sizeof(float));
  prm.counters = reinterpret_cast<int*>(reinterpret_cast<char*>(ws) + (pl.splits > 1 ? part : 0));
  const bool sacc = (group % pl.kchunk) == 0;
  return adt == FQ_BF16 ? dispatch_bits<__nv_bfloat16>(bits, sacc, pl, prm, st)
                        : dispatch_bits<__half>(bits, sacc, pl, prm, st);
}

}  // namespace fq
