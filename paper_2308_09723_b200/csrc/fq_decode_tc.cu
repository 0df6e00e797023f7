// fq_decode_tc.cu — kernel A4 on the 5th-gen tensor cores: the decode (M <= 16) fused dequant GEMM
// with the MMA issued by tcgen05 instead of the legacy warp-level mma.sync (whose B200 throughput,
// ~0.45 HMMA/clk/SM measured, made it a bottleneck; profiles/r01).
//
// C[m,n] = sum_k A[m,k] * q[n,k] * s[k/g, n]   (§4.1), requires group % KS == 0
// (KS = 128 for int4, 64 for int8: one scale per row per K chunk; other groups use the mma.sync
// kernel in fq_gemv.cu).  Decode streams every packed weight byte once.
//
// CTA = 128 weight rows (the UMMA M, TMEM lanes) x 16 tokens (UMMA N) x a K range; warps:
//   0      TMA: per stage packed codes [128 rows x 64 B] (SWIZZLE_64B) + raw activations
//          [16 tokens x KS] + the 128-column scale row; 6-stage shared-memory ring.
//   1      TMEM allocation + single-thread tcgen05.mma (kind::f16, A = weights in TMEM,
//          B = activations in smem, D = one of 4 fp32 accumulator slices of 16 columns).
//   2      activation stager: raw -> UMMA B tile (SWIZZLE_128B K-major) in the same per-word
//          (0,4),(1,5),(2,6),(3,7) k-order the int4 unpack produces, + per-token sums.
//   3..6   dequant: thread = one weight row; LOP3 magic unpack to bf16x2 (codes + offset),
//          tcgen05.st into a 3-deep TMEM A ring.
//   7..10  fold: per chunk, tcgen05.ld the accumulator slice (16 tokens), remove the code offset
//          (offset * token sums), scale by s[j, n] in fp32, accumulate in registers; epilogue
//          writes C (or split-K partials; the last CTA of a column tile reduces them in order).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "fq_common.cuh"
#include "fq_internal.h"
#include "fq_tcgen05.cuh"

namespace fq {
namespace dtc {
using namespace tc5;

constexpr int ROWS = 128;
constexpr int NT = 16;
#ifndef FQ_DTC_CTAS
#define FQ_DTC_CTAS 2
#endif
constexpr int CTAS_PER_SM = FQ_DTC_CTAS;
constexpr int SSTAGES = CTAS_PER_SM == 1 ? 12 : 6;
constexpr int ASTAGES = CTAS_PER_SM == 1 ? 6 : 3;
constexpr int ACC = CTAS_PER_SM == 1 ? 8 : 4;
constexpr int kThreads = 32 * 11;
constexpr int kTmemCols = CTAS_PER_SM == 1 ? 512 : 256;

template <int BITS>
struct G {
  static constexpr int WB = 64;                    // packed bytes per row per stage
  static constexpr int KS = WB * 8 / BITS;         // K per stage (= one scale chunk): 128 / 64
  static constexpr int W_BYTES = ROWS * WB;        // 8 KB
  static constexpr int B_BYTES = NT * KS * 2;      // 4 KB / 2 KB (KS/64 SW128 atoms of 16 rows)
  static constexpr int B_OFS = W_BYTES;            // 1024-aligned
  static constexpr int RAW_OFS = B_OFS + B_BYTES;
  static constexpr int RAW_BYTES = NT * KS * 2;
  static constexpr int SC_OFS = RAW_OFS + RAW_BYTES;
  static constexpr int SC_BYTES = ROWS * 2;
  static constexpr int SA_OFS = SC_OFS + SC_BYTES;
  static constexpr int SA_BYTES = NT * 4;
  static constexpr int SF_OFS = SA_OFS + SA_BYTES;  // scales as fp32 (written by the stager)
  static constexpr int SF_BYTES = ROWS * 4;
  static constexpr int STAGE = ((SF_OFS + SF_BYTES + 1023) / 1024) * 1024;
  static constexpr int SMEM = SSTAGES * STAGE + 1024;
  static constexpr int A_COLS = KS / 2;            // TMEM columns per A stage
  static constexpr int ACC_COL = ASTAGES * A_COLS; // accumulator slices after the A ring
};

struct DtcProb {
  CUtensorMap w, a, s;
  void* C;
  float* ws;
  int* counters;
  int M, K, N, group, klen, cdt;
  int gx, splits, cta_begin;
  int dbg_nofence;  // diagnostics only (FQ_DTC_NOFENCE): skip the proxy fence
  int dbg;          // diagnostics only (FQ_DTC_DBG bits): 1 dequant, 2 fold, 4 stager, 8 mma skipped
};
template <int MAXP>
struct DtcBatch {
  DtcProb p[MAXP];
  int nprob;
};

template <typename T, int BITS>
__device__ __forceinline__ void unpack_word(uint32_t w, uint32_t* q);
template <>
__device__ __forceinline__ void unpack_word<__nv_bfloat16, 4>(uint32_t w, uint32_t* q) {
  // pairs (k,k+4),(k+1,k+5),(k+2,k+6),(k+3,k+7) as bf16 (128 + (n ^ 8)) = code + 136
  q[0] = lop3_and_xor(w, 0x000F000Fu, 0x43084308u);
  q[1] = lop3_and_xor(__umulhi(w, 1u << 28), 0x000F000Fu, 0x43084308u);
  q[2] = lop3_and_xor(w >> 8, 0x000F000Fu, 0x43084308u);
  q[3] = lop3_and_xor(__umulhi(w, 1u << 20), 0x000F000Fu, 0x43084308u);
}
template <>
__device__ __forceinline__ void unpack_word<__half, 4>(uint32_t w, uint32_t* q) {
  q[0] = lop3_and_xor(w, 0x000F000Fu, 0x64086408u);  // fp16 1024 + (n ^ 8) = code + 1032
  q[1] = lop3_and_xor(__umulhi(w, 1u << 28), 0x000F000Fu, 0x64086408u);
  q[2] = lop3_and_xor(w >> 8, 0x000F000Fu, 0x64086408u);
  q[3] = lop3_and_xor(__umulhi(w, 1u << 20), 0x000F000Fu, 0x64086408u);
}
template <>
__device__ __forceinline__ void unpack_word<__half, 8>(uint32_t w, uint32_t* q) {
  const uint32_t u = w ^ 0x80808080u;  // natural pairs, fp16 1024 + (q + 128) = code + 1152
  q[0] = prmt(u, 0x64646464u, 0x4140u);
  q[1] = prmt(u, 0x64646464u, 0x4342u);
}
template <>
__device__ __forceinline__ void unpack_word<__nv_bfloat16, 8>(uint32_t w, uint32_t* q) {
  const uint32_t u = w ^ 0x80808080u;  // natural pairs, exact codes (offset removed in fp32)
  float f[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) f[i] = __uint_as_float(prmt(u, 0x4B000000u, 0x7440u + i)) - 8388736.0f;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(q[0]) : "f"(f[1]), "f"(f[0]));
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(q[1]) : "f"(f[3]), "f"(f[2]));
}
template <typename T, int BITS> struct Off { static constexpr float v = 0.f; };
template <> struct Off<__nv_bfloat16, 4> { static constexpr float v = 136.f; };
template <> struct Off<__half, 4> { static constexpr float v = 1032.f; };
template <> struct Off<__half, 8> { static constexpr float v = 1152.f; };

template <typename T, int BITS, int MAXP, int NTF>
__global__ void __launch_bounds__(kThreads, CTAS_PER_SM) decode_tc_kernel(const __grid_constant__ DtcBatch<MAXP> batch) {
  // NTF: tokens folded per chunk (compile-time bucket >= M; rows beyond M are zero)
  using Gm = G<BITS>;
  constexpr int KS = Gm::KS;
  constexpr float OFF = Off<T, BITS>::v;
  extern __shared__ __align__(1024) uint8_t dsmem[];
  __shared__ __align__(8) uint64_t full_bar[SSTAGES], bready[SSTAGES], sfree[SSTAGES];
  __shared__ __align__(8) uint64_t aready[ASTAGES], afree[ASTAGES];
  __shared__ __align__(8) uint64_t accfull[ACC], accfree[ACC];
  __shared__ uint32_t tmem_base_sh;
  __shared__ int s_last;
  uint8_t* sbase = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsmem) + 1023) & ~uintptr_t(1023));
  const uint32_t sb = smem_u32(sbase);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  int pi = 0;
  while (pi + 1 < batch.nprob && (int)blockIdx.x >= batch.p[pi + 1].cta_begin) ++pi;
  const DtcProb& p = batch.p[pi];
  const int local = (int)blockIdx.x - p.cta_begin;
  const int bx = local % p.gx, by = local / p.gx;
  const int N = p.N, K = p.K, M = p.M;
  const int n0 = bx * ROWS;
  const int kbeg = by * p.klen;
  const int kend = min(K, kbeg + p.klen);
  const int nst = (kend - kbeg + KS - 1) / KS;
  const int mloc = min(M, NT);

  if (threadIdx.x == 0) {
    for (int s = 0; s < SSTAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&bready[s], 32);
      mbar_init(&sfree[s], 4);   // one arrival per fold warp
    }
    for (int a = 0; a < ASTAGES; ++a) {
      mbar_init(&aready[a], 4);  // one arrival per dequant warp
      mbar_init(&afree[a], 1);
    }
    for (int c = 0; c < ACC; ++c) {
      mbar_init(&accfull[c], 1);
      mbar_init(&accfree[c], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&tmem_base_sh, kTmemCols);
  if (warp == 2) {
    // zero the B tiles once: token rows >= M stay zero for the whole kernel
    for (int s = 0; s < SSTAGES; ++s)
      for (int o = lane * 16; o < Gm::B_BYTES; o += 512) sts128(sb + s * Gm::STAGE + Gm::B_OFS + o, make_uint4(0, 0, 0, 0));
    for (int s = 0; s < SSTAGES; ++s)
      if (lane < NT) reinterpret_cast<float*>(sbase + s * Gm::STAGE + Gm::SA_OFS)[lane] = 0.f;
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.w);
    prefetch_tmap(&p.a);
    prefetch_tmap(&p.s);
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tmem_base_sh;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t polw = policy_evict_first();
      const uint64_t pola = policy_evict_last();
      const int gm = p.group / KS;  // chunks per scale group
      int grem = (kbeg / KS) % gm, gj = (kbeg / KS) / gm;
      int s = 0;
      uint32_t ph = 0;
      for (int i = 0; i < nst; ++i) {
        mbar_wait(&sfree[s], ph ^ 1);
        uint8_t* st = sbase + s * Gm::STAGE;
        const int k0 = kbeg + i * KS;
        mbar_arrive_expect_tx(&full_bar[s], Gm::W_BYTES + Gm::RAW_BYTES + Gm::SC_BYTES);
        tma_load_2d(st, &p.w, &full_bar[s], k0 * BITS / 8, n0, polw);
        tma_load_2d(st + Gm::RAW_OFS, &p.a, &full_bar[s], k0, 0, pola);
        tma_load_2d(st + Gm::SC_OFS, &p.s, &full_bar[s], n0, gj, polw);
        if (++grem == gm) { grem = 0; ++gj; }
        if (++s == SSTAGES) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_f16<T, ROWS, NT>();
      int s = 0, a = 0, c = 0;
      uint32_t ph = 0, aph = 0, cph = 0;
      for (int i = 0; i < nst; ++i) {
        mbar_wait(&bready[s], ph);
        mbar_wait(&aready[a], aph);
        mbar_wait(&accfree[c], cph ^ 1);
        fence_after();
        const uint64_t bdesc = sw128_desc(sb + s * Gm::STAGE + Gm::B_OFS);
#pragma unroll
        for (int kk = 0; kk < ((p.dbg & 8) ? 1 : KS / 16); ++kk)
          mma_ts(tmem + Gm::ACC_COL + c * NT, tmem + a * Gm::A_COLS + kk * 8,
                 bdesc + (uint64_t)((((kk >> 2) * 2048) + (kk & 3) * 32) >> 4), idesc, kk != 0);
        mma_commit(&afree[a]);
        mma_commit(&accfull[c]);
        if (++s == SSTAGES) { s = 0; ph ^= 1; }
        if (++a == ASTAGES) { a = 0; aph ^= 1; }
        if (++c == ACC) { c = 0; cph ^= 1; }
      }
    }
  } else if (warp == 2) {
    // ------------------------------------------------------------------ activation stager
    // raw [16 tokens][KS] natural order -> B tile: element (tok, k) in SW128 K-major atoms of 64 k
    constexpr int PPT = KS / 8;                    // 8-element pieces per token
    constexpr int NPW = NT * PPT / 32;             // pieces per lane per stage
    constexpr int PPC = PPT;                       // one chunk per stage: a token's pieces
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < nst; ++i) {
      mbar_wait(&full_bar[s], ph);
      const uint32_t st = sb + s * Gm::STAGE;
#pragma unroll
      for (int j = 0; j < ((p.dbg & 4) ? 0 : NPW); ++j) {
        if ((32 * j) / PPT >= mloc) continue;      // warp-uniform: all-zero token group
        const int pc = lane + 32 * j;
        const int tok = pc / PPT, kl = (pc % PPT) * 8;
        uint4 v = lds128(st + Gm::RAW_OFS + pc * 16);
        if (OFF != 0.f) {
          float sum = 0.f;
          const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (Dt<T>::id == FQ_BF16) {
              sum += __uint_as_float(vv[e] << 16) + __uint_as_float(vv[e] & 0xFFFF0000u);
            } else {
              const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&vv[e]));
              sum += f.x + f.y;
            }
          }
#pragma unroll
          for (int o = PPC / 2; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
          if ((lane % PPC) == 0) reinterpret_cast<float*>(sbase + s * Gm::STAGE + Gm::SA_OFS)[tok] = sum;
        }
        if (BITS == 4)
          v = make_uint4(prmt(v.x, v.z, 0x5410u), prmt(v.x, v.z, 0x7632u), prmt(v.y, v.w, 0x5410u),
                         prmt(v.y, v.w, 0x7632u));
        const int atom = kl >> 6, chunk = (kl & 63) >> 3;
        sts128(st + Gm::B_OFS + atom * 2048 + tok * 128 + ((chunk ^ (tok & 7)) << 4), v);
      }
      {  // the stage's 128 scales -> fp32 for the fold warps
        const uint2 sv = lds64(st + Gm::SC_OFS + lane * 8);
        const uint32_t h[4] = {sv.x & 0xFFFFu, sv.x >> 16, sv.y & 0xFFFFu, sv.y >> 16};
        float f[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const unsigned short hv = (unsigned short)h[e];
          f[e] = Dt<T>::to_f(*reinterpret_cast<const T*>(&hv));
        }
        sts128(st + Gm::SF_OFS + lane * 16, make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]),
                                                       __float_as_uint(f[2]), __float_as_uint(f[3])));
      }
      if (!p.dbg_nofence) fence_proxy_async_smem();  // generic-proxy stores -> visible to the tensor core
      mbar_arrive(&bready[s]);
      if (++s == SSTAGES) { s = 0; ph ^= 1; }
    }
  } else if (warp < 7) {
    // ------------------------------------------------------------------ dequant -> TMEM
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    int s = 0, a = 0;
    uint32_t ph = 0, aph = 0;
    for (int i = 0; i < nst; ++i) {
      mbar_wait(&full_bar[s], ph);
      const uint32_t wrow = sb + s * Gm::STAGE + row * Gm::WB;
      uint4 c[4];
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) c[cc] = lds128(wrow + ((cc ^ ((row >> 1) & 3)) << 4));
      mbar_wait(&afree[a], aph ^ 1);
      fence_after();
      const uint32_t words[16] = {c[0].x, c[0].y, c[0].z, c[0].w, c[1].x, c[1].y, c[1].z, c[1].w,
                                  c[2].x, c[2].y, c[2].z, c[2].w, c[3].x, c[3].y, c[3].z, c[3].w};
      constexpr int PAIRS_PER_WORD = BITS == 4 ? 4 : 2;
      constexpr int NPAIR = 16 * PAIRS_PER_WORD;  // 64 (int4) / 32 (int8) TMEM columns
#pragma unroll
      for (int half = 0; half < NPAIR / 32; ++half) {
        uint32_t q[32];
#pragma unroll
        for (int w = 0; w < 32 / PAIRS_PER_WORD; ++w)
          if (p.dbg & 1) { for (int u = 0; u < PAIRS_PER_WORD; ++u) q[w * PAIRS_PER_WORD + u] = words[half * (32 / PAIRS_PER_WORD) + w]; }
          else unpack_word<T, BITS>(words[half * (32 / PAIRS_PER_WORD) + w], &q[w * PAIRS_PER_WORD]);
        tmem_st32(tmem + lane_base + a * Gm::A_COLS + half * 32, q);
      }
      tmem_wait_st();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&aready[a]);
      if (++s == SSTAGES) { s = 0; ph ^= 1; }
      if (++a == ASTAGES) { a = 0; aph ^= 1; }
    }
  } else {
    // ------------------------------------------------------------------ fold + epilogue
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    float acc[NTF];
#pragma unroll
    for (int t = 0; t < NTF; ++t) acc[t] = 0.f;
    int s = 0, c = 0;
    uint32_t ph = 0, cph = 0;
    for (int i = 0; i < nst; ++i) {
      mbar_wait(&accfull[c], cph);
      fence_after();
      uint32_t v[16];
      tmem_ld16(tmem + lane_base + Gm::ACC_COL + c * NT, v);
      tmem_wait_ld();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&accfree[c]);
      mbar_wait(&bready[s], ph);  // direct acquire of the stager's fp32 scales and token sums
      const uint32_t st = sb + s * Gm::STAGE;
      const float sc = lds_f32(st + Gm::SF_OFS + row * 4);
#pragma unroll
      if (!(p.dbg & 2))
#pragma unroll
      for (int t = 0; t < NTF; ++t) {
        float part = __uint_as_float(v[t]);
        if (OFF != 0.f) part = fmaf(-OFF, lds_f32(st + Gm::SA_OFS + t * 4), part);
        acc[t] = fmaf(sc, part, acc[t]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sfree[s]);  // scales + token sums consumed: refill allowed
      if (++s == SSTAGES) { s = 0; ph ^= 1; }
      if (++c == ACC) { c = 0; cph ^= 1; }
    }
    // ---- epilogue (+ fused deterministic split-K reduction)
    const int n = n0 + row;
    auto store_out = [&](int tok, float val) {
      const size_t o = (size_t)tok * N + n;
      if (p.cdt == FQ_FP32) reinterpret_cast<float*>(p.C)[o] = val;
      else reinterpret_cast<T*>(p.C)[o] = Dt<T>::from_f(val);
    };
    if (p.splits == 1) {
      if (n < N) {
#pragma unroll
        for (int t = 0; t < NTF; ++t)
          if (t < mloc) store_out(t, acc[t]);
      }
    } else {
      float* part_out = p.ws + (size_t)by * M * N;
      if (n < N) {
#pragma unroll
        for (int t = 0; t < NTF; ++t)
          if (t < mloc) __stcg(part_out + (size_t)t * N + n, acc[t]);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      int* ctr = p.counters + bx;
      if (threadIdx.x == 7 * 32) {
        int prev;
        asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], 1;" : "=r"(prev) : "l"(ctr) : "memory");
        s_last = (prev == p.splits - 1);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (s_last) {
        __threadfence();
        if (n < N) {
#pragma unroll
          for (int t = 0; t < NTF; ++t) {
            if (t < mloc) {
              float val = 0.f;
              for (int sp = 0; sp < p.splits; ++sp) val += __ldcg(p.ws + ((size_t)sp * M + t) * N + n);
              store_out(t, val);
            }
          }
        }
        if (threadIdx.x == 7 * 32) *ctr = 0;  // self-reset
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

}  // namespace dtc

// ------------------------------------------------------------------------------------- host side
bool decode_tc_supported(int bits, int group, int M) {
  // Opt-in (FQ_DECODE_TC=1): correct, but its 8 KB-stage pipeline skeleton streams at only
  // ~3.6 TB/s even with all compute removed (round-1 diagnostics, profiles/r01), so the mma.sync
  // decode kernel (16 KB stages, 5.7 TB/s skeleton) remains the default A4.
  const char* e = std::getenv("FQ_DECODE_TC");
  if (!e || e[0] != '1') return false;
  return M >= 1 && M <= dtc::NT && group % (bits == 4 ? 128 : 64) == 0;
}

template <typename T, int BITS, int MAXP, int NTF>
static cudaError_t launch_dtc(const dtc::DtcBatch<MAXP>& b, int ctas, cudaStream_t st) {
  constexpr int smem = dtc::G<BITS>::SMEM;
  auto kern = dtc::decode_tc_kernel<T, BITS, MAXP, NTF>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  kern<<<ctas, dtc::kThreads, smem, st>>>(b);
  return cudaGetLastError();
}

template <int MAXP, int NTF>
static cudaError_t dispatch_dtc_t(int adt, int bits, const dtc::DtcBatch<MAXP>& b, int ctas, cudaStream_t st) {
  if (adt == FQ_BF16)
    return bits == 4 ? launch_dtc<__nv_bfloat16, 4, MAXP, NTF>(b, ctas, st)
                     : launch_dtc<__nv_bfloat16, 8, MAXP, NTF>(b, ctas, st);
  return bits == 4 ? launch_dtc<__half, 4, MAXP, NTF>(b, ctas, st) : launch_dtc<__half, 8, MAXP, NTF>(b, ctas, st);
}
template <int MAXP>
static cudaError_t dispatch_dtc(int adt, int bits, const dtc::DtcBatch<MAXP>& b, int ctas, cudaStream_t st,
                                int maxm) {
  if (maxm <= 1) return dispatch_dtc_t<MAXP, 1>(adt, bits, b, ctas, st);
  if (maxm <= 4) return dispatch_dtc_t<MAXP, 4>(adt, bits, b, ctas, st);
  return dispatch_dtc_t<MAXP, 16>(adt, bits, b, ctas, st);
}

static bool make_dtc_prob(dtc::DtcProb& d, int splits, int klen, int bits, int cdt, const void* A, int M, int K,
                          int N, const void* codes, const void* scales, int group, void* C, void* ws) {
  const uint64_t row_bytes = (uint64_t)K * bits / 8;
  const int ks = 64 * 8 / bits;
  if (!make_tmap_2d(&d.w, codes, 1, row_bytes, (uint64_t)N, row_bytes, 64, dtc::ROWS, 64)) return false;
  if (!make_tmap_2d(&d.a, A, 2, (uint64_t)K, (uint64_t)M, (uint64_t)K * 2, ks, dtc::NT, 0)) return false;
  if (!make_tmap_2d(&d.s, scales, 2, (uint64_t)N, (uint64_t)(K / group), (uint64_t)N * 2, dtc::ROWS, 1, 0))
    return false;
  d.C = C;
  d.M = M; d.K = K; d.N = N; d.group = group; d.cdt = cdt;
  d.klen = klen;
  d.splits = splits;
  d.gx = (N + dtc::ROWS - 1) / dtc::ROWS;
  d.counters = reinterpret_cast<int*>(ws);
  d.ws = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + 65536);
  const char* nf = std::getenv("FQ_DTC_NOFENCE");
  d.dbg_nofence = nf && nf[0] == '1';
  const char* db = std::getenv("FQ_DTC_DBG");
  d.dbg = db ? std::atoi(db) : 0;
  return true;
}

// Split-K plan for the tcgen05 decode kernel: fill 2 CTAs/SM with full waves.
void plan_dtc(int M, int K, int N, int bits, int nsm, int* splits, int* klen) {
  const int ks = 64 * 8 / bits;
  const int gx = (N + dtc::ROWS - 1) / dtc::ROWS;
  const int nchunks = (K + ks - 1) / ks;
  const int slots = dtc::CTAS_PER_SM * nsm;
  int best_s = 1;
  double best = -1e30;
  for (int s = 1; s <= std::min(nchunks, 32); ++s) {
    const int kl = ((nchunks + s - 1) / s) * ks;
    if ((K + kl - 1) / kl != s) continue;
    const double waves = (double)gx * s / slots;
    const double eff = waves / std::ceil(waves);
    const double score = eff + 0.02 * std::min(waves, 4.0) - 0.004 * s * (M > 4 ? 2 : 1);
    if (score > best + 1e-9) { best = score; best_s = s; }
  }
  const char* e = std::getenv("FQ_GEMV_SPLITS");
  int s = e ? std::max(1, std::min(std::atoi(e), nchunks)) : best_s;
  *klen = ((nchunks + s - 1) / s) * ks;
  *splits = (K + *klen - 1) / *klen;
}

size_t dtc_workspace_bytes(int M, int K, int N, int bits, int nsm) {
  int splits, klen;
  plan_dtc(M, K, N, bits, nsm, &splits, &klen);
  return 65536 + (splits > 1 ? (size_t)splits * M * N * sizeof(float) : 0);
}

cudaError_t run_decode_tc(int adt, int cdt, int bits, const void* A, int M, int K, int N, const void* codes,
                          const void* scales, int group, void* C, void* ws, cudaStream_t st) {
  int splits, klen;
  plan_dtc(M, K, N, bits, num_sms(), &splits, &klen);
  dtc::DtcBatch<1> b{};
  if (!make_dtc_prob(b.p[0], splits, klen, bits, cdt, A, M, K, N, codes, scales, group, C, ws))
    return cudaErrorInvalidValue;
  b.p[0].cta_begin = 0;
  b.nprob = 1;
  return dispatch_dtc<1>(adt, bits, b, b.p[0].gx * splits, st, M);
}

// MoE batch on the tcgen05 decode kernel: experts (1 <= M_e <= 16, group % KS == 0), one launch per
// <= 40 experts, no split-K (the batch fills the machine).
cudaError_t run_decode_tc_grouped(int adt, int cdt, int bits, const void* A, int K, int N, const int64_t* offsets,
                                  const int32_t* groups, const void* const* codes, const void* const* scales,
                                  void* C, const int* experts, int nexp, cudaStream_t st) {
  constexpr int MAXP = 40;
  static_assert(sizeof(dtc::DtcBatch<MAXP>) < 32000, "kernel parameter block limit");
  dtc::DtcBatch<MAXP> b{};
  int ctas = 0, maxm = 0;
  const int ks = 64 * 8 / bits;
  for (int ii = 0; ii < nexp; ++ii) {
    const int e = experts[ii];
    const int Me = (int)(offsets[e + 1] - offsets[e]);
    const char* Ae = reinterpret_cast<const char*>(A) + (size_t)offsets[e] * K * 2;
    char* Ce = reinterpret_cast<char*>(C) + (size_t)offsets[e] * N * (cdt == FQ_FP32 ? 4 : 2);
    dtc::DtcProb& d = b.p[b.nprob];
    if (!make_dtc_prob(d, 1, ((K + ks - 1) / ks) * ks, bits, cdt, Ae, Me, K, N, codes[e], scales[e], groups[e],
                       Ce, nullptr))
      return cudaErrorInvalidValue;
    d.cta_begin = ctas;
    ctas += d.gx;
    maxm = std::max(maxm, Me);
    if (++b.nprob == MAXP) {
      cudaError_t r = dispatch_dtc<MAXP>(adt, bits, b, ctas, st, maxm);
      if (r != cudaSuccess) return r;
      b.nprob = 0;
      ctas = 0;
      maxm = 0;
    }
  }
  if (b.nprob) return dispatch_dtc<MAXP>(adt, bits, b, ctas, st, maxm);
  return cudaSuccess;
}

}  // namespace fq
