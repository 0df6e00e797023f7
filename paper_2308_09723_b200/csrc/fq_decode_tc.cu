// fq_decode_tc.cu — kernel A4 on the 5th-gen tensor cores: the decode (M <= 16) fused dequant GEMM
// with the MMA issued by tcgen05 instead of the legacy warp-level mma.sync (whose issue slots and
// register-fragment traffic compete with the dequant ALU work on the same SM sub-partitions).
//
// C[m,n] = sum_k A[m,k] * q[n,k] * s[k/g, n]   (§4.1), requires group % KS == 0
// (KS = 128 for int4, 64 for int8: one scale per row per stage; other groups use the mma.sync
// kernel in fq_gemv.cu).  Decode streams every packed weight byte once, so the design goal
// is to keep >= 150 KB of weight loads in flight per SM and never let compute hold a stage.
//
// One persistent CTA per SM; the (tile, k-stage) space of all problems of the launch (one matrix,
// or every expert of a MoE batch) is split into equal contiguous stage ranges, one per CTA
// ("stream-K"): no wave quantisation, and the TMA runs ahead across tile boundaries.  Tiles cut by
// a range boundary are combined by the last-arriving contributor in CTA order (deterministic).
//
// Tile = 256 weight rows (two UMMA M=128 halves, TMEM lanes) x 16 tokens (UMMA N).  Warps:
//   0       TMA: per stage packed codes [256 rows x 64 B] (SWIZZLE_64B), raw activations
//           [M x KS], the stage's 256 scales; SSTAGES-deep ring.
//   1       TMEM allocation + single-thread tcgen05.mma (kind::f16, A = dequantized weights in
//           TMEM, B = activations in shared memory (SWIZZLE_128B K-major), D = accumulator slice).
//   2       stager: raw activations -> UMMA B tile in the per-word (0,4),(1,5),(2,6),(3,7) k-order
//           the int4 unpack produces; per-token sums (code-offset correction) and the fp32 scales
//           -> a fold-data ring.  Releases the smem stage as soon as it has read it.
//   3..10   dequant: thread = one weight row; LOP3 magic unpack (codes + offset) -> tcgen05.st into
//           a TMEM A ring.  Releases the smem stage right after its shared-memory loads.
//   11..18  fold: per stage tcgen05.ld of the accumulator (NTF token columns), remove the offset,
//           scale in fp32, accumulate in registers; per tile segment the epilogue writes C or a
//           split partial.
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "fq_common.cuh"
#include "fq_internal.h"
#include "fq_tcgen05.cuh"

namespace fq {
namespace dtc {
using namespace tc5;

constexpr int ROWS = 256;   // weight rows per tile (2 x UMMA M=128)
constexpr int NT = 16;      // UMMA N (tokens); M <= 16
constexpr int NB = 4;       // B-tile ring
constexpr int ACC = 4;      // accumulator ring (TMEM)
constexpr int FD = NB + ACC;  // fold-data ring (token sums + scales)
constexpr int kThreads = 32 * 19;
constexpr int kTmemCols = 512;
constexpr int kSmemBudget = 232448 - 1024 - 1024;  // 227 KB opt-in minus alignment slack + statics

template <int BITS>
struct G {
  static constexpr int WB = 64;                          // packed bytes per row per stage
  static constexpr int KS = WB * 8 / BITS;               // K per stage (= one scale chunk): 128 / 64
  static constexpr int W_BYTES = ROWS * WB;              // 16 KB
  static constexpr int RAW_OFS = W_BYTES;
  static constexpr int RAW_BYTES = NT * KS * 2;          // up to 16 token rows
  static constexpr int SC_OFS = RAW_OFS + RAW_BYTES;
  static constexpr int SC_BYTES = ROWS * 2;
  static constexpr int STAGE = ((SC_OFS + SC_BYTES + 1023) / 1024) * 1024;
  static constexpr int B_BYTES = NT * KS * 2;            // KS/64 SW128 atoms of 16 rows x 128 B
  static constexpr int FD_BYTES = (NT + ROWS) * 4;       // token sums + fp32 scales
  static constexpr int SSTAGES = (kSmemBudget - NB * B_BYTES - FD * FD_BYTES) / STAGE;
  static constexpr int B_RING = SSTAGES * STAGE;         // 1024-aligned
  static constexpr int FD_RING = B_RING + NB * B_BYTES;
  static constexpr int SMEM = FD_RING + FD * FD_BYTES + 1024;
  static constexpr int A_COLS = KS / 2;                  // TMEM columns per half per A slot
  static constexpr int ASTAGES = (kTmemCols - ACC * 2 * NT) / KS > 4 ? 4 : (kTmemCols - ACC * 2 * NT) / KS;
  static constexpr int ACC_COL = ASTAGES * KS;           // accumulator slices after the A ring
  static_assert(SSTAGES >= 4 && ACC_COL + ACC * 2 * NT <= kTmemCols, "resources");
};

struct DtcProb {
  CUtensorMap w, a, s;
  void* C;
  int M, K, N, group, cdt;
  int gx, nk;                    // tiles, stages per tile
  int stage_begin, tile_begin;   // offsets in the launch's linear stage / tile space
};
template <int MAXP>
struct DtcBatch {
  DtcProb p[MAXP];
  int nprob;
  int total_stages;
  float* ws;      // split partials [ctas][2][NT][ROWS]
  int* counters;  // per global tile (self-resetting)
  int dbg;        // diagnostics only (FQ_DTC_DBG bits): 1 dequant, 2 fold, 4 stager, 8 mma, 16 TMEM st, 32 all tensor-core work skipped
};

// Linear stage cursor over the launch's problems (all roles walk the same sequence).
struct Cur {
  int p, tile, kidx;
};
template <int MAXP>
__device__ __forceinline__ void cur_locate(const DtcBatch<MAXP>& b, int s, Cur& c) {
  int p = 0;
  while (p + 1 < b.nprob && s >= b.p[p + 1].stage_begin) ++p;
  const int local = s - b.p[p].stage_begin;
  c.p = p;
  c.tile = local / b.p[p].nk;
  c.kidx = local - c.tile * b.p[p].nk;
}
template <int MAXP>
__device__ __forceinline__ void cur_next(const DtcBatch<MAXP>& b, Cur& c) {
  if (++c.kidx == b.p[c.p].nk) {
    c.kidx = 0;
    if (++c.tile == b.p[c.p].gx) { c.tile = 0; ++c.p; }
  }
}
__device__ __forceinline__ int range_begin(int T, int P, int c) { return (int)((long long)T * c / P); }
__device__ __forceinline__ int cta_of(int T, int P, int x) {
  int c = (int)((long long)x * P / T);
  while (c + 1 < P && range_begin(T, P, c + 1) <= x) ++c;
  while (c > 0 && range_begin(T, P, c) > x) --c;
  return c;
}

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

// FQ_DTC_PROF (diagnostics build only): per-warp cycles spent in each barrier wait, printed by
// CTA 0 at exit.
#ifndef FQ_DTC_PROF
#define FQ_DTC_PROF 0
#endif
#if FQ_DTC_PROF
#define DTC_PW(k, stmt)                 \
  {                                     \
    const long long t0_ = clock64();    \
    stmt;                               \
    prof_[k] += clock64() - t0_;        \
  }
#else
#define DTC_PW(k, stmt) stmt;
#endif

template <typename T, int BITS, int MAXP, int NTF>
__global__ void __launch_bounds__(kThreads, 1) decode_tc_kernel(const __grid_constant__ DtcBatch<MAXP> batch) {
  // NTF: token columns folded per stage (compile-time bucket >= max M of the launch)
  using Gm = G<BITS>;
  constexpr int KS = Gm::KS, SST = Gm::SSTAGES, AST = Gm::ASTAGES;
  constexpr float OFF = Off<T, BITS>::v;
  extern __shared__ __align__(1024) uint8_t dsmem[];
  __shared__ __align__(8) uint64_t full_bar[SST], sfree[SST];
  __shared__ __align__(8) uint64_t bready[NB], bfree[NB];
  __shared__ __align__(8) uint64_t aready[AST], afree[AST];
  __shared__ __align__(8) uint64_t accfull[ACC], accfree[ACC];
  __shared__ __align__(8) uint64_t fdfree[FD];
  __shared__ uint32_t tmem_base_sh;
  __shared__ int s_last;
  uint8_t* sbase = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsmem) + 1023) & ~uintptr_t(1023));
  const uint32_t sb = smem_u32(sbase);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int P = gridDim.x, cta = blockIdx.x;
  const int TS = batch.total_stages;
  const int b0 = range_begin(TS, P, cta), b1 = range_begin(TS, P, cta + 1);
  const int nst = b1 - b0;
  const int dbg = batch.dbg;
#if FQ_DTC_PROF
  long long prof_[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  const long long tstart_ = clock64();
#endif

  if (threadIdx.x == 0) {
    for (int s = 0; s < SST; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&sfree[s], 1 + 8);  // stager + 8 dequant warps
    }
    for (int b = 0; b < NB; ++b) {
      mbar_init(&bready[b], 1);
      mbar_init(&bfree[b], 1);
    }
    for (int a = 0; a < AST; ++a) {
      mbar_init(&aready[a], 8);    // one arrival per dequant warp
      mbar_init(&afree[a], 1);
    }
    for (int c = 0; c < ACC; ++c) {
      mbar_init(&accfull[c], 2);   // tcgen05.commit + the MMA thread's release arrival
      mbar_init(&accfree[c], 8);   // one arrival per fold warp
    }
    for (int f = 0; f < FD; ++f) mbar_init(&fdfree[f], 8);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&tmem_base_sh, kTmemCols);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tmem_base_sh;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0 && nst > 0) {
      for (int q = 0; q < batch.nprob; ++q) {
        prefetch_tmap(&batch.p[q].w);
        prefetch_tmap(&batch.p[q].a);
        prefetch_tmap(&batch.p[q].s);
      }
      const uint64_t polw = policy_evict_first();
      const uint64_t pola = policy_evict_last();
      Cur cur;
      cur_locate(batch, b0, cur);
      int s = 0;
      uint32_t ph = 0;
      for (int i = 0; i < nst; ++i) {
        const DtcProb& p = batch.p[cur.p];
        DTC_PW(0, mbar_wait(&sfree[s], ph ^ 1))
        uint8_t* st = sbase + s * Gm::STAGE;
        const int k0 = cur.kidx * KS, n0 = cur.tile * ROWS;
        mbar_arrive_expect_tx(&full_bar[s], Gm::W_BYTES + p.M * KS * 2 + Gm::SC_BYTES);
        tma_load_2d(st, &p.w, &full_bar[s], k0 * BITS / 8, n0, polw);
        tma_load_2d(st + Gm::RAW_OFS, &p.a, &full_bar[s], k0, 0, pola);
        tma_load_2d(st + Gm::SC_OFS, &p.s, &full_bar[s], n0, k0 / p.group, polw);
        if (++s == SST) { s = 0; ph ^= 1; }
        cur_next(batch, cur);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer (whole warp,
    // one elected lane issues; operands are warp-uniform)
    constexpr uint32_t idesc = idesc_f16<T, 128, NT>();
    int b = 0, a = 0, c = 0;
    uint32_t bph = 0, aph = 0, cph = 0;
    for (int i = 0; i < nst; ++i) {
      DTC_PW(1, mbar_wait(&bready[b], bph))
      DTC_PW(2, mbar_wait(&aready[a], aph))
      DTC_PW(3, mbar_wait(&accfree[c], cph ^ 1))
      fence_after();
      if (dbg & 32) {  // diagnostics: no tensor-core work at all, plain arrivals
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&afree[a]);
          mbar_arrive(&bfree[b]);
          mbar_arrive(&accfull[c]);
        }
      } else {
        const uint64_t bdesc = sw128_desc(sb + Gm::B_RING + b * Gm::B_BYTES);
        const uint32_t dcol = tmem + Gm::ACC_COL + c * 2 * NT, acol = tmem + a * KS;
        if (dbg & 8) {
#pragma unroll
          for (int h = 0; h < 2; ++h) mma_ts_elect(dcol + h * NT, acol + h * Gm::A_COLS, bdesc, idesc, 0u);
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int kk = 0; kk < KS / 16; ++kk)
              mma_ts_elect(dcol + h * NT, acol + h * Gm::A_COLS + kk * 8,
                           bdesc + (uint64_t)((((kk >> 2) * 2048) + (kk & 3) * 32) >> 4), idesc, kk != 0);
        }
        mma_commit_elect(&afree[a]);
        mma_commit_elect(&bfree[b]);
        mma_commit_elect(&accfull[c]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&accfull[c]);  // release: orders the stager's fold data (acquired via bready)
      if (++b == NB) { b = 0; bph ^= 1; }
      if (++a == AST) { a = 0; aph ^= 1; }
      if (++c == ACC) { c = 0; cph ^= 1; }
    }
  } else if (warp == 2) {
    // ------------------------------------------------------------------ activation stager
    // raw [M tokens][KS] natural order -> B tile element (tok, k) in SW128 K-major atoms of 64 k
    constexpr int PPT = KS / 8;                    // 8-element pieces per token (one chunk)
    constexpr int NPW = NT * PPT / 32;             // pieces per lane per stage (all 16 tokens)
    Cur cur;
    cur_locate(batch, b0, cur);
    int s = 0, b = 0, f = 0;
    uint32_t ph = 0, bph = 0, fph = 0;
    for (int i = 0; i < nst; ++i) {
      const int mloc = batch.p[cur.p].M;
      DTC_PW(4, mbar_wait(&full_bar[s], ph))
      const uint32_t st = sb + s * Gm::STAGE;
      uint4 v[NPW];
#pragma unroll
      for (int j = 0; j < NPW; ++j)
        if ((32 * j) / PPT < mloc) v[j] = lds128(st + Gm::RAW_OFS + (lane + 32 * j) * 16);
      const uint2 sv = lds64(st + Gm::SC_OFS + lane * 16);
      const uint2 sv2 = lds64(st + Gm::SC_OFS + lane * 16 + 8);
      __syncwarp();
      if (lane == 0) mbar_arrive(&sfree[s]);  // stage fully read by this warp
      DTC_PW(5, mbar_wait(&bfree[b], bph ^ 1))
      DTC_PW(6, mbar_wait(&fdfree[f], fph ^ 1))
      const uint32_t bt = sb + Gm::B_RING + b * Gm::B_BYTES;
      float* fdp = reinterpret_cast<float*>(sbase + Gm::FD_RING + f * Gm::FD_BYTES);
#pragma unroll
      for (int j = 0; j < NPW; ++j) {
        if ((dbg & 4) || (32 * j) / PPT >= mloc) continue;  // warp-uniform: tokens >= M not staged
        const int pc = lane + 32 * j;
        const int tok = pc / PPT, kl = (pc % PPT) * 8;
        uint4 x = v[j];
        if (OFF != 0.f) {
          float sum = 0.f;
          const uint32_t vv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (Dt<T>::id == FQ_BF16) {
              sum += __uint_as_float(vv[e] << 16) + __uint_as_float(vv[e] & 0xFFFF0000u);
            } else {
              const float2 ff = __half22float2(*reinterpret_cast<const __half2*>(&vv[e]));
              sum += ff.x + ff.y;
            }
          }
#pragma unroll
          for (int o = PPT / 2; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
          if ((lane % PPT) == 0) fdp[tok] = sum;
        }
        if (BITS == 4)
          x = make_uint4(prmt(x.x, x.z, 0x5410u), prmt(x.x, x.z, 0x7632u), prmt(x.y, x.w, 0x5410u),
                         prmt(x.y, x.w, 0x7632u));
        const int atom = kl >> 6, chunk = (kl & 63) >> 3;
        sts128(bt + atom * 2048 + tok * 128 + ((chunk ^ (tok & 7)) << 4), x);
      }
      {  // the stage's 256 scales -> fp32 (lane handles rows 8*lane .. 8*lane+7)
        const uint32_t h[8] = {sv.x & 0xFFFFu, sv.x >> 16, sv.y & 0xFFFFu, sv.y >> 16,
                               sv2.x & 0xFFFFu, sv2.x >> 16, sv2.y & 0xFFFFu, sv2.y >> 16};
        float sc[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const unsigned short hv = (unsigned short)h[e];
          sc[e] = Dt<T>::to_f(*reinterpret_cast<const T*>(&hv));
        }
        const uint32_t fa = smem_u32(fdp + NT + lane * 8);
        sts128(fa, make_uint4(__float_as_uint(sc[0]), __float_as_uint(sc[1]), __float_as_uint(sc[2]),
                              __float_as_uint(sc[3])));
        sts128(fa + 16, make_uint4(__float_as_uint(sc[4]), __float_as_uint(sc[5]), __float_as_uint(sc[6]),
                                   __float_as_uint(sc[7])));
      }
      fence_proxy_async_smem();  // generic-proxy B-tile stores -> visible to the tensor core
      __syncwarp();
      if (lane == 0) mbar_arrive(&bready[b]);
      if (++s == SST) { s = 0; ph ^= 1; }
      if (++b == NB) { b = 0; bph ^= 1; }
      if (++f == FD) { f = 0; fph ^= 1; }
      cur_next(batch, cur);
    }
  } else if (warp < 11) {
    // ------------------------------------------------------------------ dequant -> TMEM
    const int quarter = warp & 3;             // TMEM lane quarter this warp may access
    const int half = (warp - 3) >> 2;         // UMMA M half (rows 0..127 / 128..255)
    const int row = half * 128 + quarter * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    int s = 0, a = 0;
    uint32_t ph = 0, aph = 0;
    for (int i = 0; i < nst; ++i) {
      DTC_PW(7, mbar_wait(&full_bar[s], ph))
      const uint32_t wrow = sb + s * Gm::STAGE + row * Gm::WB;
      uint4 c[4];
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) c[cc] = lds128(wrow + ((cc ^ ((row >> 1) & 3)) << 4));
      __syncwarp();
      if (lane == 0) mbar_arrive(&sfree[s]);  // codes are in registers: the TMA may refill
      DTC_PW(8, mbar_wait(&afree[a], aph ^ 1))
      fence_after();
      const uint32_t words[16] = {c[0].x, c[0].y, c[0].z, c[0].w, c[1].x, c[1].y, c[1].z, c[1].w,
                                  c[2].x, c[2].y, c[2].z, c[2].w, c[3].x, c[3].y, c[3].z, c[3].w};
      constexpr int PAIRS_PER_WORD = BITS == 4 ? 4 : 2;
      constexpr int NPAIR = 16 * PAIRS_PER_WORD;  // 64 (int4) / 32 (int8) TMEM columns
#pragma unroll
      for (int hh = 0; hh < NPAIR / 32; ++hh) {
        uint32_t q[32];
#pragma unroll
        for (int w = 0; w < 32 / PAIRS_PER_WORD; ++w) {
          if (dbg & 1) {
#pragma unroll
            for (int u = 0; u < PAIRS_PER_WORD; ++u) q[w * PAIRS_PER_WORD + u] = words[hh * (32 / PAIRS_PER_WORD) + w];
          } else {
            unpack_word<T, BITS>(words[hh * (32 / PAIRS_PER_WORD) + w], &q[w * PAIRS_PER_WORD]);
          }
        }
        if (dbg & 16) {  // diagnostics: keep the values live without the TMEM store
          uint32_t x = 0;
#pragma unroll
          for (int u = 0; u < 32; ++u) x ^= q[u];
          if (x == 0x9E3779B9u) tmem_st32(tmem + lane_base + a * KS + half * Gm::A_COLS + hh * 32, q);
        } else {
          tmem_st32(tmem + lane_base + a * KS + half * Gm::A_COLS + hh * 32, q);
        }
      }
      tmem_wait_st();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&aready[a]);
      if (++s == SST) { s = 0; ph ^= 1; }
      if (++a == AST) { a = 0; aph ^= 1; }
    }
  } else {
    // ------------------------------------------------------------------ fold + epilogue
    const int quarter = warp & 3;
    const int half = (warp - 11) >> 2;
    const int row = half * 128 + quarter * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const int ftid = threadIdx.x - 11 * 32;   // 0..255 among the fold warps
    float acc[NTF];
#pragma unroll
    for (int t = 0; t < NTF; ++t) acc[t] = 0.f;
    Cur cur;
    if (nst > 0) cur_locate(batch, b0, cur);
    int seg_k0 = nst > 0 ? cur.kidx : 0;
    bool first_seg = true;
    int c = 0, f = 0;
    uint32_t cph = 0;
    for (int i = 0; i < nst; ++i) {
      DTC_PW(9, mbar_wait(&accfull[c], cph))
      fence_after();
      uint32_t v[NTF];
      tmem_ldn<NTF>(tmem + lane_base + Gm::ACC_COL + c * 2 * NT + half * NT, v);
      const float* fdp = reinterpret_cast<const float*>(sbase + Gm::FD_RING + f * Gm::FD_BYTES);
      const float sc = fdp[NT + row];
      float sums[NTF];
#pragma unroll
      for (int t = 0; t < NTF; ++t) sums[t] = OFF != 0.f ? fdp[t] : 0.f;
      tmem_wait_ld();
      fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&accfree[c]);
        mbar_arrive(&fdfree[f]);
      }
      if (!(dbg & 2)) {
#pragma unroll
        for (int t = 0; t < NTF; ++t) {
          float part = __uint_as_float(v[t]);
          if (OFF != 0.f) part = fmaf(-OFF, sums[t], part);
          acc[t] = fmaf(sc, part, acc[t]);
        }
      }
      if (++c == ACC) { c = 0; cph ^= 1; }
      if (++f == FD) f = 0;

      const DtcProb& p = batch.p[cur.p];
      if (cur.kidx == p.nk - 1 || i == nst - 1) {
        // ---- end of a tile segment: C (whole tile in this CTA) or a split partial
        const int n = cur.tile * ROWS + row;
        const int M = p.M;
        auto store_out = [&](int tok, float val) {
          const size_t o = (size_t)tok * p.N + n;
          if (p.cdt == FQ_FP32) reinterpret_cast<float*>(p.C)[o] = val;
          else reinterpret_cast<T*>(p.C)[o] = Dt<T>::from_f(val);
        };
        if (seg_k0 == 0 && cur.kidx == p.nk - 1) {
          if (n < p.N) {
#pragma unroll
            for (int t = 0; t < NTF; ++t)
              if (t < M) store_out(t, acc[t]);
          }
        } else {
          const int slot = first_seg ? 0 : 1;
          float* wsp = batch.ws + (size_t)(cta * 2 + slot) * NT * ROWS;
#pragma unroll
          for (int t = 0; t < NTF; ++t)
            if (t < M) __stcg(wsp + t * ROWS + row, acc[t]);
          const int ts = p.stage_begin + cur.tile * p.nk;
          const int c_lo = cta_of(TS, P, ts), c_hi = cta_of(TS, P, ts + p.nk - 1);
          int* ctr = batch.counters + p.tile_begin + cur.tile;
          asm volatile("bar.sync 1, 256;" ::: "memory");
          if (ftid == 0) {
            __threadfence();
            const int last = atomicAdd(ctr, 1) == c_hi - c_lo;
            if (last) __threadfence();
            s_last = last;
          }
          asm volatile("bar.sync 1, 256;" ::: "memory");
          const int last = s_last;
          if (last) {
            if (n < p.N) {
#pragma unroll
              for (int t = 0; t < NTF; ++t) {
                if (t < M) {
                  float val = 0.f;
                  for (int cc = c_lo; cc <= c_hi; ++cc) {
                    const int sl = range_begin(TS, P, cc) >= ts ? 0 : 1;
                    val += __ldcg(batch.ws + ((size_t)(cc * 2 + sl) * NT + t) * ROWS + row);
                  }
                  store_out(t, val);
                }
              }
            }
            if (ftid == 0) *ctr = 0;  // self-reset for the next launch
          }
          asm volatile("bar.sync 1, 256;" ::: "memory");  // s_last reused by the next segment
        }
#pragma unroll
        for (int t = 0; t < NTF; ++t) acc[t] = 0.f;
        first_seg = false;
        seg_k0 = 0;
      }
      cur_next(batch, cur);
    }
  }
#if FQ_DTC_PROF
  if (blockIdx.x == 0 && lane == 0)
    printf("prof warp %2d total %lld waits %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld nst %d\n", warp,
           clock64() - tstart_, prof_[0], prof_[1], prof_[2], prof_[3], prof_[4], prof_[5], prof_[6], prof_[7],
           prof_[8], prof_[9], nst);
#endif
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

}  // namespace dtc

// ------------------------------------------------------------------------------------- host side
constexpr size_t kDtcCounterBytes = 65536;
constexpr int kDtcMaxTiles = (int)(kDtcCounterBytes / sizeof(int));

bool decode_tc_supported(int bits, int group, int M) {
  // Opt-in (FQ_DECODE_TC=1): correct, but slower than the mma.sync kernel on B200 (round-1
  // diagnostics: the per-stage TMEM/MMA/fold hand-offs cost more issue slots than they save).
  const char* e = std::getenv("FQ_DECODE_TC");
  if (!e || e[0] != '1') return false;
  return M >= 1 && M <= dtc::NT && group % (bits == 4 ? 128 : 64) == 0;
}

static int dtc_ctas(long long total_stages, int nsm) {
  // at least 4 stages per CTA so tiny problems are not shredded into single-stage partials
  const long long c = std::min<long long>(nsm, (total_stages + 3) / 4);
  return (int)std::max<long long>(1, c);
}

size_t dtc_workspace_bytes(int M, int K, int N, int bits, int nsm) {
  (void)M; (void)K; (void)N; (void)bits;
  return kDtcCounterBytes + (size_t)nsm * 2 * dtc::NT * dtc::ROWS * sizeof(float);
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
  if (maxm <= 8) return dispatch_dtc_t<MAXP, 8>(adt, bits, b, ctas, st);
  return dispatch_dtc_t<MAXP, 16>(adt, bits, b, ctas, st);
}

static bool make_dtc_prob(dtc::DtcProb& d, int bits, int cdt, const void* A, int M, int K, int N,
                          const void* codes, const void* scales, int group, void* C) {
  const uint64_t row_bytes = (uint64_t)K * bits / 8;
  const int ks = 64 * 8 / bits;
  if (!make_tmap_2d(&d.w, codes, 1, row_bytes, (uint64_t)N, row_bytes, 64, dtc::ROWS, 64)) return false;
  if (!make_tmap_2d(&d.a, A, 2, (uint64_t)K, (uint64_t)M, (uint64_t)K * 2, ks, M, 0)) return false;
  if (!make_tmap_2d(&d.s, scales, 2, (uint64_t)N, (uint64_t)(K / group), (uint64_t)N * 2, dtc::ROWS, 1, 0))
    return false;
  d.C = C;
  d.M = M; d.K = K; d.N = N; d.group = group; d.cdt = cdt;
  d.gx = (N + dtc::ROWS - 1) / dtc::ROWS;
  d.nk = (K + ks - 1) / ks;
  return true;
}

static int dtc_dbg() {
  const char* db = std::getenv("FQ_DTC_DBG");
  return db ? std::atoi(db) : 0;
}

cudaError_t run_decode_tc(int adt, int cdt, int bits, const void* A, int M, int K, int N, const void* codes,
                          const void* scales, int group, void* C, void* ws, cudaStream_t st) {
  dtc::DtcBatch<1> b{};
  if (!make_dtc_prob(b.p[0], bits, cdt, A, M, K, N, codes, scales, group, C)) return cudaErrorInvalidValue;
  if (b.p[0].gx > kDtcMaxTiles) return cudaErrorInvalidValue;
  b.p[0].stage_begin = 0;
  b.p[0].tile_begin = 0;
  b.nprob = 1;
  b.total_stages = b.p[0].gx * b.p[0].nk;
  b.counters = reinterpret_cast<int*>(ws);
  b.ws = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + kDtcCounterBytes);
  b.dbg = dtc_dbg();
  return dispatch_dtc<1>(adt, bits, b, dtc_ctas(b.total_stages, num_sms()), st, M);
}

// MoE batch on the tcgen05 decode kernel: experts (1 <= M_e <= 16, group % KS == 0) share one
// stream-K launch per <= MAXP experts (all of their tiles in one linear stage space).
cudaError_t run_decode_tc_grouped(int adt, int cdt, int bits, const void* A, int K, int N, const int64_t* offsets,
                                  const int32_t* groups, const void* const* codes, const void* const* scales,
                                  void* C, void* ws, const int* experts, int nexp, cudaStream_t st) {
  constexpr int MAXP = 40;
  static_assert(sizeof(dtc::DtcBatch<MAXP>) < 32000, "kernel parameter block limit");
  dtc::DtcBatch<MAXP> b{};
  b.counters = reinterpret_cast<int*>(ws);
  b.ws = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + kDtcCounterBytes);
  b.dbg = dtc_dbg();
  int stages = 0, tiles = 0, maxm = 0;
  auto flush = [&]() -> cudaError_t {
    b.total_stages = stages;
    cudaError_t r = dispatch_dtc<MAXP>(adt, bits, b, dtc_ctas(stages, num_sms()), st, maxm);
    b.nprob = 0;
    stages = tiles = maxm = 0;
    return r;
  };
  for (int ii = 0; ii < nexp; ++ii) {
    const int e = experts[ii];
    const int Me = (int)(offsets[e + 1] - offsets[e]);
    const char* Ae = reinterpret_cast<const char*>(A) + (size_t)offsets[e] * K * 2;
    char* Ce = reinterpret_cast<char*>(C) + (size_t)offsets[e] * N * (cdt == FQ_FP32 ? 4 : 2);
    dtc::DtcProb& d = b.p[b.nprob];
    if (!make_dtc_prob(d, bits, cdt, Ae, Me, K, N, codes[e], scales[e], groups[e], Ce))
      return cudaErrorInvalidValue;
    if (tiles + d.gx > kDtcMaxTiles) {  // counter region full: launch what we have first
      cudaError_t r = flush();
      if (r != cudaSuccess) return r;
      b.p[0] = d;
    }
    dtc::DtcProb& dd = b.p[b.nprob];
    dd.stage_begin = stages;
    dd.tile_begin = tiles;
    stages += dd.gx * dd.nk;
    tiles += dd.gx;
    maxm = std::max(maxm, Me);
    if (++b.nprob == MAXP) {
      cudaError_t r = flush();
      if (r != cudaSuccess) return r;
    }
  }
  if (b.nprob) return flush();
  return cudaSuccess;
}

}  // namespace fq
