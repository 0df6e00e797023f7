// fq_gemm_tc.cu — kernel A6: large-M (prefill) fused dequant GEMM on the 5th-gen tensor cores.
//
// Same math as A4 (§4.1): C[m,n] = sum_k A[m,k] * (q[n,k] * s[k/g, n]), weights
// dequantized to the activation dtype before the tensor-core MMA ("dequantize the weights to match
// the data type of the activation and perform floating-point tensor core math"), fp32
// accumulation.  The paper notes that in this compute-bound regime "the conversions from integer
// to float bottleneck our kernels, rather than tensor core math"; the B200 design keeps the
// conversion off the tensor core's critical path by warp specialisation and by writing the
// dequantized weights straight into tensor memory (no shared-memory round trip):
//
//   tile = 128 weight rows (output columns n) x bn tokens (bn = round_up(M, 16) <= 256), persistent
//   CTAs.  Kernel variant by the launch's widest token tile: 256 tokens with 64-k stages and 8
//   dequant warps; 128 / 64 tokens with 128-k stages (two activation boxes, 64 / 128-byte code
//   rows) and 16 dequant warps.
//   warp 0      TMA producer: activations [bn tokens x 64 k] per box (SWIZZLE_128B, the UMMA K-major
//               canonical layout) + packed codes [128 rows x BK k] (SWIZZLE_32B/64B/128B by row
//               bytes) + the K block's scale rows, one mbarrier ring.
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer:
//                 D[n, tok] (fp32, TMEM, bn columns) += A[n, k] (bf16, TMEM) * B[k, tok] (smem)
//               "kind::f16", M=128, N=bn, K=16; tcgen05.commit releases the stage.
//   warps 2..   dequant: thread = one weight row (its TMEM lane) x BK / (warps / 4) k; codes ->
//               exact bf16 codes (PRMT/IMAD/LOP3 magic-number unpack, natural (k,k+1) pairs) ->
//               * scale -> tcgen05.st into the stage's A slot.  After the last K block of a work
//               item the same warps drain the accumulator (tcgen05.ld) and store C, or an fp32
//               split-K partial that the last-arriving split reduces in split order.
//   TMEM: accumulator columns [0, BNMAX) + one A slot of BK/2 columns per stage.
//   Two-half tiles (HM = 2, the <= 64-token variant): 256 weight rows per tile as two UMMA M=128
//   halves that share each staged activation tile, so a stage carries twice the code bytes for the
//   same activation bytes (the small-M regime is bound by code bytes in flight per SM).  The
//   halves' A operands then need 2 x BK/2 TMEM columns per K block, fewer slots than smem stages:
//   the A slots form their own ring (released by the MMA commit) behind the smem stage ring.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "fq_common.cuh"
#include "fq_internal.h"
#include "fq_tcgen05.cuh"

namespace fq {
namespace tc {

constexpr int BM = 128;        // weight rows per tile (UMMA M)
constexpr int BN = 256;        // max tokens per tile (UMMA N); a problem with M < 256 uses
                               // bn = round_up(M, 16) (TcProb::bn): no wasted MMA / activation TMA
constexpr int BKA = 64;        // K per activation TMA box (one SWIZZLE_128B atom of bf16)
// K per stage (template BK): 64, or 128 for the 64/128-token variants -- two activation boxes, and
// 64-byte (int4) / 128-byte (int8) code rows, which TMA streams far better than 32-byte rows
// Dequant warps per CTA: dq_warps(BNMAX) / 4 per TMEM lane quarter, each covering BK / parts k of a
// K block.  Measured: 16 warps are faster for the small-tile variants (memory/latency-bound
// regime), 8 for the 256-token variant (tensor-bound prefill).
#ifndef FQ_TC_DBG
#define FQ_TC_DBG 0  // diagnostics only: 1 = no MMA, 2 = no dequant / tcgen05.st, 3 = both (TMA pipeline alone)
#endif
#ifndef FQ_TC_DQW
#define FQ_TC_DQW 0  // diagnostics: force 8 or 16 for every variant
#endif
#ifndef FQ_TC_CPS_SMALL
#define FQ_TC_CPS_SMALL 2  // max CTAs per SM of the <= 64-token int4 one-half variants (host rule: tc_use_cps2)
#endif
__host__ __device__ constexpr int dq_warps(int bnmax, int cps = 1) {
  return FQ_TC_DQW ? FQ_TC_DQW : ((bnmax == 256 || cps == 2) ? 8 : 16);
}
__host__ __device__ constexpr int tc_threads(int bnmax, int cps = 1) { return 32 * (2 + dq_warps(bnmax, cps)); }
constexpr int kTmemCols = 512;
constexpr int kAccCol = 0;                 // accumulator columns [0, BNMAX)
__host__ __device__ constexpr int sc_rows_max(int bk) { return bk / 16 + 1; }  // >= ceil((bk-1)/g) + 1, g >= 16
constexpr int kSmemMax = 227 * 1024 - 2048;

// Stage geometry of one kernel variant.  BNMAX = widest token tile it serves: a small-M variant
// has small activation tiles, so it keeps many more K blocks (codes) in flight -- at M <= 128 the
// kernel is bound by HBM latency x bytes in flight, not by the tensor cores.
//   TMEM: accumulator columns [0, BNMAX), A slot s at BNMAX + 32 s (one per stage).
// CPS = CTAs per SM: 2 halves each CTA's TMEM (256 columns) and shared memory and uses 8 dequant
// warps -- two independent pipelines per SM (<= 64-token int4 one-half tiles; see tc_use_cps2).
template <int BITS, int BNMAX, int BK, int HM, int CPS = 1>
struct Geo {
  static constexpr int BMT = BM * HM;                         // weight rows per tile
  static constexpr int ACT_BOX = BNMAX * BKA * 2;             // one activation box slot (SW128 atoms)
  static constexpr int ACT_BYTES = ACT_BOX * (BK / BKA);
  static constexpr int CODE_BYTES_ROW = BK * BITS / 8;        // 32 / 64 / 128 bytes
  static constexpr int CODE_HALF = BM * CODE_BYTES_ROW;       // codes of one 128-row half
  static constexpr int CODE_BYTES = CODE_HALF * HM;
  static constexpr int SC_OFS = ACT_BYTES + CODE_BYTES;       // scale rows of the K block
  static constexpr int SC_ROWS = sc_rows_max(BK);
  static constexpr int SC_HALF = SC_ROWS * BM * 2;            // scale rows of one half
  static constexpr int SC_BYTES = SC_HALF * HM;
  static constexpr int STAGE = ((SC_OFS + SC_BYTES + 1023) / 1024) * 1024;
  static constexpr int TMEM = kTmemCols / CPS;
  static constexpr int S_SMEM = ((kSmemMax + 2048) / CPS - 2048 - 1024) / STAGE;
  static constexpr int A_HALF = BK / 2;                       // TMEM columns of one half's A operand
  static constexpr int A_COLS = A_HALF * HM;                  // TMEM columns of one A slot
  static constexpr int ACC_COLS = BNMAX * HM;                 // accumulator columns (half h at h*BNMAX)
  static constexpr int S_TMEM = (TMEM - ACC_COLS) / A_COLS;
  // One-half tiles of >= 64 tokens: one A slot per smem stage (slot index = stage index).  Two-half
  // tiles and the 32-token variant: more smem stages than TMEM holds A slots, so the A slots form a
  // separate ring behind the stage ring.
  static constexpr int S0 = (HM == 1 && BNMAX > 32 && CPS == 1 && S_TMEM < S_SMEM) ? S_TMEM : S_SMEM;
  static constexpr int STAGES = S0 > 16 ? 16 : S0;
  static constexpr int ASLOTS = S_TMEM < STAGES ? S_TMEM : STAGES;
  static constexpr bool SEP_A = ASLOTS < STAGES;
  static constexpr int SMEM = STAGES * STAGE + 1024;
  static constexpr int A_COL = ACC_COLS;
  static_assert(STAGES >= (HM == 1 ? 4 : 3) && ASLOTS >= 2, "stages");
};

using namespace tc5;

// Natural (k, k+1) pairs of an int4 word (k..k+7) as exact codes in T: byte i holds (k+2i, k+2i+1).
template <typename T>
__device__ __forceinline__ void i4_nat_pairs(uint32_t w, uint32_t (&q)[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t x = prmt(w, 0u, 0x4440u + i);  // byte i, zero extended
    const uint32_t y = x * 0x1001u;                // lo nibble at bits 0-3, hi nibble at 16-19
    const uint32_t v = lop3_and_xor(y, 0x000F000Fu, Dt<T>::kMagic4);
    if (Dt<T>::id == FQ_BF16) asm("sub.rn.bf16x2 %0, %1, %2;" : "=r"(q[i]) : "r"(v), "r"(Dt<T>::kBias4));
    else asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(q[i]) : "r"(v), "r"(Dt<T>::kBias4));
  }
}
// Natural pairs of an int8 word (k..k+3): exact codes.
template <typename T>
__device__ __forceinline__ void i8_nat_pairs(uint32_t w, uint32_t (&q)[2]) {
  const uint32_t u = w ^ 0x80808080u;
  if (Dt<T>::id == FQ_FP16) {
    asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(q[0]) : "r"(prmt(u, 0x64646464u, 0x4140u)), "r"(0x64806480u));
    asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(q[1]) : "r"(prmt(u, 0x64646464u, 0x4342u)), "r"(0x64806480u));
  } else {
    float f[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) f[i] = __uint_as_float(prmt(u, 0x4B000000u, 0x7440u + i)) - 8388736.0f;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(q[0]) : "f"(f[1]), "f"(f[0]));
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(q[1]) : "f"(f[3]), "f"(f[2]));
  }
}
template <typename T>
__device__ __forceinline__ uint32_t mul2x(uint32_t a, uint32_t b) {
  uint32_t d;
  if (Dt<T>::id == FQ_BF16) asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  else asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

// Tile raster: groups of up to 8 token tiles; inside a group the token tile varies fastest, so the
// ~148 concurrently running tiles cover <= 8 activation row-blocks and ~18 weight row-blocks and
// their K slices are shared through L2 (plain m-fastest order re-streams the activations of every
// weight tile from HBM once M exceeds ~2048 tokens).
__device__ __forceinline__ void tile_coords(int tile, int m_tiles, int n_tiles, int GM, int& mt, int& nt) {
  const int group = tile / (GM * n_tiles);
  const int gm = min(GM, m_tiles - group * GM);
  const int local = tile - group * GM * n_tiles;
  mt = group * GM + local % gm;
  nt = local / gm;
}

// One GEMM of a batch (MoE experts: one launch covers every large expert; tiles are numbered
// consecutively across problems and the persistent CTAs walk the global tile list).
struct TcProb {
  CUtensorMap a, q;  // activations [M][K] (box 256 x 64, SWIZZLE_128B); codes [N][K*b/8]
  CUtensorMap s;     // scales [G][N] (box sc_rows_max(BK) rows x 128 columns, OOB rows zero)
  int bk;            // K per stage of the kernel variant this problem was prepared for
  int hm;            // 128-row halves per tile of that variant (tile = 128 * hm weight rows)
  const void* scales;
  void* C;
  int M, K, N, group, cdt;
  int m_tiles, n_tiles;
  int bn;            // tokens per tile (UMMA N): min(256, round_up(M, 16))
  int gm;            // token tiles per raster group
  int tile_begin;
  int splits, kbs;   // split-K (few output tiles): K-block ranges of kbs blocks per work item
  float* ws;         // split-K fp32 partials [tiles * splits][bn][128]
  int* ctr;          // split-K arrival counters per output tile (self-resetting)
  // MoE batch with DEVICE expert offsets (fq_gemm_grouped_dev): rows offs[e] .. offs[e+1]-1 of the
  // whole A / C (the activation map spans all `rows`); M is the launch's token bound.
  const int64_t* offs;
  int e, rows;
  int skip;          // the expert's first `skip` tokens are served by the decode kernel (device offsets)
  int32_t* status;   // nullable: bit 2 = more tokens than the bound / offsets outside [0, rows]
};
// this problem's first row and token count (device offsets clamped to the rows and the bound)
__device__ __forceinline__ void prob_rows(const TcProb& p, int& row0, int& Me) {
  row0 = 0;
  Me = p.M;
  if (p.offs) {
    const int64_t o0 = p.offs[p.e], o1 = p.offs[p.e + 1];
    const int64_t lo = max((int64_t)0, min(o0, (int64_t)p.rows)), hi = max(lo, min(o1, (int64_t)p.rows));
    row0 = (int)lo + p.skip;
    Me = (int)max((int64_t)0, min(hi - lo - p.skip, (int64_t)p.M));
  }
}
// work item -> (token tile, weight-row tile, K-block range); work items of one output tile are
// consecutive (its K splits run concurrently on neighbouring CTAs)
template <int BK>
__device__ __forceinline__ void work_coords(const TcProb& p, int item, int& mt, int& nt, int& t, int& ks,
                                            int& kb0, int& kb1) {
  const int local = item - p.tile_begin;
  t = local / p.splits;
  ks = local - t * p.splits;
  tile_coords(t, p.m_tiles, p.n_tiles, p.gm, mt, nt);
  const int kblocks = (p.K + BK - 1) / BK;
  kb0 = ks * p.kbs;
  kb1 = min(kblocks, kb0 + p.kbs);
}
template <int MAXP>
struct TcBatch {
  TcProb p[MAXP];
  int nprob, total_tiles;
};

template <int MAXP>
__device__ __forceinline__ const TcProb& find_prob(const TcBatch<MAXP>& b, int tile) {
  int pi = 0;
  while (pi + 1 < b.nprob && tile >= b.p[pi + 1].tile_begin) ++pi;
  return b.p[pi];
}

// 16-byte chunk c of code row r in shared memory under the TMA swizzle of ROWB-byte rows
template <int ROWB>
__device__ __forceinline__ int swz_chunk(int c, int r) {
  return ROWB == 32 ? c ^ ((r >> 2) & 1) : ROWB == 64 ? c ^ ((r >> 1) & 3) : c ^ (r & 7);
}

template <typename T, int BITS, int MAXP, int BNMAX, int BK, int HM, int DQG, int CPS>
__global__ void __launch_bounds__(tc_threads(BNMAX, CPS), CPS)
    gemm_tc_kernel(const __grid_constant__ TcBatch<MAXP> batch) {
  constexpr int kDqWarps = dq_warps(BNMAX, CPS);
  constexpr int kParts = kDqWarps / 4;
  // With 16 dequant warps, two groups of 8 take alternate K blocks, so one group's tcgen05.st /
  // wait::st / arrive latency overlaps the other's loads and unpacking (each group covers a whole
  // K block: two warps per TMEM lane quarter, kKPW = BK / 2).
  constexpr int kDqGroups = kDqWarps == 16 ? DQG : 1;
  constexpr int kPartsG = kParts / kDqGroups;
  constexpr int kKPW = BK / kPartsG;  // k per dequant thread per K block (16 / 32 / 64)
  using Gm = Geo<BITS, BNMAX, BK, HM, CPS>;
  constexpr int STAGES = Gm::STAGES;
  constexpr int ASLOTS = Gm::ASLOTS;
  constexpr bool kSepA = Gm::SEP_A;  // A slots in their own ring (see Geo)
  constexpr int BMT = Gm::BMT;
  constexpr int kACol = Gm::A_COL;
  extern __shared__ __align__(1024) uint8_t dsmem[];
  __shared__ __align__(8) uint64_t full_bar[STAGES], afull_bar[ASLOTS], empty_bar[STAGES], aempty_bar[ASLOTS];
  __shared__ __align__(8) uint64_t acc_full, acc_empty;
  __shared__ uint32_t tmem_base_sh;
  __shared__ int s_last;
  uint8_t* sbase = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsmem) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = batch.total_tiles;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < ASLOTS; ++a) {
      mbar_init(&afull_bar[a], kDqWarps / kDqGroups);  // one arrival per warp of the block's group
      mbar_init(&aempty_bar[a], 1);        // MMA commit (separate slot ring only)
    }
    mbar_init(&acc_full, 1);
    mbar_init(&acc_empty, kDqWarps);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&tmem_base_sh, Gm::TMEM);
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < batch.nprob; ++i) {
      prefetch_tmap(&batch.p[i].a);
      prefetch_tmap(&batch.p[i].q);
      prefetch_tmap(&batch.p[i].s);
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tmem_base_sh;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t pol_a = policy_evict_last();
      const uint64_t pol_q = policy_evict_first();
      int s = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const TcProb& p = find_prob(batch, tile);
        int mt, nt, tt, ks, kb0, kb1;
        work_coords<BK>(p, tile, mt, nt, tt, ks, kb0, kb1);
        int row0, Me;
        prob_rows(p, row0, Me);
        if (mt * p.bn >= Me) continue;  // device offsets: token tile beyond this expert's tokens
        // first scale row of the K block = floor(BK kb / g), division-free after the first block
        const int grp = p.group;  // hoisted out of the parameter space
        // halves entirely past the last weight row are not loaded (their TMEM rows are never stored)
        const int nh = HM == 1 ? 1 : min(HM, (p.N - nt * BMT + BM - 1) / BM);
        const uint32_t tx = p.bn * BK * 2 + nh * (Gm::CODE_HALF + Gm::SC_HALF);
        const int arow = row0 + mt * p.bn, wrow = nt * BMT;
        int j0 = (kb0 * BK) / grp, r0 = (kb0 * BK) - j0 * grp;
        for (int kb = kb0; kb < kb1; ++kb, r0 += BK) {
          while (r0 >= grp) { r0 -= grp; ++j0; }
          mbar_wait(&empty_bar[s], ph ^ 1);
          uint8_t* st = sbase + s * Gm::STAGE;
          mbar_arrive_expect_tx(&full_bar[s], tx);
          for (int hh = 0; hh < nh; ++hh)
            tma_load_2d(st + Gm::SC_OFS + hh * Gm::SC_HALF, &p.s, &full_bar[s], wrow + hh * BM, j0, pol_q);
#pragma unroll
          for (int h = 0; h < BK / BKA; ++h)
            tma_load_2d(st + h * Gm::ACT_BOX, &p.a, &full_bar[s], kb * BK + h * BKA, arow, pol_a);
          for (int hh = 0; hh < nh; ++hh)
            tma_load_2d(st + Gm::ACT_BYTES + hh * Gm::CODE_HALF, &p.q, &full_bar[s], kb * Gm::CODE_BYTES_ROW,
                        wrow + hh * BM, pol_q);
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t sb = smem_u32(sbase);
      int s = 0, a = 0;
      uint32_t ph = 0, aph = 0, acc_ph = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const TcProb& pp = find_prob(batch, tile);
        int mt_, nt_, tt_, ks_, kb0, kb1;
        work_coords<BK>(pp, tile, mt_, nt_, tt_, ks_, kb0, kb1);
        int row0_, Me_;
        prob_rows(pp, row0_, Me_);
        if (mt_ * pp.bn >= Me_) continue;
        // N = bn; with device offsets, only the tile's real tokens (rounded up to 16): a partly filled
        // tile of a small expert costs proportionally less tensor-core time
        const int nn = pp.offs ? min(pp.bn, (Me_ - mt_ * pp.bn + 15) / 16 * 16) : pp.bn;
        const uint32_t idesc = idesc_f16<T, BM, 16>() + ((uint32_t)((nn >> 3) - 2) << 17);
        mbar_wait(&acc_empty, acc_ph ^ 1);  // epilogue drained the accumulator
        fence_after();
        for (int kb = kb0; kb < kb1; ++kb) {
          const int slot = kSepA ? a : s;
          mbar_wait(&full_bar[s], ph);
          mbar_wait(&afull_bar[slot], kSepA ? aph : ph);
          fence_after();
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t bdesc = sw128_desc(sb + s * Gm::STAGE + (kk / 4) * Gm::ACT_BOX);
#pragma unroll
            for (int h = 0; h < HM; ++h)
              if (!(FQ_TC_DBG & 1))
                mma_ts(tmem + kAccCol + h * BNMAX, tmem + kACol + slot * Gm::A_COLS + h * Gm::A_HALF + kk * 8,
                       bdesc + (uint64_t)((kk % 4) * 2), idesc, (kb != kb0) || (kk != 0));
          }
          mma_commit(&empty_bar[s]);
          if (kSepA) {
            mma_commit(&aempty_bar[slot]);
            if (++a == ASLOTS) { a = 0; aph ^= 1; }
          }
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
        mma_commit(&acc_full);
        acc_ph ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------------ dequant + epilogue
    const int dq = warp - 2;
    const int quarter = warp & 3;            // TMEM lane quarter this warp may access
    const int half = dq >> 2;                // accumulator (token) part this warp drains
    const int kp = half % kPartsG;           // which kKPW k of the K block this warp dequantizes
    const int dgrp = half / kPartsG;         // its group: K blocks with (block counter % groups) == dgrp
    const int row = quarter * 32 + lane;     // weight row within the tile == TMEM lane
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t sb = smem_u32(sbase);
    int s = 0, a = 0, blk = 0;
    uint32_t ph = 0, aph = 0, acc_ph = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const TcProb& p = find_prob(batch, tile);
      const int N = p.N;
      int mt, nt, tt, ks, kb0, kb1;
      work_coords<BK>(p, tile, mt, nt, tt, ks, kb0, kb1);
      int row0, M;
      prob_rows(p, row0, M);
      if (mt * p.bn >= M) continue;
      const int grp = p.group;                     // hoisted: p lives in the parameter space
      const bool one_scale = grp % kKPW == 0;      // this thread's kKPW k lie in one group
      int j0 = (kb0 * BK) / grp, r0 = kb0 * BK - j0 * grp;  // first staged scale row
      // group of this thread's first k (kb0*BK + half*kKPW) and its offset in the group
      int jb = (kb0 * BK + kp * kKPW) / grp, gk = kb0 * BK + kp * kKPW - jb * grp;
      const uint32_t srow = sb + Gm::SC_OFS + row * 2;
      for (int kb = kb0; kb < kb1; ++kb) {
        // scales of this thread's 8-k words from the TMA-staged rows: word w lies in group
        // jb + t, t = [gk + 8w >= g] + [gk + 8w >= 2g]; row index in smem = group - j0.
        const int slot = kSepA ? a : s;
        if (kDqGroups == 1 || (blk % kDqGroups) == dgrp) {
        mbar_wait(&full_bar[s], ph);
        constexpr int NW = kKPW / 8;  // 8-k words of this thread
#pragma unroll
        for (int h = 0; h < HM; ++h) {
          uint32_t sc[NW];
          const uint32_t srh = srow + s * Gm::STAGE + h * Gm::SC_HALF;
          if (one_scale) {
            const uint32_t v = lds_u16(srh + (jb - j0) * BM * 2);
            const uint32_t v2 = prmt(v, v, 0x1010u);
#pragma unroll
            for (int w = 0; w < NW; ++w) sc[w] = v2;
          } else {
#pragma unroll
            for (int w = 0; w < NW; ++w) {
              const int o = gk + 8 * w;  // < grp + kKPW: at most kKPW / 16 group boundaries
              int jr = jb - j0;
#pragma unroll
              for (int m = 1; m <= kKPW / 16; ++m) jr += (o >= m * grp);
              const uint32_t v = lds_u16(srh + jr * BM * 2);
              sc[w] = prmt(v, v, 0x1010u);
            }
          }
          const uint32_t qbase = sb + s * Gm::STAGE + Gm::ACT_BYTES + h * Gm::CODE_HALF + row * Gm::CODE_BYTES_ROW;
          uint32_t out[kKPW / 2];
          if (FQ_TC_DBG & 2) {
          } else if (BITS == 4) {
            // kKPW/2 bytes of the swizzled code row
            constexpr int ROWB = Gm::CODE_BYTES_ROW;
            uint32_t words[NW];
            if constexpr (kKPW >= 32) {
#pragma unroll
              for (int i = 0; i < kKPW / 32; ++i) {
                const uint4 c = lds128(qbase + (swz_chunk<ROWB>(kp * (kKPW / 32) + i, row) << 4));
                words[4 * i] = c.x; words[4 * i + 1] = c.y; words[4 * i + 2] = c.z; words[4 * i + 3] = c.w;
              }
            } else {
              const uint2 c = lds64(qbase + (swz_chunk<ROWB>(kp >> 1, row) << 4) + (kp & 1) * 8);
              words[0] = c.x; words[1] = c.y;
            }
#pragma unroll
            for (int w = 0; w < NW; ++w) {
              uint32_t q[4];
              i4_nat_pairs<T>(words[w], q);
#pragma unroll
              for (int i = 0; i < 4; ++i) out[4 * w + i] = mul2x<T>(q[i], sc[w]);
            }
          } else {
            // kKPW bytes of the swizzled code row
#pragma unroll
            for (int hh = 0; hh < kKPW / 16; ++hh) {
              const int cidx = kp * (kKPW / 16) + hh;
              const uint4 c = lds128(qbase + (swz_chunk<Gm::CODE_BYTES_ROW>(cidx, row) << 4));
              const uint32_t words[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
              for (int w = 0; w < 4; ++w) {
                uint32_t q[2];
                i8_nat_pairs<T>(words[w], q);
                const uint32_t scw = sc[hh * 2 + (w >> 1)];
                out[8 * hh + 2 * w] = mul2x<T>(q[0], scw);
                out[8 * hh + 2 * w + 1] = mul2x<T>(q[1], scw);
              }
            }
          }
          // separate slot ring: the MMAs that last read this A slot must have completed
          if (kSepA && h == 0) {
            mbar_wait(&aempty_bar[slot], aph ^ 1);
            fence_after();
          }
          const uint32_t acol = tmem + lane_base + kACol + slot * Gm::A_COLS + h * Gm::A_HALF;
          if (FQ_TC_DBG & 2) {
          } else if constexpr (kKPW == 64)
            tmem_st32(acol + kp * 32, *reinterpret_cast<const uint32_t(*)[32]>(out));
          else if constexpr (kKPW == 32)
            tmem_st16(acol + kp * 16, *reinterpret_cast<const uint32_t(*)[16]>(out));
          else
            tmem_st8(acol + kp * 8, *reinterpret_cast<const uint32_t(*)[8]>(out));
        }
        tmem_wait_st();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&afull_bar[slot]);
        }
        ++blk;
        if (kSepA && ++a == ASLOTS) { a = 0; aph ^= 1; }
        if (++s == STAGES) { s = 0; ph ^= 1; }
        r0 += BK;
        while (r0 >= grp) { r0 -= grp; ++j0; }
        gk += BK;
        while (gk >= grp) { gk -= grp; ++jb; }
      }
      // ---- epilogue: accumulator row `row` (weight n), tokens [half*TPP, half*TPP+TPP)
      mbar_wait(&acc_full, acc_ph);
      acc_ph ^= 1;
      fence_after();
      constexpr int TPP = 256 / kParts;  // accumulator (token) columns drained per dequant warp
      const int tok_base = mt * p.bn + half * TPP;
      // split-K: this item's fp32 partial [bn][BMT] of output tile tt, slot ks
      float* part = p.splits > 1 ? p.ws + (size_t)(tt * p.splits + ks) * p.bn * BMT : nullptr;
#pragma unroll
      for (int h = 0; h < HM; ++h) {
        const int n = nt * BMT + h * BM + row;
        auto store = [&](int tok, float f) {
          if (p.cdt == FQ_FP32) reinterpret_cast<float*>(p.C)[(size_t)(row0 + tok) * N + n] = f;
          else reinterpret_cast<T*>(p.C)[(size_t)(row0 + tok) * N + n] = Dt<T>::from_f(f);
        };
#pragma unroll 1
        for (int c0 = 0; c0 < TPP && half * TPP + c0 < p.bn; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tmem + lane_base + kAccCol + h * BNMAX + half * TPP + c0, v);
          tmem_wait_ld();
          if (part) {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (half * TPP + c0 + i < p.bn)
                __stcg(part + (half * TPP + c0 + i) * BMT + h * BM + row, __uint_as_float(v[i]));
          } else if (n < N) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const int tok = tok_base + c0 + i;
              if (tok < M) store(tok, __uint_as_float(v[i]));
            }
          }
        }
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty);  // the accumulator is free for the next item
      if (part) {
        // last-arriving split of the tile sums the partials in split order (deterministic)
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kDqWarps));
        if (threadIdx.x == 64) {
          __threadfence();
          const int last = atomicAdd(&p.ctr[tt], 1) == p.splits - 1;
          if (last) __threadfence();
          s_last = last;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kDqWarps));
        if (s_last) {
          // thread -> (row = tid % BMT, tokens tid / BMT + NPAR i); 4 tokens per round so
          // their split loads are in flight together; rows are contiguous -> coalesced
          const float* base = p.ws + (size_t)tt * p.splits * p.bn * BMT;
          constexpr int NPAR = kDqWarps * 32 / BMT;  // threads per row
          static_assert(NPAR >= 1, "fixup: one thread per row at least");
          const int tid = threadIdx.x - 64, r = tid & (BMT - 1);
          const int nr = nt * BMT + r;
          const int tmax = min(p.bn, M - mt * p.bn);
          if (nr < N) {
            for (int tl0 = tid / BMT; tl0 < tmax; tl0 += 4 * NPAR) {
              float acc[4] = {0.f, 0.f, 0.f, 0.f};
              for (int q = 0; q < p.splits; ++q) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  const int tl = tl0 + NPAR * u;
                  if (tl < tmax) acc[u] += __ldcg(base + ((size_t)q * p.bn + tl) * BMT + r);
                }
              }
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int tl = tl0 + NPAR * u;
                if (tl < tmax) {
                  const size_t o = (size_t)(row0 + mt * p.bn + tl) * N + nr;
                  if (p.cdt == FQ_FP32) reinterpret_cast<float*>(p.C)[o] = acc[u];
                  else reinterpret_cast<T*>(p.C)[o] = Dt<T>::from_f(acc[u]);
                }
              }
            }
          }
          if (threadIdx.x == 64) p.ctr[tt] = 0;  // self-reset for the next launch
        }
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    fence_after();
    tmem_dealloc(tmem, Gm::TMEM);
  }
}

}  // namespace tc

// ------------------------------------------------------------------------------------- host side
// K per stage of the kernel variant serving a launch whose widest token tile is bnmax tokens:
// 128 for the 64/128-token variants (64-byte int4 code rows), 64 for the 256-token variant (its
// activation tiles leave no room for 128-k stages).
static int tc_bk(int bnmax) { return bnmax > 128 ? 64 : 128; }
// 128-row halves per tile (tile = 128 * hm weight rows) for the 64/128-token variants.  Two halves
// carry twice the code bytes per staged activation tile, which is what bounds the small-M regime;
// but with half as many tiles a matrix needs more K splits to fill the SMs, and short split items
// (pipeline fill + fixup, which stalls the dequant warps) lose more than the halves gain.  Measured
// (tools/tc_mid.py, tools/paper_microbench.py): two halves win for the MoE batch (M_e = 32 / 64 / 128:
// -20 / -28 / -17%) and for long-K matrices with fewer one-half tiles than SMs (OPT-175B FC2,
// M = 48..128: -30..-40%); they lose for OPT-175B FC1 (384 one-half tiles: +7..+16%) and for the
// OPT-13B/30B matrices (K <= 28672: split items of 5-40 K blocks, up to 1.9x slower).  Rule: two
// halves for MoE batches, and for a single GEMM when its one-half tiles do not fill the SMs and the
// two-half split plan keeps >= 64 K blocks (8192 k) per item.  Tune::hm = 1 | 2 overrides.
static int tc_bn(int M);
static int tc_splits_hm(int M, int K, int N, int bits, int hm, int* kbs_out, int forced_splits);
static int tc_bnmax(int bn) { return bn <= 32 ? 32 : bn <= 64 ? 64 : bn <= 128 ? 128 : 256; }
// persistent CTA slots of the variant serving token tiles of bn tokens
static int tc_slots(int bn, int bits, int hm) { (void)bn; (void)bits; (void)hm; return num_sms(); }
static bool tc_hm_ok(int bn, int bits) { (void)bits; return bn <= 128 && tc_bk(bn) == 128; }
// Two CTAs per SM (tc::Geo CPS = 2) for int4 one-half tiles of <= 64 tokens when the tiles fill the
// GPU without a K split: measured (profiles/r02/a6_two_ctas_per_sm.txt) OPT-175B FC1 M = 48 / 64
// 179 -> 140 us, OPT-30B QKV 78 -> 59 us, MoE g128 M_e = 64 1184 -> 1011 us; with a K split (few
// tiles: OPT-13B FFN2) the 16-warp single CTA stays faster.
static bool tc_use_cps2(int bn, int bits, int hm, long long items) {
  return FQ_TC_CPS_SMALL == 2 && bn <= 64 && bits == 4 && hm == 1 && items >= num_sms();
}
static int tc_hm_batch(int bnmax, int bits) {  // MoE batch: two CTAs per SM beat two halves at <= 64 tokens
  if (FQ_TC_CPS_SMALL == 2 && bnmax <= 64 && bits == 4) return 1;
  return tc_hm_ok(bnmax, bits) ? 2 : 1;
}
// Two CTAs per SM with a K split (one-half tiles that do not fill the GPU): only when every item
// keeps >= 64 K blocks, so the split fixup stays rare (OPT-175B FC2 M = 64: 141 -> 132 us; short
// items, e.g. OPT-13B FFN2, lose).  Returns the split count, 0 if the plan does not apply.
static int tc_cps2_split(int M, int K, int N, int bits, int* kbs_out) {
  const int bn = tc_bn(M);
  if (FQ_TC_CPS_SMALL != 2 || bn > 64 || bits != 4) return 0;
  const int tiles = ((M + bn - 1) / bn) * ((N + tc::BM - 1) / tc::BM);
  if (tiles >= num_sms()) return 0;  // no split needed: the plain two-CTA rule applies
  const int kblocks = (K + 127) / 128;
  const int s = std::max(1, std::min(kblocks, 2 * num_sms() / std::max(1, tiles)));
  const int kbs = (kblocks + s - 1) / s;
  if (kbs < 64) return 0;
  if (kbs_out) *kbs_out = kbs;
  return (kblocks + kbs - 1) / kbs;
}
static int tc_hm_gemm(int M, int K, int N, int bits, const Tune& tune) {
  const int bn = tc_bn(M);
  if (!tc_hm_ok(bn, bits)) return 1;
  if (tune.hm == 1 || tune.hm == 2) return tune.hm;
  if (tune.splits == 0 && tc_cps2_split(M, K, N, bits, nullptr) > 1) return 1;
  const long long tiles1 = (long long)((M + bn - 1) / bn) * ((N + tc::BM - 1) / tc::BM);
  if (tiles1 >= tc_slots(bn, bits, 1)) return 1;
  int kbs2 = 0;
  tc_splits_hm(M, K, N, bits, 2, &kbs2, 0);
  return kbs2 >= 64 ? 2 : 1;
}
static int tc_bn(int M) { return std::min(tc::BN, (M + 15) / 16 * 16); }

static bool make_tc_prob(tc::TcProb& d, int bits, const void* A, int M, int K, int N, const void* codes,
                         const void* scales, int group, void* C, int cdt, int bk, int hm) {
  d.bn = tc_bn(M);
  d.bk = bk;
  d.hm = hm;
  if (!make_tmap_2d(&d.a, A, 2, (uint64_t)K, (uint64_t)M, (uint64_t)K * 2, tc::BKA, d.bn, 128)) return false;
  const uint64_t row_bytes = (uint64_t)K * bits / 8;
  const int code_row = bk * bits / 8;  // box row bytes = swizzle span (32 / 64 / 128)
  if (!make_tmap_2d(&d.q, codes, 1, row_bytes, (uint64_t)N, row_bytes, code_row, tc::BM, code_row)) return false;
  if (!make_tmap_2d(&d.s, scales, 2, (uint64_t)N, (uint64_t)(K / group), (uint64_t)N * 2, tc::BM,
                    tc::sc_rows_max(bk), 0))
    return false;
  d.scales = scales;
  d.C = C;
  d.M = M; d.K = K; d.N = N; d.group = group; d.cdt = cdt;
  d.m_tiles = (M + d.bn - 1) / d.bn;
  d.n_tiles = (N + tc::BM * hm - 1) / (tc::BM * hm);
  d.gm = 8;
  d.splits = 1;
  d.kbs = (K + bk - 1) / bk;
  d.ws = nullptr;
  d.ctr = nullptr;
  return true;
}

// Split-K plan of one GEMM: when its output tiles cannot fill the SMs (e.g. M <= 256 on a weight
// matrix of < 148 x 128 rows), K is cut into ranges of >= 512 k so ~one work item per SM runs.
// Two-half tiles (fewer, larger tiles): the split count minimises (code bytes + partial traffic) /
// last-round efficiency of the persistent schedule, e.g. OPT-175B FC1 at M <= 64: 192 tiles on
// 148 SMs (65% in the last round) -> 3 splits (576 items, 97%) for 24% more traffic.
constexpr size_t kTcCounterBytes = 65536;
static int tc_splits_hm(int M, int K, int N, int bits, int hm, int* kbs_out, int forced_splits) {
  const int bn = tc_bn(M);
  const int bk = tc_bk(bn);
  const int tiles = ((M + bn - 1) / bn) * ((N + tc::BM * hm - 1) / (tc::BM * hm));
  const int kblocks = (K + bk - 1) / bk;
  const int smax = std::max(1, kblocks / (512 / bk));
  int s;
  if (forced_splits > 0) {
    s = forced_splits;
  } else if (hm == 1) {
    s = tc_slots(bn, bits, hm) / std::max(1, tiles);
  } else {
    const double code = (double)N * K * bits / 8;
    double best = 1e300;
    s = 1;
    for (int c = 1; c <= std::min(8, smax); ++c) {
      const int kbs = (kblocks + c - 1) / c, ce = (kblocks + kbs - 1) / kbs;
      const double items = (double)tiles * ce, rounds = items / tc_slots(bn, bits, hm);
      const double eff = rounds / std::ceil(rounds);
      const double part = ce > 1 ? 2.0 * items * bn * tc::BM * hm * sizeof(float) : 0.0;
      const double cost = (code + part) / eff;
      if (cost < best * 0.99) { best = cost; s = c; }
    }
  }
  s = std::max(1, std::min(s, smax));
  if (tiles > (int)(kTcCounterBytes / sizeof(int))) s = 1;
  const int kbs = (kblocks + s - 1) / s;
  if (kbs_out) *kbs_out = kbs;
  return (kblocks + kbs - 1) / kbs;
}
static int tc_splits(int M, int K, int N, int bits, const Tune& tune, int* kbs_out = nullptr) {
  const int hm = tc_hm_gemm(M, K, N, bits, tune);
  if (hm == 1 && tune.splits == 0) {
    const int s2 = tc_cps2_split(M, K, N, bits, kbs_out);
    if (s2 > 1) return s2;
  }
  return tc_splits_hm(M, K, N, bits, hm, kbs_out, tune.splits);
}
size_t gemm_tc_workspace_bytes(int M, int K, int N, int bits, const Tune& tune) {
  const int s = tc_splits(M, K, N, bits, tune);
  if (s == 1) return 256;
  const int bn = tc_bn(M);
  const int bmt = tc::BM * tc_hm_gemm(M, K, N, bits, tune);
  const size_t tiles = (size_t)((M + bn - 1) / bn) * ((N + bmt - 1) / bmt);
  return kTcCounterBytes + tiles * s * bn * bmt * sizeof(float);
}

template <typename T, int BITS, int MAXP, int BNMAX, int BK, int HM, int DQG, int CPS = 1>
static cudaError_t launch_tc(const tc::TcBatch<MAXP>& b, cudaStream_t st) {
  using Gm = tc::Geo<BITS, BNMAX, BK, HM, CPS>;
  auto kern = tc::gemm_tc_kernel<T, BITS, MAXP, BNMAX, BK, HM, DQG, CPS>;
  cudaError_t e = ensure_smem_attr<tc::gemm_tc_kernel<T, BITS, MAXP, BNMAX, BK, HM, DQG, CPS>>(Gm::SMEM);
  if (e != cudaSuccess) return e;
  const int grid = std::min(b.total_tiles, num_sms() * CPS);
  kern<<<grid, tc::tc_threads(BNMAX, CPS), Gm::SMEM, st>>>(b);
  return cudaGetLastError();
}

// dqg: dequant warp groups (2 = two groups of 8 warps on alternate K blocks; int4, 128-k stages,
// 16-warp variants only -- see the kernel).
template <int MAXP, int BNMAX, int BK, int HM = 1>
static cudaError_t dispatch_tc_bn(int adt, int bits, const tc::TcBatch<MAXP>& b, cudaStream_t st, int dqg = 1) {
  if (bits != 4 && bits != 8) return cudaErrorInvalidValue;  // int4 / int8 kernels only
  if constexpr (BK == 128 && tc::dq_warps(BNMAX) == 16) {
    if (dqg == 2 && bits == 4)
      return adt == FQ_BF16 ? launch_tc<__nv_bfloat16, 4, MAXP, BNMAX, BK, HM, 2>(b, st)
                            : launch_tc<__half, 4, MAXP, BNMAX, BK, HM, 2>(b, st);
  }
  if (adt == FQ_BF16)
    return bits == 4 ? launch_tc<__nv_bfloat16, 4, MAXP, BNMAX, BK, HM, 1>(b, st)
                     : launch_tc<__nv_bfloat16, 8, MAXP, BNMAX, BK, HM, 1>(b, st);
  return bits == 4 ? launch_tc<__half, 4, MAXP, BNMAX, BK, HM, 1>(b, st) : launch_tc<__half, 8, MAXP, BNMAX, BK, HM, 1>(b, st);
}
// kernel variant = the widest token tile of the launch (64 / 128 / 256 tokens) and the stage K its
// problems were prepared for
template <int MAXP>
static cudaError_t dispatch_tc(int adt, int bits, const tc::TcBatch<MAXP>& b, cudaStream_t st, int forced_dqg = 0) {
  int bn = 0;
  for (int i = 0; i < b.nprob; ++i) bn = std::max(bn, b.p[i].bn);
  bool split = false, short_items = false;
  for (int i = 0; i < b.nprob; ++i) {
    split |= b.p[i].splits > 1;
    short_items |= b.p[i].splits > 1 && b.p[i].kbs < 64;
  }
  const bool cps2 = split ? (FQ_TC_CPS_SMALL == 2 && bn <= 64 && bits == 4 && b.p[0].hm == 1 && !short_items)
                          : tc_use_cps2(bn, bits, b.p[0].hm, b.total_tiles);
  if (cps2 && b.p[0].bk == 128) {  // int4, one-half, <= 64 tokens
    const bool v32 = bn <= 32;
    if (adt == FQ_BF16)
      return v32 ? launch_tc<__nv_bfloat16, 4, MAXP, 32, 128, 1, 1, 2>(b, st)
                 : launch_tc<__nv_bfloat16, 4, MAXP, 64, 128, 1, 1, 2>(b, st);
    return v32 ? launch_tc<__half, 4, MAXP, 32, 128, 1, 1, 2>(b, st) : launch_tc<__half, 4, MAXP, 64, 128, 1, 1, 2>(b, st);
  }
  const int bk = b.p[0].bk, hm = b.p[0].hm;
  for (int i = 1; i < b.nprob; ++i)
    if (b.p[i].bk != bk || b.p[i].hm != hm) return cudaErrorInvalidValue;
  if (bn > 128) return (bk == 64 && hm == 1) ? dispatch_tc_bn<MAXP, 256, 64>(adt, bits, b, st) : cudaErrorInvalidValue;
  // <= 32-token variant: the small activation tile leaves room for more code stages in flight
  const bool v32 = bn <= 32 && bk == 128;
  // Two alternating dequant warp groups (each thread then covers 64 k of a block): measured
  // (profiles/r01/a6_two_half_tiles.txt) OPT-175B FC2 int4 M = 48..128 -8..-12%, FC1 int4 -1.5%,
  // MoE g128 -3%; but +10-13% on MoE batches with 16-element groups (8 scale words per thread) and
  // +5% on int8 FC1 -> int4 with every group a multiple of 64 only.  Tune::dqg = 1 | 2 overrides.
  int dqg = bits == 4 ? 2 : 1;
  for (int i = 0; i < b.nprob; ++i)
    if (b.p[i].group % 64) dqg = 1;
  if (forced_dqg) dqg = forced_dqg == 2 ? 2 : 1;
  if (hm == 2) {
    if (bk != 128) return cudaErrorInvalidValue;
    if (v32) return dispatch_tc_bn<MAXP, 32, 128, 2>(adt, bits, b, st, dqg);
    return bn <= 64 ? dispatch_tc_bn<MAXP, 64, 128, 2>(adt, bits, b, st, dqg)
                    : dispatch_tc_bn<MAXP, 128, 128, 2>(adt, bits, b, st, dqg);
  }
  if (v32) return dispatch_tc_bn<MAXP, 32, 128>(adt, bits, b, st, dqg);
  if (bn <= 64)
    return bk == 128 ? dispatch_tc_bn<MAXP, 64, 128>(adt, bits, b, st, dqg) : dispatch_tc_bn<MAXP, 64, 64>(adt, bits, b, st);
  return bk == 128 ? dispatch_tc_bn<MAXP, 128, 128>(adt, bits, b, st, dqg) : dispatch_tc_bn<MAXP, 128, 64>(adt, bits, b, st);
}

cudaError_t run_gemm_tc(int adt, int cdt, int bits, const void* A, int M, int K, int N, const void* codes,
                        const void* scales, int group, void* C, void* ws, size_t ws_bytes, cudaStream_t st,
                        const Tune& tune) {
  tc::TcBatch<1> b{};
  tc::TcProb& d = b.p[0];
  if (!make_tc_prob(d, bits, A, M, K, N, codes, scales, group, C, cdt, tc_bk(tc_bn(M)),
                    tc_hm_gemm(M, K, N, bits, tune)))
    return cudaErrorInvalidValue;
  int kbs = 0;
  const int s = tc_splits(M, K, N, bits, tune, &kbs);
  if (s > 1 && ws && ws_bytes >= gemm_tc_workspace_bytes(M, K, N, bits, tune)) {
    d.kbs = kbs;
    d.splits = s;
    d.ctr = reinterpret_cast<int*>(ws);
    d.ws = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + kTcCounterBytes);
  }
  d.tile_begin = 0;
  b.nprob = 1;
  b.total_tiles = d.m_tiles * d.n_tiles * d.splits;
  return dispatch_tc<1>(adt, bits, b, st, tune.dqg);
}

// MoE with DEVICE expert offsets (fq_gemm_grouped_dev): every listed expert is laid out for `Mmax`
// tokens; tiles beyond an expert's device token count are skipped by all warps of the CTA.
cudaError_t run_gemm_tc_grouped_dev(int adt, int cdt, int bits, const void* A, int64_t T, int K, int N,
                                    const int64_t* offs_dev, const int32_t* groups, const void* const* codes,
                                    const void* const* scales, void* C, int Mmax, const int* experts, int nexp,
                                    const int* skips, int32_t* status, cudaStream_t st) {
  constexpr int MAXP = 48;
  tc::TcBatch<MAXP> b{};
  int mmax = 1;  // one tile geometry for the launch: the largest token range left to this kernel
  for (int ii = 0; ii < nexp; ++ii) mmax = std::max(mmax, Mmax - skips[ii]);
  const int bn = tc_bn(mmax), bk = tc_bk(bn), hm = tc_hm_batch(bn, bits);
  for (int ii = 0; ii < nexp; ++ii) {
    const int e = experts[ii];
    tc::TcProb& d = b.p[b.nprob];
    if (!make_tc_prob(d, bits, A, Mmax - skips[ii], K, N, codes[e], scales[e], groups[e], C, cdt, bk, hm))
      return cudaErrorInvalidValue;
    d.skip = skips[ii];
    d.gm = 1;  // token tiles slowest: an expert's live tiles (its first ones) stay contiguous, so the
               // persistent CTAs' strided schedule spreads them instead of collecting them on a few
    if (!make_tmap_2d(&d.a, A, 2, (uint64_t)K, (uint64_t)T, (uint64_t)K * 2, tc::BKA, d.bn, 128))  // all T rows
      return cudaErrorInvalidValue;
    d.offs = offs_dev;
    d.e = e;
    d.rows = (int)T;
    d.status = status;
    d.tile_begin = b.total_tiles;
    b.total_tiles += d.m_tiles * d.n_tiles;
    if (++b.nprob == MAXP) {
      cudaError_t r = dispatch_tc<MAXP>(adt, bits, b, st);
      if (r != cudaSuccess) return r;
      b.nprob = 0;
      b.total_tiles = 0;
    }
  }
  if (b.nprob) return dispatch_tc<MAXP>(adt, bits, b, st);
  return cudaSuccess;
}

// MoE: every listed expert (M_e > 16) in one persistent launch per <= 48 experts.
cudaError_t run_gemm_tc_grouped(int adt, int cdt, int bits, const void* A, int K, int N, const int64_t* offsets,
                                const int32_t* groups, const void* const* codes, const void* const* scales,
                                void* C, const int* experts, int nexp, cudaStream_t st) {
  constexpr int MAXP = 48;
  static_assert(sizeof(tc::TcBatch<MAXP>) < 32000, "kernel parameter block limit");
  tc::TcBatch<MAXP> b{};
  int bnmax = 0;  // one stage K for every launch of the call (all chunks fit its variant)
  for (int ii = 0; ii < nexp; ++ii)
    bnmax = std::max(bnmax, tc_bn((int)(offsets[experts[ii] + 1] - offsets[experts[ii]])));
  const int bk = tc_bk(bnmax), hm = tc_hm_batch(bnmax, bits);
  for (int ii = 0; ii < nexp; ++ii) {
    const int e = experts[ii];
    const int Me = (int)(offsets[e + 1] - offsets[e]);
    const char* Ae = reinterpret_cast<const char*>(A) + (size_t)offsets[e] * K * 2;
    char* Ce = reinterpret_cast<char*>(C) + (size_t)offsets[e] * N * (cdt == FQ_FP32 ? 4 : 2);
    tc::TcProb& d = b.p[b.nprob];
    if (!make_tc_prob(d, bits, Ae, Me, K, N, codes[e], scales[e], groups[e], Ce, cdt, bk, hm)) return cudaErrorInvalidValue;
    d.tile_begin = b.total_tiles;
    b.total_tiles += d.m_tiles * d.n_tiles;
    if (++b.nprob == MAXP) {
      cudaError_t r = dispatch_tc<MAXP>(adt, bits, b, st);
      if (r != cudaSuccess) return r;
      b.nprob = 0;
      b.total_tiles = 0;
    }
  }
  if (b.nprob) return dispatch_tc<MAXP>(adt, bits, b, st);
  return cudaSuccess;
}

}  // namespace fq
