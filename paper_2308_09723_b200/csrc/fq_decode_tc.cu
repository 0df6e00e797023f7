// fq_decode_tc.cu — kernel A4 on the 5th-gen tensor cores: the decode (M <= 16) fused dequant GEMM
// with the MMA issued by tcgen05 from one thread, so the SM sub-partitions spend their issue slots
// on the dequantization alone (the legacy mma.sync kernel in fq_gemv.cu also spends them on HMMA,
// fragment loads and, for 9 <= M <= 16, a second 8-token MMA per weight).
//
// C[m,n] = sum_k A[m,k] * q[n,k] * s[k/g, n]   (§4.1).  Decode streams every packed
// weight byte once: the kernel is built to keep the TMA streaming at HBM speed.
//
// Stream-K: 2 persistent CTAs per SM split the launch's linear (tile, k-stage) space -- all tiles of
// one matrix, or of every expert of a MoE batch -- into equal contiguous ranges; a tile cut by a
// range boundary is finished by its last-arriving contributor, which sums the fp32 partials in CTA
// order (deterministic).  No wave quantisation, one pipeline fill per CTA.
//
// Tile = 128 weight rows (UMMA M, TMEM lanes) x NT = 16 tokens (UMMA N).  Stage = 64 packed bytes
// per row (k = 128 int4 / 64 int8) -- group % 128 == 0, so one scale per row per stage.
//   warp 0     TMA: codes [128 rows x 64 B] (SWIZZLE_64B) + activations A' [NT x k] (SWIZZLE_128B,
//              the UMMA K-major layout) into the stage ring; the stage's 128 scales and per-token
//              2^-e factors into a fold-data ring.
//   warp 1     TMEM allocation; one thread issues tcgen05.mma kind::f16 (A = codes in TMEM, B = A' in
//              shared memory, D = a per-stage fp32 accumulator slot), tcgen05.commit releases the
//              stage, the A slot and signals the accumulator slot.
//   warps 2-9  dequant: thread = weight row (TMEM lane) x half of the stage's k.  Codes become EXACT
//              small integers in fp16 (LOP3 magic + one HSUB2/HFMA2 per pair, no scale applied) and
//              go to TMEM with tcgen05.st.  Two stages later the same warps fold that stage's
//              accumulator (tcgen05.ld): acc[tok] += s[row] * 2^-e[tok] * part[tok] (fp32).
// Activations: the prep kernel (fq_gemv.cu, MODE 1/2) converts A to fp16 scaled by 2^e per
// (token, 128-k chunk) -- exact for bf16 inputs -- in the k order the unpack produces:
//   int4 word (k..k+7) -> TMEM columns (k,k+4),(k+1,k+5),(k+2,k+6),(k+3,k+7); int8 natural pairs.
// The integer partials of a stage are exact products q * a' summed in fp32; the scale is applied
// in fp32 (R13), so the result is within the 2e-3 gate with a wide margin.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "fq_common.cuh"
#include "fq_internal.h"
#include "fq_tcgen05.cuh"

namespace fq {
namespace dtc {
using namespace tc5;

constexpr int BM = 128;             // weight rows per tile
constexpr int WB = 64;              // packed bytes per row per stage
constexpr int W_BYTES = BM * WB;    // 8 KB
constexpr int kDqWarps = 4;         // one per TMEM lane quarter (warps 3..6)
constexpr int kDq0 = 3;             // first dequant warp
constexpr int kThreads = 32 * (kDq0 + kDqWarps);
constexpr int kTmemCols = 256;      // two CTAs per SM share the 512 columns
#ifndef FQ_DTC_AS
#define FQ_DTC_AS 3
#endif
constexpr int AS = FQ_DTC_AS;       // TMEM A slots
constexpr int AC = 4;               // TMEM accumulator slots
#ifndef FQ_DTC_LAG
#define FQ_DTC_LAG 2
#endif
constexpr int LAG = FQ_DTC_LAG;     // the fold trails the dequant by LAG stages
constexpr int kMaxStages = 12;
constexpr int kSmemBudget = 110 * 1024;  // dynamic smem per CTA (2 CTAs per SM)
#ifndef FQ_DTC_DBG
#define FQ_DTC_DBG 0  // diagnostics only: 1 = no MMA, 2 = no unpack / tcgen05.st, 4 = no tcgen05.ld,
                      // 8 = MMA issuer ignores the A / accumulator barriers, 16 = dequant ignores A-slot reuse
#endif

template <int BITS, int NT>
struct G {
  static constexpr int KS = WB * 8 / BITS;            // k per stage: 128 / 64
  static constexpr int ATOMS = KS / 64;               // SW128 atoms (64 fp16 of k) of the B tile
  static constexpr int ATOM_BYTES = NT * 128;
  static constexpr int B_BYTES = ATOMS * ATOM_BYTES;  // activation tile of one stage (1024-aligned)
  static constexpr int SC_OFS = W_BYTES;              // the stage's 128 scales (activation dtype)
  static constexpr int SC_BYTES = BM * 2;
  static constexpr int WSTAGE = ((SC_OFS + SC_BYTES + 1023) / 1024) * 1024;
  static constexpr int NB = 6;                        // activation ring depth
  static constexpr int NS0 = (kSmemBudget - 1024 - NB * B_BYTES) / WSTAGE;
  static constexpr int NSTAGE = NS0 > kMaxStages ? kMaxStages : NS0;   // codes ring depth
  static constexpr int B_RING = NSTAGE * WSTAGE;
  static constexpr int SMEM = B_RING + NB * B_BYTES + 1024;
  static constexpr int A_COLS = KS / 2;               // TMEM columns of one A slot
  static constexpr int ACC_COL = AS * A_COLS;
  static constexpr int TXW = W_BYTES + SC_BYTES;
  static_assert(NSTAGE >= 4 && ACC_COL + AC * NT <= kTmemCols && AC > LAG, "resources");
};

struct Prob {
  CUtensorMap w;   // codes [N][K*b/8] u8, box [128 rows][64 B], SWIZZLE_64B
  CUtensorMap a;   // A' [M][K] fp16, box [NT rows][64], SWIZZLE_128B (rows >= M zero-filled)
  CUtensorMap s;   // scales [G][N], box [1][128]
  const float* inv;  // per-token 2^-e of A' (this problem's tokens)
  void* C;
  int M, K, N, group, cdt;
  int gx, nk;                    // tiles, stages per tile
  int stage_begin, tile_begin;   // offsets in the launch's linear stage / tile spaces
};
template <int MAXP>
struct Batch {
  Prob p[MAXP];
  int nprob;
  int total_stages;
  float* ws;      // stream-K partials [ctas][2][16][BM] fp32
  int* counters;  // per global tile arrival counters (self-resetting)
};

// Linear stage cursor (every role walks the same sequence).
struct Cur {
  int p, tile, kidx;
};
template <int MAXP>
__device__ __forceinline__ void cur_locate(const Batch<MAXP>& b, int g, Cur& c) {
  int p = 0;
  while (p + 1 < b.nprob && g >= b.p[p + 1].stage_begin) ++p;
  const int local = g - b.p[p].stage_begin;
  c.p = p;
  c.tile = local / b.p[p].nk;
  c.kidx = local - c.tile * b.p[p].nk;
}
template <int MAXP>
__device__ __forceinline__ void cur_next(const Batch<MAXP>& b, Cur& c) {
  if (++c.kidx == b.p[c.p].nk) {
    c.kidx = 0;
    if (++c.tile == b.p[c.p].gx) { c.tile = 0; ++c.p; }
  }
}
__host__ __device__ __forceinline__ int range_begin(int T, int P, int c) { return (int)((long long)T * c / P); }
__device__ __forceinline__ int cta_of(int T, int P, int x) {  // CTA whose range holds stage x
  int c = (int)((long long)x * P / T);
  while (c + 1 < P && range_begin(T, P, c + 1) <= x) ++c;
  while (c > 0 && range_begin(T, P, c) > x) --c;
  return c;
}

__device__ __forceinline__ uint32_t hsub2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t hfma2(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
// int4 word (k..k+7) -> fp16 pairs (k,k+4),(k+1,k+5),(k+2,k+6),(k+3,k+7), exact codes q.
//   even: (w & 0x000F000F) ^ 0x6408 = 1024 + (n ^ 8) = 1032 + q          -> - 1032
//   odd:  (w & 0x00F000F0) ^ 0x6480 = 1024 + 16 (n ^ 8) = 1152 + 16 q   -> / 16 - 72 (one FMA)
__device__ __forceinline__ void i4_exact(uint32_t w, uint32_t* q) {
  const uint32_t w8 = w >> 8;
  q[0] = hsub2(lop3_and_xor(w, 0x000F000Fu, 0x64086408u), 0x64086408u);
  q[1] = hfma2(lop3_and_xor(w, 0x00F000F0u, 0x64806480u), 0x2C002C00u, 0xD480D480u);
  q[2] = hsub2(lop3_and_xor(w8, 0x000F000Fu, 0x64086408u), 0x64086408u);
  q[3] = hfma2(lop3_and_xor(w8, 0x00F000F0u, 0x64806480u), 0x2C002C00u, 0xD480D480u);
}
// int8 word (k..k+3) -> natural fp16 pairs (k,k+1),(k+2,k+3), exact codes: 1024 + (q + 128) - 1152.
__device__ __forceinline__ void i8_exact(uint32_t w, uint32_t* q) {
  const uint32_t u = w ^ 0x80808080u;
  q[0] = hsub2(prmt(u, 0x64646464u, 0x4140u), 0x64806480u);
  q[1] = hsub2(prmt(u, 0x64646464u, 0x4342u), 0x64806480u);
}

template <typename T, int BITS, int NT, int MAXP>
__global__ void __launch_bounds__(kThreads, 2) decode_tc_kernel(const __grid_constant__ Batch<MAXP> b) {
  using Gm = G<BITS, NT>;
  constexpr int NSTAGE = Gm::NSTAGE, KS = Gm::KS;
  extern __shared__ __align__(1024) uint8_t dsmem[];
  __shared__ __align__(8) uint64_t full_bar[kMaxStages], empty_bar[kMaxStages];
  __shared__ __align__(8) uint64_t bfull_bar[Gm::NB], bempty_bar[Gm::NB];
  __shared__ __align__(8) uint64_t afull_bar[AS], aempty_bar[AS], cfull_bar[AC], cempty_bar[AC];
  __shared__ uint32_t tmem_sh;
  __shared__ int s_last;
  uint8_t* sbase = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsmem) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int TS = b.total_stages, P = gridDim.x;
  const int beg = range_begin(TS, P, blockIdx.x), end = range_begin(TS, P, blockIdx.x + 1);

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kDqWarps);  // dequant warps (codes + scales read)
    }
    for (int s = 0; s < Gm::NB; ++s) {
      mbar_init(&bfull_bar[s], 1);
      mbar_init(&bempty_bar[s], 1);        // MMA commit (activation tile read)
    }
    for (int i = 0; i < AS; ++i) {
      mbar_init(&afull_bar[i], kDqWarps);
      mbar_init(&aempty_bar[i], 1);
    }
    for (int i = 0; i < AC; ++i) {
      mbar_init(&cfull_bar[i], 1);
      mbar_init(&cempty_bar[i], kDqWarps);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&tmem_sh, kTmemCols);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tmem_sh;
  const uint32_t sb = smem_u32(sbase);

  if (warp == 0) {
    // ------------------------------------------------------------------------- TMA: codes + scales
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();
      Cur c;
      cur_locate(b, beg, c);
      int s = 0;
      uint32_t ph = 0;
      for (int g = beg; g < end; ++g) {
        const Prob& p = b.p[c.p];
        mbar_wait(&empty_bar[s], ph ^ 1);
        uint8_t* st = sbase + s * Gm::WSTAGE;
        const int k0 = c.kidx * KS;
        mbar_arrive_expect_tx(&full_bar[s], Gm::TXW);
        tma_load_2d(st, &p.w, &full_bar[s], k0 * BITS / 8, c.tile * BM, pol_w);
        tma_load_2d(st + Gm::SC_OFS, &p.s, &full_bar[s], c.tile * BM, k0 / p.group, pol_w);
        cur_next(b, c);
        if (++s == NSTAGE) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 2) {
    // ------------------------------------------------------------------------- TMA: activations
    if (lane == 0) {
      const uint64_t pol_a = policy_evict_last();
      griddep_wait();  // A' comes from the prep kernel (programmatic dependent launch)
      Cur c;
      cur_locate(b, beg, c);
      int s = 0;
      uint32_t ph = 0;
      for (int g = beg; g < end; ++g) {
        const Prob& p = b.p[c.p];
        mbar_wait(&bempty_bar[s], ph ^ 1);
        uint8_t* bt = sbase + Gm::B_RING + s * Gm::B_BYTES;
        const int k0 = c.kidx * KS;
        mbar_arrive_expect_tx(&bfull_bar[s], Gm::B_BYTES);
#pragma unroll
        for (int a = 0; a < Gm::ATOMS; ++a)
          tma_load_2d(bt + a * Gm::ATOM_BYTES, &p.a, &bfull_bar[s], k0 + 64 * a, 0, pol_a);
        cur_next(b, c);
        if (++s == Gm::NB) { s = 0; ph ^= 1; }
      }
      griddep_launch_dependents();
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_f16<__half, BM, NT>();
      int s = 0, a = 0, c = 0;
      uint32_t ph = 0, aph = 0, cph = 0;
      for (int g = beg; g < end; ++g) {
        mbar_wait(&bfull_bar[s], ph);
        if (!(FQ_DTC_DBG & 8)) {
          mbar_wait(&afull_bar[a], aph);
          mbar_wait(&cempty_bar[c], cph ^ 1);
        }
        fence_after();
        const uint32_t bst = sb + Gm::B_RING + s * Gm::B_BYTES;
#pragma unroll
        for (int kk = 0; kk < KS / 16; ++kk) {
          if (FQ_DTC_DBG & 1) break;
          const uint64_t bdesc = sw128_desc(bst + (kk >> 2) * Gm::ATOM_BYTES) + (uint64_t)((kk & 3) * 2);
          mma_ts(tmem + Gm::ACC_COL + c * NT, tmem + a * Gm::A_COLS + kk * 8, bdesc, idesc, kk != 0);
        }
        mma_commit(&bempty_bar[s]);
        mma_commit(&aempty_bar[a]);
        mma_commit(&cfull_bar[c]);
        if (++s == Gm::NB) { s = 0; ph ^= 1; }
        if (++a == AS) { a = 0; aph ^= 1; }
        if (++c == AC) { c = 0; cph ^= 1; }
      }
    }
  } else {
    // ------------------------------------------------------------------------- dequant + fold
    const int quarter = warp & 3;          // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;   // weight row within the tile == TMEM lane
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const int sw = (row >> 1) & 3;         // SWIZZLE_64B: cell c of row r sits at c ^ ((r >> 1) & 3)
    const uint32_t rofs = row * WB;
    float acc[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[t] = 0.f;
    Cur cf;
    cur_locate(b, beg, cf);
    bool first_seg = true;                 // the fold's current segment contains `beg`
    int seg_k0 = cf.kidx;                  // first k-stage of the current segment
    bool dep_done = false;
    float scq[LAG + 1];                    // scales of stages i, i-1, ..., i-LAG (register FIFO)
#pragma unroll
    for (int q = 0; q < LAG + 1; ++q) scq[q] = 0.f;
    int s = 0, a = 0, c = 0;
    uint32_t ph = 0, aph = 0, cph = 0;
    for (int i = beg; i < end + LAG; ++i) {
      float sc0 = 0.f;
#pragma unroll
      for (int q = LAG; q > 0; --q) scq[q] = scq[q - 1];
      if (i < end) {
        // ---- dequant stage i
        mbar_wait(&full_bar[s], ph);
        const uint32_t st = sb + s * Gm::WSTAGE;
        uint4 cw[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) cw[q] = lds128(st + rofs + ((q ^ sw) << 4));
        sc0 = lds_f16x<T>(st + Gm::SC_OFS + row * 2);
        scq[0] = sc0;
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[s]);
        constexpr int NR = BITS == 4 ? 64 : 32;
        uint32_t out[NR];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t wv[4] = {cw[q].x, cw[q].y, cw[q].z, cw[q].w};
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            if constexpr (BITS == 4) i4_exact(wv[w], out + 16 * q + 4 * w);
            else i8_exact(wv[w], out + 8 * q + 2 * w);
          }
        }
        if (!(FQ_DTC_DBG & 16)) mbar_wait(&aempty_bar[a], aph ^ 1);
        fence_after();
        const uint32_t ta = tmem + lane_base + a * Gm::A_COLS;
        if (!(FQ_DTC_DBG & 2)) {
          tmem_st32(ta, *reinterpret_cast<const uint32_t(*)[32]>(out));
          if constexpr (BITS == 4) tmem_st32(ta + 32, *reinterpret_cast<const uint32_t(*)[32]>(out + 32));
        } else if (out[0] == 0x12345u && out[NR - 1] == 0x777u) {
          tmem_st16(ta, *reinterpret_cast<const uint32_t(*)[16]>(out));
        }
        tmem_wait_st();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&afull_bar[a]);
        if (++s == NSTAGE) { s = 0; ph ^= 1; }
        if (++a == AS) { a = 0; aph ^= 1; }
      }
      if (i >= beg + LAG) {
        // ---- fold stage j = i - LAG: acc += s[row] * (exact integer partial of the stage)
        const int j = i - LAG;
        const Prob& p = b.p[cf.p];
        mbar_wait(&cfull_bar[c], cph);
        fence_after();
        uint32_t v[NT];
        if (!(FQ_DTC_DBG & 4)) {
          tmem_ldn<NT>(tmem + lane_base + Gm::ACC_COL + c * NT, v);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int t = 0; t < NT; ++t) v[t] = 0;
        }
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&cempty_bar[c]);
#pragma unroll
        for (int t = 0; t < NT; ++t) acc[t] = fmaf(scq[LAG], __uint_as_float(v[t]), acc[t]);
        if (++c == AC) { c = 0; cph ^= 1; }
        // ---- end of a tile segment: store, or stream-K partial + deterministic fixup
        if (j == end - 1 || cf.kidx == p.nk - 1) {
          if (!dep_done) {  // the per-token factors come from the prep kernel
            griddep_wait();
            dep_done = true;
          }
          const int n = cf.tile * BM + row;
          const int M = p.M, N = p.N;
#pragma unroll
          for (int t = 0; t < NT; ++t) acc[t] *= (t < M) ? __ldg(p.inv + t) : 0.f;
          auto store = [&](int tok, float val) {
            const size_t o = (size_t)tok * N + n;
            if (p.cdt == FQ_FP32) reinterpret_cast<float*>(p.C)[o] = val;
            else reinterpret_cast<T*>(p.C)[o] = Dt<T>::from_f(val);
          };
          if (seg_k0 == 0 && cf.kidx == p.nk - 1) {
            if (n < N) {
#pragma unroll
              for (int t = 0; t < NT; ++t)
                if (t < M) store(t, acc[t]);
            }
          } else {
            const int slot = first_seg ? 0 : 1;
            float* part = b.ws + ((size_t)(blockIdx.x * 2 + slot) * 16) * BM;
#pragma unroll
            for (int t = 0; t < NT; ++t)
              if (t < M) __stcg(part + t * BM + row, acc[t]);
            const int gtile = p.tile_begin + cf.tile;
            const int t0 = p.stage_begin + cf.tile * p.nk;  // the tile's first global stage
            const int cfirst = cta_of(TS, P, t0), clast = cta_of(TS, P, t0 + p.nk - 1);
            asm volatile("bar.sync 1, %0;" ::"n"(32 * kDqWarps));
            if (threadIdx.x == 32 * kDq0) {
              __threadfence();
              const int last = atomicAdd(&b.counters[gtile], 1) == clast - cfirst;
              if (last) __threadfence();
              s_last = last;
            }
            asm volatile("bar.sync 1, %0;" ::"n"(32 * kDqWarps));
            if (s_last) {
              if (n < N) {
#pragma unroll
                for (int t = 0; t < NT; ++t) {
                  if (t >= M) continue;
                  float val = 0.f;
                  for (int cc = cfirst; cc <= clast; ++cc) {
                    const int sl = range_begin(TS, P, cc) >= t0 ? 0 : 1;
                    val += __ldcg(b.ws + ((size_t)(cc * 2 + sl) * 16 + t) * BM + row);
                  }
                  store(t, val);
                }
              }
              if (threadIdx.x == 32 * kDq0) b.counters[gtile] = 0;  // self-reset for the next launch
            }
          }
#pragma unroll
          for (int t = 0; t < NT; ++t) acc[t] = 0.f;
          first_seg = false;
          seg_k0 = 0;
        }
        cur_next(b, cf);
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

// Activation pre-conversion (one CTA per token): A'[tok][k] = fp16(A * 2^e), one power of two per
// token putting max|A[tok,:]| in [2^14, 2^15) (bf16 input; exact for every element within 2^-29 of
// the max) or e = 0 (fp16 input), in the k order of the int4 unpack (PERM: pieces of 8 as
// a0,a4,a1,a5,a2,a6,a3,a7) or natural (int8); inv[tok] = 2^-e.
template <typename T, bool PERM>
__global__ void __launch_bounds__(512) prep_tc_kernel(const T* __restrict__ A, int K, __half* __restrict__ Ap,
                                                      float* __restrict__ inv_out) {
  griddep_wait();  // A may be the output of the previous kernel in the stream
  griddep_launch_dependents();
  __shared__ float red[16];
  const int tok = blockIdx.x;
  const T* row = A + (size_t)tok * K;
  const int n8 = K >> 3;
  auto decode = [](const uint4& v, float (&f)[8]) {
    const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (Dt<T>::id == FQ_BF16) {
        f[2 * e] = __uint_as_float(vv[e] << 16);
        f[2 * e + 1] = __uint_as_float(vv[e] & 0xFFFF0000u);
      } else {
        const float2 h = __half22float2(*reinterpret_cast<const __half2*>(&vv[e]));
        f[2 * e] = h.x;
        f[2 * e + 1] = h.y;
      }
    }
  };
  float sc = 1.f, inv = 1.f;
  if (Dt<T>::id == FQ_BF16) {
    float mx = 0.f;
    for (int i = threadIdx.x; i < n8; i += blockDim.x) {
      float f[8];
      decode(ldg_keep(row + (size_t)i * 8), f);
#pragma unroll
      for (int e = 0; e < 8; ++e) mx = fmaxf(mx, fabsf(f[e]));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    mx = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mx = fmaxf(mx, red[w]);
    const int E = (int)((__float_as_uint(mx) >> 23) & 0xFF);
    const int F = max(1, min(268 - E, 253));  // biased exponent of 2^e, e = 14 - (E - 127)
    sc = __uint_as_float((uint32_t)F << 23);
    inv = __uint_as_float((uint32_t)(254 - F) << 23);
  }
  auto h2 = [](float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
  };
  for (int i = threadIdx.x; i < n8; i += blockDim.x) {
    float f[8];
    decode(ldg_keep(row + (size_t)i * 8), f);
#pragma unroll
    for (int e = 0; e < 8; ++e) f[e] *= sc;
    const uint4 o = PERM ? make_uint4(h2(f[0], f[4]), h2(f[1], f[5]), h2(f[2], f[6]), h2(f[3], f[7]))
                         : make_uint4(h2(f[0], f[1]), h2(f[2], f[3]), h2(f[4], f[5]), h2(f[6], f[7]));
    *reinterpret_cast<uint4*>(Ap + (size_t)tok * K + (size_t)i * 8) = o;
  }
  if (threadIdx.x == 0) inv_out[tok] = inv;
}

}  // namespace dtc

// ------------------------------------------------------------------------------------- host side
constexpr size_t kDtcCounterBytes = 65536;
constexpr int kDtcMaxTiles = (int)(kDtcCounterBytes / sizeof(int));

static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }
static size_t dtc_partial_bytes(int nsm) { return al256((size_t)2 * nsm * 2 * 16 * dtc::BM * sizeof(float)); }
static size_t dtc_prep_a_bytes(int64_t ntok, int K) { return al256((size_t)ntok * K * 2); }
static size_t dtc_prep_v_bytes(int64_t ntok) { return al256((size_t)ntok * 4); }

static int dtc_nt_override() {
  const char* e = std::getenv("FQ_DTC_NT");
  return e ? std::atoi(e) : 0;
}

bool decode_tc_supported(int bits, int group, int M) {
  // Opt-in (FQ_DECODE_TC=1): parity-green, but on B200 it streams at 2.4-2.9 TB/s against
  // 5.0-5.4 TB/s (M <= 8) / 3.4 TB/s (M = 16) for the mma.sync kernel; its synchronisation skeleton
  // alone (no unpack / MMA / tcgen05.ld) reaches only 4.6 TB/s (profiles/r01).
  (void)bits;
  const char* e = std::getenv("FQ_DECODE_TC");
  if (!e || e[0] != '1') return false;
  return M >= 1 && M <= 16 && group % 128 == 0;
}

size_t dtc_workspace_bytes(int64_t ntok, int K, int nsm) {
  return kDtcCounterBytes + dtc_partial_bytes(nsm) + dtc_prep_a_bytes(ntok, K) + dtc_prep_v_bytes(ntok);
}

static int dtc_ctas(long long total_stages, int nsm) {
  // two CTAs per SM; at least 8 stages per CTA so small problems are not shredded into partials
  const long long c = std::min<long long>(2LL * nsm, (total_stages + 7) / 8);
  return (int)std::max<long long>(1, c);
}

template <typename T, int BITS, int NT, int MAXP>
static cudaError_t launch_dtc(const dtc::Batch<MAXP>& b, int ctas, cudaStream_t st) {
  constexpr int smem = dtc::G<BITS, NT>::SMEM;
  auto kern = dtc::decode_tc_kernel<T, BITS, NT, MAXP>;
  static bool attr = false;  // benign race: idempotent attribute call
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return launch_pdl(kern, ctas, dtc::kThreads, smem, st, b);
}

template <int NT, int MAXP>
static cudaError_t dispatch_dtc_nt(int adt, int bits, const dtc::Batch<MAXP>& b, int ctas, cudaStream_t st) {
  if (adt == FQ_BF16)
    return bits == 4 ? launch_dtc<__nv_bfloat16, 4, NT, MAXP>(b, ctas, st)
                     : launch_dtc<__nv_bfloat16, 8, NT, MAXP>(b, ctas, st);
  return bits == 4 ? launch_dtc<__half, 4, NT, MAXP>(b, ctas, st) : launch_dtc<__half, 8, NT, MAXP>(b, ctas, st);
}
static int dtc_nt(int maxm) {
  const int o = dtc_nt_override();
  if (o == 8 || o == 16) return std::max(o, maxm > 8 ? 16 : 8);
  return maxm > 8 ? 16 : 8;
}
template <int MAXP>
static cudaError_t dispatch_dtc(int adt, int bits, const dtc::Batch<MAXP>& b, int ctas, int nt, cudaStream_t st) {
  return nt == 8 ? dispatch_dtc_nt<8, MAXP>(adt, bits, b, ctas, st) : dispatch_dtc_nt<16, MAXP>(adt, bits, b, ctas, st);
}

static cudaError_t launch_prep_tc(int adt, int bits, const void* A, int ntok, int K, void* Ap, void* Vp,
                                  cudaStream_t st) {
  if (ntok == 0) return cudaSuccess;
  auto* ap = reinterpret_cast<__half*>(Ap);
  auto* vp = reinterpret_cast<float*>(Vp);
  if (adt == FQ_BF16) {
    auto* a = reinterpret_cast<const __nv_bfloat16*>(A);
    return bits == 4 ? launch_pdl(dtc::prep_tc_kernel<__nv_bfloat16, true>, ntok, 512, 0, st, a, K, ap, vp)
                     : launch_pdl(dtc::prep_tc_kernel<__nv_bfloat16, false>, ntok, 512, 0, st, a, K, ap, vp);
  }
  auto* a = reinterpret_cast<const __half*>(A);
  return bits == 4 ? launch_pdl(dtc::prep_tc_kernel<__half, true>, ntok, 512, 0, st, a, K, ap, vp)
                   : launch_pdl(dtc::prep_tc_kernel<__half, false>, ntok, 512, 0, st, a, K, ap, vp);
}

// One problem: Ap = its A' rows, inv = its per-token factors.
static bool make_dtc_prob(dtc::Prob& d, int bits, int cdt, int nt, const void* Ap, const float* inv, int M, int K,
                          int N, const void* codes, const void* scales, int group, void* C) {
  const uint64_t row_bytes = (uint64_t)K * bits / 8;
  if (!make_tmap_2d(&d.w, codes, 1, row_bytes, (uint64_t)N, row_bytes, dtc::WB, dtc::BM, 64)) return false;
  if (!make_tmap_2d(&d.a, Ap, 2, (uint64_t)K, (uint64_t)M, (uint64_t)K * 2, 64, nt, 128)) return false;
  if (!make_tmap_2d(&d.s, scales, 2, (uint64_t)N, (uint64_t)(K / group), (uint64_t)N * 2, dtc::BM, 1, 0))
    return false;
  d.inv = inv;
  d.C = C;
  d.M = M; d.K = K; d.N = N; d.group = group; d.cdt = cdt;
  d.gx = (N + dtc::BM - 1) / dtc::BM;
  d.nk = (K + (64 * 8 / bits) - 1) / (64 * 8 / bits);
  return true;
}

cudaError_t run_decode_tc(int adt, int cdt, int bits, const void* A, int M, int K, int N, const void* codes,
                          const void* scales, int group, void* C, void* ws, cudaStream_t st) {
  const int nsm = num_sms();
  char* base = reinterpret_cast<char*>(ws);
  char* Ap = base + kDtcCounterBytes + dtc_partial_bytes(nsm);
  float* Vp = reinterpret_cast<float*>(Ap + dtc_prep_a_bytes(M, K));
  cudaError_t r = launch_prep_tc(adt, bits, A, M, K, Ap, Vp, st);
  if (r != cudaSuccess) return r;
  const int nt = dtc_nt(M);
  dtc::Batch<1> b{};
  if (!make_dtc_prob(b.p[0], bits, cdt, nt, Ap, Vp, M, K, N, codes, scales, group, C)) return cudaErrorInvalidValue;
  if (b.p[0].gx > kDtcMaxTiles) return cudaErrorInvalidValue;
  b.p[0].stage_begin = 0;
  b.p[0].tile_begin = 0;
  b.nprob = 1;
  b.total_stages = b.p[0].gx * b.p[0].nk;
  b.counters = reinterpret_cast<int*>(base);
  b.ws = reinterpret_cast<float*>(base + kDtcCounterBytes);
  return dispatch_dtc<1>(adt, bits, b, dtc_ctas(b.total_stages, nsm), nt, st);
}

// MoE batch: experts (1 <= M_e <= 16, group % 128 == 0) share one stream-K launch per <= MAXP experts
// (all of their tiles in one linear stage space).  A' is prepared once for all T tokens.
cudaError_t run_decode_tc_grouped(int adt, int cdt, int bits, const void* A, int K, int N, const int64_t* offsets,
                                  const int32_t* groups, const void* const* codes, const void* const* scales,
                                  void* C, void* ws, int64_t T, const int* experts, int nexp, cudaStream_t st) {
  constexpr int MAXP = 48;
  static_assert(sizeof(dtc::Batch<MAXP>) < 32000, "kernel parameter block limit");
  const int nsm = num_sms();
  char* base = reinterpret_cast<char*>(ws);
  char* Ap = base + kDtcCounterBytes + dtc_partial_bytes(nsm);
  float* Vp = reinterpret_cast<float*>(Ap + dtc_prep_a_bytes(T, K));
  cudaError_t r = launch_prep_tc(adt, bits, A, (int)T, K, Ap, Vp, st);
  if (r != cudaSuccess) return r;
  int maxm = 0;
  for (int ii = 0; ii < nexp; ++ii)
    maxm = std::max(maxm, (int)(offsets[experts[ii] + 1] - offsets[experts[ii]]));
  const int nt = dtc_nt(maxm);
  dtc::Batch<MAXP> b{};
  b.counters = reinterpret_cast<int*>(base);
  b.ws = reinterpret_cast<float*>(base + kDtcCounterBytes);
  int stages = 0, tiles = 0;
  auto flush = [&]() -> cudaError_t {
    b.total_stages = stages;
    cudaError_t rr = dispatch_dtc<MAXP>(adt, bits, b, dtc_ctas(stages, nsm), nt, st);
    b.nprob = 0;
    stages = tiles = 0;
    return rr;
  };
  for (int ii = 0; ii < nexp; ++ii) {
    const int e = experts[ii];
    const int Me = (int)(offsets[e + 1] - offsets[e]);
    char* Ce = reinterpret_cast<char*>(C) + (size_t)offsets[e] * N * (cdt == FQ_FP32 ? 4 : 2);
    dtc::Prob d;
    if (!make_dtc_prob(d, bits, cdt, nt, Ap + (size_t)offsets[e] * K * 2, Vp + offsets[e], Me, K, N, codes[e],
                       scales[e], groups[e], Ce))
      return cudaErrorInvalidValue;
    if (tiles + d.gx > kDtcMaxTiles) {  // counter region full: launch what we have first
      cudaError_t rr = flush();
      if (rr != cudaSuccess) return rr;
    }
    d.stage_begin = stages;
    d.tile_begin = tiles;
    b.p[b.nprob] = d;
    stages += d.gx * d.nk;
    tiles += d.gx;
    if (++b.nprob == MAXP) {
      cudaError_t rr = flush();
      if (rr != cudaSuccess) return rr;
    }
  }
  if (b.nprob) return flush();
  return cudaSuccess;
}

}  // namespace fq
