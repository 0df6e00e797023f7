// fq_gemv.cu — kernels A4 (decode GEMM) and A5 (deterministic split-K fixup, fused).
//
// Computes C[m,n] = sum_k A[m,k] * q[n,k] * s[k/g, n]  (§4.1: "dequantize the weights to
// match the data type of the activation and perform floating-point tensor core math").  Decode is
// "bottlenecked by memory bandwidth ... weights typically dominate the memory traffic": the
// kernel's job is to stream every packed weight byte exactly once at HBM speed.
//
// Warp-specialised, TMA-pipelined (B200 design):
//   warp 0 (producer): per pipeline stage, one 2-D TMA load of the packed weight tile
//     [256 columns n x 128 bytes of K] (SWIZZLE_128B) into shared memory, plus the activation slice
//     of the stage, copied with 16-byte loads and written to shared memory already in the
//     per-thread MMA fragment order (so consumers need no shuffles).  mbarrier full/empty ring.
//   warps 1..8 (consumers): each owns 32 output columns (2 tiles of 16).  Swap-AB mma.sync
//     m16n8k16: the MMA's 16 "rows" are output columns n, its 8 "columns" are tokens.  Codes are
//     unpacked in registers: int4 with one LOP3 per bf16x2 pair (mask 0x000F000F yields the pair
//     (k, k+4) as 128+(n^8)) and one subtract; the activations were stored by the producer with the
//     same (0,4),(1,5),(2,6),(3,7) permutation of each 8-k word.  int8: bytes -> exact bf16/fp16.
//   Scales: if group % KCHUNK == 0 every MMA of a K chunk lies in one group: the chunk accumulates
//     exact integer-weight partials in a fresh fp32 fragment, folded in with one FFMA by s[j,n].
//     Otherwise (small/odd groups) q*s is formed in the activation dtype before the MMA.
//   Split-K (grid.y): fp32 partials ws[S][M][N]; the last CTA of each column tile (self-resetting
//     arrival counter) reduces them in split order -> deterministic output.
//   Token tiles (grid.z): 16 tokens per tile (M > 16 re-streams the weights per tile; the
//     tensor-core prefill kernel A6 is the large-M path).
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "fq_common.cuh"
#include "fq_internal.h"

namespace fq {

#ifndef FQ_DEC_CW
#define FQ_DEC_CW 8
#endif
#ifndef FQ_DEC_EARLY
#define FQ_DEC_EARLY 1  // consumers release a stage as soon as its data is in registers
#endif
#ifndef FQ_DEC_EARLY2
#define FQ_DEC_EARLY2 1  // two 8-token MMA tiles (9 <= M <= 16): release before the MMAs (r02, 96 registers: -2%, profiles/r02/decode_early2_ab.txt)
#endif
constexpr int kConsumerWarps = FQ_DEC_CW;
// TMA warp + consumers (+ one activation-stager warp unless the activations were pre-converted)
template <bool PRE> constexpr int dec_threads() { return 32 * (1 + kConsumerWarps + (PRE ? 0 : 1)); }
constexpr int kRowsPerCta = 32 * kConsumerWarps;      // consumer warp = 2 tiles x 16 columns
constexpr int kWBoxes = (kRowsPerCta + 255) / 256;    // TMA boxes are at most 256 rows
constexpr int kWBoxRows = kRowsPerCta / kWBoxes;
static_assert(kWBoxRows * kWBoxes == kRowsPerCta && kWBoxRows % 8 == 0, "weight box split");
constexpr int kWBytesPerRow = 64;     // packed bytes of one column per stage, int4 / int8 (SWIZZLE_64B rows)
// int3 / int2: 128 k per stage as 48- / 32-byte rows of the canonical bit stream
// (unswizzled: the consumers' 12- / 8-byte reads of 8 rows x 4 threads hit distinct banks)
__host__ __device__ constexpr int wb_row(int bits) { return bits >= 4 ? kWBytesPerRow : 16 * bits; }
template <int BITS> constexpr int stage_w() { return kRowsPerCta * wb_row(BITS); }
constexpr int kStageW = kRowsPerCta * kWBytesPerRow;
constexpr int kMaxDecStages = 6;

template <int BITS>
struct DecGeom {
  static constexpr int KS = wb_row(BITS) * 8 / BITS;  // K per stage: 128 (int2/3/4) / 64 (int8)
  static constexpr int SEG = BITS <= 4 ? 32 : 16;      // K per thread per column per chunk
  static constexpr int KCH = 4 * SEG;                  // K per chunk (one quad): 128 / 64
  static constexpr int CHUNKS = KS / KCH;              // 2
  static constexpr int PIECES = SEG / 8;               // 16-byte activation pieces per thread/chunk
  static constexpr int ROWB = KS * 2;                  // token row stride of the staged activations
};

// Stage = [packed weights 256 x 64 B][activations MT*8 x KS (TMA, then permuted in place by the
// stager)][256 scales][per-token activation sums].  As many stages as fit two CTAs per SM.
// SACC == 3 ("double stage", int4 nibble path, <= 16 tokens, groups % 128 == 0): TWO 128-k chunks per
// stage -- two code boxes, one activation / sum / scale TMA each covering both chunks -- so the TMA
// operations, barrier round trips and loop overhead per weight byte halve.  Its stages do not fit
// the 1024-byte-rounded layout three times, so the code tiles of all stages form one ring (512-byte
// aligned for SWIZZLE_64B) and the small operands a second one behind it.  Small-operand offsets are
// relative to the stage's small-operand base: code(s) = s * CS, small(s) = SB + s * SS.
template <int BITS, int MT, int SACC>
struct DecStage {
  using G = DecGeom<BITS>;
  static constexpr bool DS = SACC == 3;
  static constexpr int NCH = DS ? 2 : 1;  // 128-k chunks per stage
  static constexpr int CODE = stage_w<BITS>() * NCH;
  static constexpr int ACT_BYTES = MT * 8 * G::ROWB * NCH;
  static constexpr int SC_BYTES = kRowsPerCta * 2 * (DS ? 2 : (SACC ? SACC : 8));  // scale rows (<= 8)
  static constexpr int SUM_BYTES = MT * 8 * 16 * NCH;  // per token and chunk: correction, 2^-e (+pad)
  static constexpr int ACT_OFS = 0;
  static constexpr int SC_OFS = ACT_OFS + ACT_BYTES;  // TMA destinations: 128-byte aligned
  static constexpr int SUM_OFS = SC_OFS + SC_BYTES;
  static constexpr int SMALL = SUM_OFS + SUM_BYTES;
  static_assert(CODE % 512 == 0 && ACT_BYTES % 128 == 0 && SC_BYTES % 128 == 0, "TMA smem alignment");
  // per CTA at 2 CTAs/SM: 115712 B of static (1024: the barriers, padded by the aligned extern
  // declaration) + dynamic shared memory
  static constexpr int PER = DS ? CODE + SMALL : ((CODE + SMALL + 1023) / 1024) * 1024;
  static constexpr int kBudget = DS ? 115712 - 1024 : 115712 - 1024 - 256;
  static constexpr int N = kBudget / PER < kMaxDecStages ? kBudget / PER : kMaxDecStages;
  static constexpr int CS = DS ? CODE : PER, SS = DS ? SMALL : PER, SB = DS ? N * CODE : CODE;
  static constexpr int SMEM = DS ? N * PER : N * PER + 1024;
};

// One decode problem (a matrix, its activation slice and output slice) of a batch.  A single
// launch can cover several problems (MoE experts): CTAs are numbered consecutively across the
// problems and each CTA finds its problem from `cta_begin`.  The TMA descriptors live in the
// __grid_constant__ parameter block (TMA accepts param-space descriptors).
struct DecProb {
  CUtensorMap w;  // packed codes [N][K*bits/8] u8, box [256 rows][64 B], SWIZZLE_64B
  CUtensorMap a;  // activations [M][K] 16-bit, box [MT*8 rows][K per stage]
  CUtensorMap s;  // scales [G][N] 16-bit, box [1 row][256 columns]
  CUtensorMap sm; // nibble path: per-(chunk, token) {correction, 2^-e, 0, 0} fp32, box [1][MT*8*4]
  const void* scales;
  void* C;
  float* ws;      // split-K partials [splits][M][N]
  int* counters;  // [ktiles][gx]
  int M, K, N, group, klen, cdt;
  int gx, splits, ktiles, cta_begin;
  int tok_base;   // nibble path: global token index of row 0 (parity of the pre-converted layout)
  int sc_rows;    // per-element-scale path: scale rows per stage staged by TMA (KS / group), 0 = read
                  // from global memory (groups that do not divide the stage)
  int sc_shift;   // log2(group) when sc_rows > 0
  const XRPeers* xr;  // fused row-parallel all-reduce (NEXT-1), device copy of the peer table; or null
  // MoE batch with DEVICE expert offsets (fq_gemm_grouped_dev): rows offs[e] .. offs[e+1]-1 of the
  // whole A / A' / C; M is then an upper bound (the launch geometry) and `a`, `sm`, C span all rows.
  const int64_t* offs;
  int e;
  int rows;          // rows of A / C (device offsets are clamped to them)
  int bound;         // the call's token bound (tokens beyond it: status bit 2)
  int tskip;         // this launch serves the expert's tokens [tskip, tskip + M)
  int32_t* status;   // nullable: bit 2 = some expert had more tokens than the launch bound / bad offsets
};
template <int MAXP>
struct DecBatch {
  DecProb p[MAXP];
  int nprob;
};

template <typename T>
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1);
template <>
__device__ __forceinline__ void mma16816<__nv_bfloat16>(float (&d)[4], const uint32_t (&a)[4],
                                                        uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
template <>
__device__ __forceinline__ void mma16816<__half>(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                                 uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <typename T>
__device__ __forceinline__ uint32_t sub2(uint32_t a, uint32_t b);
template <>
__device__ __forceinline__ uint32_t sub2<__nv_bfloat16>(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("sub.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
template <>
__device__ __forceinline__ uint32_t sub2<__half>(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
template <typename T>
__device__ __forceinline__ uint32_t mul2(uint32_t a, uint32_t b);
template <>
__device__ __forceinline__ uint32_t mul2<__nv_bfloat16>(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
template <>
__device__ __forceinline__ uint32_t mul2<__half>(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

// int4 word (k..k+7) -> pairs (k,k+4),(k+1,k+5),(k+2,k+6),(k+3,k+7) holding the exact codes.
template <typename T>
__device__ __forceinline__ void i4_pairs(uint32_t w, uint32_t (&q)[4]) {
  constexpr uint32_t mask = 0x000F000Fu;
  q[0] = sub2<T>(lop3_and_xor(w, mask, Dt<T>::kMagic4), Dt<T>::kBias4);
  q[1] = sub2<T>(lop3_and_xor(__umulhi(w, 1u << 28), mask, Dt<T>::kMagic4), Dt<T>::kBias4);  // w >> 4
  q[2] = sub2<T>(lop3_and_xor(w >> 8, mask, Dt<T>::kMagic4), Dt<T>::kBias4);
  q[3] = sub2<T>(lop3_and_xor(__umulhi(w, 1u << 20), mask, Dt<T>::kMagic4), Dt<T>::kBias4);  // w >> 12
}

// Same pairs WITHOUT the subtract: the values are q + OFF exactly (OFF = 136 bf16, 1032 fp16).
// The scale-on-accumulator path uses these and removes OFF * sum(a) per chunk afterwards (the
// activation sums are produced once per CTA by the producer warp), saving one HADD2 per pair.
template <typename T>
__device__ __forceinline__ void i4_pairs_off(uint32_t w, uint32_t (&q)[4]) {
  constexpr uint32_t mask = 0x000F000Fu;
  q[0] = lop3_and_xor(w, mask, Dt<T>::kMagic4);
  q[1] = lop3_and_xor(__umulhi(w, 1u << 28), mask, Dt<T>::kMagic4);  // w >> 4
  q[2] = lop3_and_xor(w >> 8, mask, Dt<T>::kMagic4);  // (SHF; an IMAD.HI here measured slower)
  q[3] = lop3_and_xor(__umulhi(w, 1u << 20), mask, Dt<T>::kMagic4);  // w >> 12
}
// "Nibble" unpack (FQ_NIB, int4 scale-on-accumulator path): the odd codes of a word are taken
// straight from bits 4..7 of each 16-bit half, which the magic makes worth 16x their value
// (exponent of 128/1024, mantissa bits 4..7), so one shift serves four pairs:
//   even pairs (k,k+4),(k+2,k+6): 128 + (n^8) = q + 136   (fp16: q + 1032)
//   odd  pairs (k+1,k+5),(k+3,k+7): 16 * (q + 16)        (fp16: 16 * (q + 72))
// The trick needs >= 8 mantissa bits, so the MMA runs in fp16 (10 bits) for bf16 inputs too:
// the stager re-encodes each token's activations of a chunk as fp16 after scaling them by a power
// of two 2^e that puts the chunk's max |a| in [2^14, 2^15) -- exact for every element within
// 2^31 of that max (bf16 has 8 significant bits, fp16 normals 11) -- and the fold multiplies the
// chunk's partial by 2^-e.  The stager also divides the odd activations by 16 (exact) and stores
// the per-token correction 1032 * sum_even(a') + 72 * sum_odd(a') (a' the scaled activations),
// removed once per chunk.
#ifndef FQ_NIB
#define FQ_NIB 1
#endif
#ifndef FQ_FOLD2
#define FQ_FOLD2 1  // the prep kernel stores -2^-e * correction; the fold is two FFMAs per output
#endif
template <typename T> struct Nib;
template <> struct Nib<__nv_bfloat16> {
  static constexpr uint32_t lo = 0x43084308u, hi = 0x43804380u, sixteenth = 0x3D803D80u;
  static constexpr float off_even = 136.f, off_odd = 16.f;
};
template <> struct Nib<__half> {
  static constexpr uint32_t lo = 0x64086408u, hi = 0x64806480u, sixteenth = 0x2C002C00u;
  static constexpr float off_even = 1032.f, off_odd = 72.f;
};
template <typename T>
__device__ __forceinline__ void i4_pairs_nib(uint32_t w, uint32_t (&q)[4]) {
  const uint32_t w8 = w >> 8;
  q[0] = lop3_and_xor(w, 0x000F000Fu, Nib<T>::lo);
  q[1] = lop3_and_xor(w, 0x00F000F0u, Nib<T>::hi);
  q[2] = lop3_and_xor(w8, 0x000F000Fu, Nib<T>::lo);
  q[3] = lop3_and_xor(w8, 0x00F000F0u, Nib<T>::hi);
}

template <typename T, int BITS> struct CodeOffset { static constexpr float v = 0.f; };
template <> struct CodeOffset<__nv_bfloat16, 4> { static constexpr float v = 136.f; };
template <> struct CodeOffset<__half, 4> { static constexpr float v = 1032.f; };
template <> struct CodeOffset<__half, 8> { static constexpr float v = 1152.f; };

// int8 word (k..k+3) -> natural pairs (k,k+1),(k+2,k+3) holding the exact codes.
template <typename T>
__device__ __forceinline__ void i8_pairs(uint32_t w, uint32_t (&q)[2]);
template <>
__device__ __forceinline__ void i8_pairs<__half>(uint32_t w, uint32_t (&q)[2]) {
  const uint32_t u = w ^ 0x80808080u;                                 // u = q + 128
  q[0] = sub2<__half>(prmt(u, 0x64646464u, 0x4140u), 0x64806480u);  // (1024+u) - 1152
  q[1] = sub2<__half>(prmt(u, 0x64646464u, 0x4342u), 0x64806480u);
}
template <>
__device__ __forceinline__ void i8_pairs<__nv_bfloat16>(uint32_t w, uint32_t (&q)[2]) {
  const uint32_t u = w ^ 0x80808080u;
  float f[4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    f[i] = __uint_as_float(prmt(u, 0x4B000000u, 0x7440u + i)) - 8388736.0f;  // (2^23+u) - (2^23+128)
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(f[2 * i + 1]), "f"(f[2 * i]));
    q[i] = r;
  }
}

__device__ __forceinline__ void i8_pairs_off_half(uint32_t w, uint32_t (&q)[2]) {
  const uint32_t u = w ^ 0x80808080u;         // values 1024 + u = q + 1152
  q[0] = prmt(u, 0x64646464u, 0x4140u);
  q[1] = prmt(u, 0x64646464u, 0x4342u);
}

template <typename T>
__device__ __forceinline__ float lds_scale(uint32_t addr) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
  return Dt<T>::to_f(*reinterpret_cast<T*>(&v));
}

template <typename T>
__device__ __forceinline__ uint32_t splat_scale(const T* scales, size_t idx) {
  const unsigned short s = __ldg(reinterpret_cast<const unsigned short*>(scales) + idx);
  return (uint32_t)s | ((uint32_t)s << 16);
}

// MMA row m of a 16-column tile -> tile row.  With 64-byte rows the two columns a 128-bit
// shared-memory phase touches (m = 2i, 2i+1) sit in different bank halves, and SWIZZLE_64B spreads
// the four 16-byte cells of a row: conflict-free.
__device__ __forceinline__ int prow(int m) { return m; }
// physical 16-byte cell of logical cell c in tile row R under CU_TENSOR_MAP_SWIZZLE_64B
__device__ __forceinline__ int swz64(int c, int R) { return c ^ ((R >> 1) & 3); }

// DBG (diagnostics build -DFQ_DIAG only, selected by FQ_DEC_DEBUG for bf16/int4/M<=8; 4 = skeleton
// streaming codes only): 1 = no MMA (fake FADD accumulate), 2 = no dequant (raw code words as MMA
// operands), 3 = consumers skip all compute.  The product build instantiates DBG = 0 only.
// int3 / int2: the 32 codes k = 32t .. 32t+31 of a thread, read from the canonical
// little-endian bit stream (12 / 8 bytes) and re-laid as four int4 words (code k + i at nibble i,
// sign-extended to 4 bits), so everything downstream is the int4 path.  Spreading the 3-bit fields of
// a 24-bit run x into nibbles takes three shift-and-select steps (12 / 6 / 3 bits apart); the
// garbage each step drags along lands in bit 3 of the nibbles, which the sign extension overwrites.
template <int BITS>
__device__ __forceinline__ uint4 lowbit_words(uint32_t addr) {
  uint32_t x[4];
  if (BITS == 3) {
    const uint32_t w0 = lds32(addr), w1 = lds32(addr + 4), w2 = lds32(addr + 8);
    x[0] = w0;
    x[1] = __funnelshift_r(w0, w1, 24);
    x[2] = __funnelshift_r(w1, w2, 16);
    x[3] = w2 >> 8;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t y = x[j];
      y = lop3_sel(y, y << 4, 0x0000FFFFu);   // fields 0-3 at bits 0-11, fields 4-7 at 16-27
      y = lop3_sel(y, y << 2, 0x00FF00FFu);   // per half: fields (0,1) at 0-5, (2,3) at 8-13
      y = lop3_sel(y, y << 1, 0x0F0F0F0Fu);   // per byte: even field at 0-2, odd at 4-6
      x[j] = lop3_sel(y, y << 1, 0x77777777u);  // bit 3 of every nibble = bit 2 (sign extension)
    }
  } else {
    const uint2 w = lds64(addr);
    x[0] = w.x;
    x[1] = w.x >> 16;
    x[2] = w.y;
    x[3] = w.y >> 16;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t y = x[j];
      y = lop3_sel(y, y << 8, 0x0000FFFFu);   // fields 0-3 at bits 0-7, fields 4-7 at 16-23
      y = lop3_sel(y, y << 4, 0x00FF00FFu);   // per half: fields (0,1) at 0-3, (2,3) at 8-11
      y = lop3_sel(y, y << 2, 0x0F0F0F0Fu);   // per byte: even field at 0-1, odd at 4-5
      y = lop3_sel(y, y << 1, 0x33333333u);   // bit 2 = bit 1
      x[j] = lop3_sel(y, y << 1, 0x77777777u);  // bit 3 = bit 2 (= bit 1)
    }
  }
  return make_uint4(x[0], x[1], x[2], x[3]);
}

#ifdef FQ_DIAG
// Diagnostics build only: per-CTA timeline of the last decode launch (globaltimer ns):
// {smid, start, first stage landed, main loop done, exit, producer past griddep_wait} --
// read with fq_diag_timeline() (tools/dec_timeline.py).
constexpr int kDiagCtas = 4096;
__device__ unsigned long long g_diag_tl[kDiagCtas][8];
__device__ __forceinline__ unsigned long long diag_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define FQ_TL(slot, v) do { if (threadIdx.x == 32 && blockIdx.x < kDiagCtas) g_diag_tl[blockIdx.x][slot] = (v); } while (0)
#endif
template <typename T, int BITS, int MT, int SACC, int DBG, int MAXP>
// Register caps (two CTAs per SM fit up to 112 / 96 registers at 288 / 320 threads), set without
// ptxas's launch_bounds heuristic.
#ifndef FQ_DEC_NIB_MAXREG
#define FQ_DEC_NIB_MAXREG 96  // measured: faster than 104 or 112 (which ptxas schedules worse)
#endif
// Two CTAs of 9 warps per SM need <= 96 registers: the register file is four 16K banks, one per SM
// sub-partition, and 18 warps put 5 on some sub-partition (5 x 32 x 104 > 16384 would leave ONE CTA
// per SM -- measured: FC1 M=16 99 -> 85 us, M=32 166 -> 148 us with the 96 cap;
// profiles/r02/decode_regcap_ab.txt).
#ifndef FQ_DEC_NIB2_MAXREG
#define FQ_DEC_NIB2_MAXREG 96  // two 8-token MMA tiles (9 <= M <= 16)
#endif
#ifndef FQ_DEC_NIB4_MAXREG
#define FQ_DEC_NIB4_MAXREG 96  // four 8-token MMA tiles (17 <= M <= 32)
#endif
__global__ void __maxnreg__((FQ_NIB && BITS <= 4 && SACC)
                               ? (MT == 4 ? FQ_DEC_NIB4_MAXREG : MT == 2 ? FQ_DEC_NIB2_MAXREG : FQ_DEC_NIB_MAXREG)
                               : 96)
decode_kernel(const __grid_constant__ DecBatch<MAXP> batch) {
  using G = DecGeom<BITS>;
  using SG = DecStage<BITS, MT, SACC>;
  constexpr int KS = G::KS, SEG = G::SEG, KCH = G::KCH, CHUNKS = G::CHUNKS, PIECES = G::PIECES;
  constexpr int ROWB = G::ROWB;
  constexpr int NSTG = SG::N;
  constexpr int ACT_OFS = SG::ACT_OFS, SUM_OFS = SG::SUM_OFS, SC_OFS = SG::SC_OFS;
  constexpr bool DS = SG::DS;
  constexpr int KSS = KS * SG::NCH;  // K per stage
  constexpr int CS = SG::CS, SS = SG::SS, SB = SG::SB;  // code(s) = s * CS, small operands: SB + s * SS
  constexpr int SC_BYTES = SG::SC_BYTES;
  constexpr int RAW_BYTES = SG::ACT_BYTES;
  // Nibble path: activations were pre-converted by prep_acts_kernel (fp16, fragment order) and
  // arrive by TMA with their per-chunk {correction, 2^-e}; there is no stager warp.
  constexpr bool NIB = FQ_NIB && BITS <= 4 && SACC;
  static_assert(!DS || (NIB && BITS >= 2 && BITS <= 4 && MT <= 2), "double stages: int4/3/2 nibble path, <= 16 tokens");
  // GS = 2 (int4, group 64, nibble path): each thread's four 8-code words come from the four 32-k
  // blocks of the stage (4 x LDS.32 instead of one LDS.128), so the MMAs of words 0-1 and 2-3 cover
  // the two 64-k groups separately; two exact partials per stage, folded with their own scales.
  constexpr int GS = SACC == 2 ? 2 : 1;
  static_assert(GS == 1 || NIB, "group split only on the nibble path");
  using TC = typename std::conditional<NIB, __half, T>::type;  // MMA operand type
  constexpr float OFF = NIB ? 1.f : (SACC ? CodeOffset<T, BITS>::v : 0.f);  // NIB: sums hold the correction
  constexpr int PPC = KCH / 8;  // 8-element pieces per chunk (16 int4, 8 int8): divides 32
  // MT = 4 (17..32 tokens): the activation fragments are read from shared memory per 8-code word
  // (LAZY) instead of all up front, so the stage is held until the MMAs are done
  constexpr bool LAZY = MT == 4;
  constexpr bool EARLY = LAZY ? false : (MT == 2 ? FQ_DEC_EARLY2 : FQ_DEC_EARLY);

  extern __shared__ __align__(1024) uint8_t dsmem[];
  __shared__ __align__(8) uint64_t full_bar[kMaxDecStages], empty_bar[kMaxDecStages], raw_bar[kMaxDecStages];
  __shared__ int s_last;
  uint8_t* sbase = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsmem) + 1023) & ~uintptr_t(1023));
  if (DS && sbase != dsmem) __trap();  // exact-size layout: the dynamic base must be 1024-byte aligned

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef FQ_DIAG
  { unsigned sm; asm("mov.u32 %0, %%smid;" : "=r"(sm)); FQ_TL(0, sm); FQ_TL(1, diag_now()); }
#endif
  int pi = 0;
  while (pi + 1 < batch.nprob && (int)blockIdx.x >= batch.p[pi + 1].cta_begin) ++pi;
  const DecProb& p = batch.p[pi];
  const int local = (int)blockIdx.x - p.cta_begin;
  const int bx = local % p.gx, by = (local / p.gx) % p.splits, bz = local / (p.gx * p.splits);
  const int N = p.N, K = p.K;
  const int n0 = bx * kRowsPerCta;
  const int kbeg = by * p.klen;
  const int kend = min(K, kbeg + p.klen);
  const int nst = (kend - kbeg + KSS - 1) / KSS;
  const int tok0 = bz * MT * 8;
  int M = p.M, row0 = 0;  // row0: first row of this problem in A / A' / C (device offsets only)
  if (p.offs) {
    griddep_wait();  // the offsets may come from the previous kernel (the router)
    const int64_t o0 = p.offs[p.e], o1 = p.offs[p.e + 1];
    // rows outside [0, rows) or beyond the launch's token bound are not computed (status bit 2)
    const int64_t lo = max((int64_t)0, min(o0, (int64_t)p.rows)), hi = max(lo, min(o1, (int64_t)p.rows));
    row0 = (int)lo + p.tskip;
    M = (int)max((int64_t)0, min(hi - lo - p.tskip, (int64_t)p.M));
    if (threadIdx.x == 0 && blockIdx.x == p.cta_begin && p.status && (hi - lo > p.bound || lo != o0 || hi != o1))
      atomicOr(p.status, 4);
    if (tok0 >= M) return;  // token tile beyond this expert's tokens: the whole CTA leaves
  }
  const int tok_base = p.offs ? row0 : p.tok_base;  // global token index of row 0 (nibble parity)

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTG; ++s) {
      mbar_init(&full_bar[s], NIB ? 1 : 1 + 32);  // TMA expect_tx arrival (+ 32 stager lanes)
      mbar_init(&raw_bar[s], 1);                   // activation TMA (stager path)
      mbar_init(&empty_bar[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.w);
    prefetch_tmap(&p.a);
    if (SACC) prefetch_tmap(&p.s);
    if (NIB) prefetch_tmap(&p.sm);
  }
  __syncthreads();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (one lane)
    if (lane == 0) {
      const uint64_t polw = policy_evict_first();
      const uint64_t pola = policy_evict_last();
      // chunk c = kbeg/KCH + i (one chunk per stage) lies in scale group c / gm
      const int gm = SACC == 1 ? p.group / KCH : 1;
      int grem = SACC == 1 ? (kbeg / KCH) % gm : 0, gj = SACC == 1 ? (kbeg / KCH) / gm : 0;
      auto issue_w = [&](int i, int s) {  // the stage's packed weights + scales (+ expect_tx)
        uint8_t* st = sbase + s * CS;
        uint8_t* xs = sbase + SB + s * SS;
        const int k0 = kbeg + i * KSS;
        const int scb = DS ? SG::SC_BYTES : SACC ? SACC * kRowsPerCta * 2 : p.sc_rows * kRowsPerCta * 2;
        if (DBG == 4) {  // diagnostics: codes only
          mbar_arrive_expect_tx(&full_bar[s], stage_w<BITS>());
          tma_load_2d(st, &p.w, &full_bar[s], k0 * BITS / 8, n0, polw);
          return;
        }
        mbar_arrive_expect_tx(&full_bar[s], SG::CODE + scb + (NIB ? SG::ACT_BYTES + SG::SUM_BYTES : 0));
#pragma unroll
        for (int ch = 0; ch < SG::NCH; ++ch)
#pragma unroll
          for (int bx2 = 0; bx2 < kWBoxes; ++bx2)
            tma_load_2d(st + ch * stage_w<BITS>() + bx2 * kWBoxRows * wb_row(BITS), &p.w, &full_bar[s],
                        (k0 + ch * KS) * BITS / 8, n0 + bx2 * kWBoxRows, polw);
        if (DS) {  // scale rows k0 / g and the next (box of 2): chunk 1 uses the second iff it starts a group
#pragma unroll
          for (int bx2 = 0; bx2 < kWBoxes; ++bx2)
            tma_load_2d(xs + SC_OFS + bx2 * kWBoxRows * 2, &p.s, &full_bar[s], n0 + bx2 * kWBoxRows,
                        k0 / p.group, polw);
        } else if (SACC) {
#pragma unroll
          for (int bx2 = 0; bx2 < kWBoxes; ++bx2)
            tma_load_2d(xs + SC_OFS + bx2 * kWBoxRows * 2, &p.s, &full_bar[s], n0 + bx2 * kWBoxRows,
                        GS == 2 ? (k0 >> 6) : gj, polw);  // GS: the stage's two 64-k rows (box of 2)
          if (++grem == gm) { grem = 0; ++gj; }
        } else if (p.sc_rows) {
#pragma unroll
          for (int bx2 = 0; bx2 < kWBoxes; ++bx2)
            tma_load_2d(xs + SC_OFS + bx2 * kWBoxRows * 2, &p.s, &full_bar[s], n0 + bx2 * kWBoxRows,
                        k0 >> p.sc_shift, polw);
        }
      };
      auto issue_a = [&](int i, int s) {  // the stage's activations (+ per-chunk sums)
        if (DBG == 4) return;
        uint8_t* st = sbase + SB + s * SS;  // the stage's small operands
        const int k0 = kbeg + i * KSS;
        if (NIB) {
          tma_load_2d(st + ACT_OFS, &p.a, &full_bar[s], k0, row0 + tok0, pola);
          tma_load_2d(st + SUM_OFS, &p.sm, &full_bar[s], (row0 + tok0) * 4, k0 / KCH, pola);
        } else {
          mbar_arrive_expect_tx(&raw_bar[s], RAW_BYTES);
          tma_load_2d(st + ACT_OFS, &p.a, &raw_bar[s], k0, row0 + tok0, pola);
        }
      };
      // Weights are constants: the first NSTG stages are requested before waiting for the grid
      // this launch depends on (programmatic dependent launch: the activations may still be in
      // flight from the previous kernel in the stream).
      const int npre = min(nst, NSTG);
#ifdef FQ_DIAG
      if (blockIdx.x < kDiagCtas) g_diag_tl[blockIdx.x][6] = diag_now();
#endif
      for (int i = 0; i < npre; ++i) issue_w(i, i);
#ifdef FQ_DIAG
      if (blockIdx.x < kDiagCtas) g_diag_tl[blockIdx.x][7] = diag_now();
#endif
#ifndef FQ_DEC_EARLY_TRIGGER
#define FQ_DEC_EARLY_TRIGGER 1
#endif
      // The next kernel in the stream (the next GEMM's prep, which triggers its decode kernel at once)
      // may launch as soon as every CTA of this grid has started: its CTAs take the SM slots this
      // grid's early finishers leave and pre-stream their weights; everything they read or write that
      // this grid touches is ordered behind their griddep_wait.
      if (FQ_DEC_EARLY_TRIGGER) griddep_launch_dependents();
      griddep_wait();
#ifdef FQ_DIAG
      if (blockIdx.x < kDiagCtas) g_diag_tl[blockIdx.x][5] = diag_now();
#endif
      for (int i = 0; i < npre; ++i) issue_a(i, i);
      int s = npre % NSTG;
      uint32_t ph = npre == NSTG ? 1u : 0u;
      for (int i = npre; i < nst; ++i) {
        mbar_wait(&empty_bar[s], ph ^ 1);
        issue_w(i, s);
        issue_a(i, s);
        if (++s == NSTG) { s = 0; ph ^= 1; }
      }
      if (!FQ_DEC_EARLY_TRIGGER) griddep_launch_dependents();
    }
    return;
  }
  if (!NIB && warp > kConsumerWarps) {
    // ------------------------------------------------------------ activation stagers
    // The TMA leaves [MT*8 tokens][KS] in natural order (rows >= M zero-filled).  Each 8-element
    // piece is permuted in place into the consumers' fragment order: words (0,4),(1,5),(2,6),(3,7)
    // (int4), cell c -> (c % PIECES) * 4 + c / PIECES, XOR (token & 1) * 4 (puts the two tokens of
    // a 128-bit shared-memory phase in different bank halves); plus the per-token sums and, on
    // the nibble path, the fp16 re-encoding.
    constexpr int CELLS = KS / 8;  // 16-byte pieces per token row
    constexpr int NPIECE = MT * 8 * CELLS;
    static_assert(NPIECE % 32 == 0 && 32 % CELLS == 0, "piece groups of whole tokens");
    constexpr int NPW = NPIECE / 32;
    const int mloc = min(M - tok0, MT * 8);  // tokens >= mloc are TMA zero fill: left alone
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < nst; ++i) {
      mbar_wait(&raw_bar[s], ph);
      uint8_t* st = sbase + SB + s * SS;  // the stage's small operands
      const uint32_t stu = smem_u32(st);
      uint4 vj[NPW];
#pragma unroll
      for (int j = 0; j < NPW; ++j)
        if ((32 * j) / CELLS < mloc) vj[j] = lds128(stu + ACT_OFS + (lane + 32 * j) * 16);
      __syncwarp();  // every read of this warp's tokens precedes the in-place writes
#pragma unroll
      for (int j = 0; j < NPW; ++j) {
        if ((32 * j) / CELLS >= mloc) continue;  // warp-uniform
        const int pc = lane + 32 * j;
        const int tl = pc / CELLS;           // local token
        const int kl = (pc % CELLS) * 8;     // local k of this 8-element piece
        const int r = kl % KCH, tq = r / SEG, w16 = (r % SEG) / 8;
        const uint4 va = vj[j];
        uint4 v = va;
        {
          if (OFF != 0.f) {
            // sum of the 8 activations, reduced over the PPC lanes of this chunk (aligned groups)
            float sum = 0.f;
            const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
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
            for (int o = PPC / 2; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            if ((lane % PPC) == 0) reinterpret_cast<float*>(st + SUM_OFS)[tl] = sum;
          }
          if (BITS <= 4) {
            v = make_uint4(prmt(v.x, v.z, 0x5410u), prmt(v.x, v.z, 0x7632u), prmt(v.y, v.w, 0x5410u),
                           prmt(v.y, v.w, 0x7632u));
          }
        }
        sts128(stu + ACT_OFS + tl * ROWB + (((w16 * 4 + tq) ^ ((tl & 1) << 2)) << 4), v);
      }
      mbar_arrive(&full_bar[s]);
      if (++s == NSTG) { s = 0; ph ^= 1; }
    }
    return;
  }

  // --------------------------------------------------------------------------- consumers
  static_assert(CHUNKS == 1, "one MMA chunk (one scale) per stage");
  const T* __restrict__ S = reinterpret_cast<const T*>(p.scales);
  const int cw = warp - 1;
  const int gq = lane >> 2, t = lane & 3;
  int Rg[2], Rh[2], ng[2], nh[2];
  uint32_t wofs_g[2], wofs_h[2];  // per-thread byte offsets inside a stage (swizzled cells)
#pragma unroll
  for (int rt = 0; rt < 2; ++rt) {
    Rg[rt] = cw * 32 + rt * 16 + prow(gq);
    Rh[rt] = Rg[rt] + 8;
    ng[rt] = min(n0 + Rg[rt], N - 1);
    nh[rt] = min(n0 + Rh[rt], N - 1);
    if (BITS < 4) {  // bytes [t * wb/4, +wb/4) of the unswizzled bit-stream row = k 32t .. 32t+31
      wofs_g[rt] = Rg[rt] * wb_row(BITS) + t * (wb_row(BITS) / 4);
      wofs_h[rt] = Rh[rt] * wb_row(BITS) + t * (wb_row(BITS) / 4);
    } else {
      wofs_g[rt] = Rg[rt] * kWBytesPerRow + (swz64(t, Rg[rt]) << 4);
      wofs_h[rt] = Rh[rt] * kWBytesPerRow + (swz64(t, Rh[rt]) << 4);
    }
  }
  uint32_t aofs[MT][PIECES];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int w16 = 0; w16 < PIECES; ++w16)
      aofs[mt][w16] = ACT_OFS + (mt * 8 + gq) * ROWB * SG::NCH +
                      (((w16 * 4 + t) ^ (((NIB ? tok_base + tok0 + gq : gq) & 1) << 2)) << 4);
  const uint32_t saofs = NIB ? SUM_OFS + 2 * t * 16 : SUM_OFS + 2 * t * 4;
  float acc[2][MT][4];
#pragma unroll
  for (int rt = 0; rt < 2; ++rt)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[rt][mt][i] = 0.f;

  const uint32_t sb = smem_u32(sbase);
  // Everything a consumer thread reads from one stage, in registers.
  struct StageOps {
    float sg[2][GS], sh[2][GS];       // the stage's scales (TMA-staged with the weights), per 64-k group
    uint4 b[LAZY ? 1 : MT][PIECES];   // activation fragments
    float2 sa[MT][GS], iv[MT];        // per-token corrections / inverse power-of-two scales
    uint4 wgv[2], whv[2];             // code words of rows g / h of both row tiles
    uint32_t scg[2][4], sch[2][4];    // per-element-scale path: splatted scale words
  };
  // wst: the chunk's codes; xst: the stage's small operands; DS chunk 1: ach / sch = activation / sum
  // offsets of the chunk, srow = byte offset of its scale row
  auto load_ops = [&](uint32_t wst, uint32_t xst, StageOps& o, int ach = 0, int sch = 0, int srow = 0) {
    if (SACC) {
#pragma unroll
      for (int rt = 0; rt < 2; ++rt)
#pragma unroll
        for (int gi = 0; gi < GS; ++gi) {
          o.sg[rt][gi] = lds_scale<T>(xst + SC_OFS + srow + gi * kRowsPerCta * 2 + Rg[rt] * 2);
          o.sh[rt][gi] = lds_scale<T>(xst + SC_OFS + srow + gi * kRowsPerCta * 2 + Rh[rt] * 2);
        }
    }
    if (DBG == 3 || DBG == 4) return;
    if (!LAZY) {
#pragma unroll
      for (int mt = 0; mt < (LAZY ? 1 : MT); ++mt)
#pragma unroll
        for (int w16 = 0; w16 < PIECES; ++w16) o.b[mt][w16] = lds128(xst + ach + aofs[mt][w16]);
    }
    if (NIB) {  // {corr, 2^-e, corr_lo, corr_hi} of tokens 2t and 2t+1 (lo / hi: the 64-k halves)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        if (GS == 1) {
          const float2 x0 = lds64f(xst + sch + saofs + mt * 128), x1 = lds64f(xst + sch + saofs + mt * 128 + 16);
          o.sa[mt][0] = make_float2(x0.x, x1.x);
          o.iv[mt] = make_float2(x0.y, x1.y);
        } else {
          const uint4 x0 = lds128(xst + sch + saofs + mt * 128), x1 = lds128(xst + sch + saofs + mt * 128 + 16);
          o.sa[mt][0] = make_float2(__uint_as_float(x0.z), __uint_as_float(x1.z));
          o.sa[mt][GS - 1] = make_float2(__uint_as_float(x0.w), __uint_as_float(x1.w));
          o.iv[mt] = make_float2(__uint_as_float(x0.y), __uint_as_float(x1.y));
        }
      }
    } else if (OFF != 0.f) {
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) o.sa[mt][0] = lds64f(xst + sch + saofs + mt * 32);
    }
#pragma unroll
    for (int rt = 0; rt < 2; ++rt) {
      if (BITS < 4) {
        o.wgv[rt] = lowbit_words<BITS>(wst + wofs_g[rt]);
        o.whv[rt] = lowbit_words<BITS>(wst + wofs_h[rt]);
      } else if (GS == 1) {
        o.wgv[rt] = lds128(wst + wofs_g[rt]);
        o.whv[rt] = lds128(wst + wofs_h[rt]);
      } else {  // word w = 8 codes at k = 32 w + 8 t: cell w (swizzled), word t of the cell
        uint32_t g4[4], h4[4];
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          g4[w] = lds32(wst + Rg[rt] * kWBytesPerRow + (swz64(w, Rg[rt]) << 4) + t * 4);
          h4[w] = lds32(wst + Rh[rt] * kWBytesPerRow + (swz64(w, Rh[rt]) << 4) + t * 4);
        }
        o.wgv[rt] = make_uint4(g4[0], g4[1], g4[2], g4[3]);
        o.whv[rt] = make_uint4(h4[0], h4[1], h4[2], h4[3]);
      }
    }
    // per-element-scale path with TMA-staged scale rows: into registers before the stage is
    // released (the producer may overwrite it right after the early release)
    if (!SACC && p.sc_rows) {
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const uint32_t so = xst + SC_OFS + (((t * SEG + w * (SEG / 4)) >> p.sc_shift) * kRowsPerCta) * 2;
#pragma unroll
        for (int rt = 0; rt < 2; ++rt) {
          const uint32_t vg = lds_u16(so + Rg[rt] * 2), vh = lds_u16(so + Rh[rt] * 2);
          o.scg[rt][w] = vg | (vg << 16);
          o.sch[rt][w] = vh | (vh << 16);
        }
      }
    }
  };
  auto compute = [&](const StageOps& o, uint32_t xst, int k0) {
    if (DBG == 3 || DBG == 4) return;
#pragma unroll
    for (int rt = 0; rt < 2; ++rt) {
      const uint4 wg = o.wgv[rt];
      const uint4 wh = o.whv[rt];
      const uint32_t wgw[4] = {wg.x, wg.y, wg.z, wg.w};
      const uint32_t whw[4] = {wh.x, wh.y, wh.z, wh.w};
      float part[GS][MT][4];
      if (SACC) {
#pragma unroll
        for (int gi = 0; gi < GS; ++gi)
#pragma unroll
          for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int q = 0; q < 4; ++q) part[gi][mt][q] = 0.f;
      }
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        uint32_t sgs = 0, shs = 0;
        if (!SACC) {  // small / odd groups: q*s in the activation dtype before the MMA
          if (p.sc_rows) {  // the stage's scale rows (TMA-staged, read with the stage)
            sgs = o.scg[rt][w];
            shs = o.sch[rt][w];
          } else {
            // past the end of K (the last, partial stage) the codes and activations are TMA zero
            // fill: clamp to the last group so the scale read stays in bounds (and finite)
            const int kw = min(k0 + t * SEG + w * (SEG / 4), p.K - 1);
            const size_t j = (size_t)(kw / p.group) * N;
            sgs = splat_scale<T>(S, j + ng[rt]);
            shs = splat_scale<T>(S, j + nh[rt]);
          }
        }
        float(*dst)[4] = SACC ? part[(w * GS) >> 2] : acc[rt];
        if (BITS <= 4) {
          uint32_t qg[4], qh[4];
          if (DBG == 2) {
#pragma unroll
            for (int q = 0; q < 4; ++q) { qg[q] = wgw[w] + q; qh[q] = whw[w] + q; }
          } else if (NIB) {
            i4_pairs_nib<TC>(wgw[w], qg);
            i4_pairs_nib<TC>(whw[w], qh);
          } else if (OFF != 0.f) {
            i4_pairs_off<T>(wgw[w], qg);
            i4_pairs_off<T>(whw[w], qh);
          } else {
            i4_pairs<T>(wgw[w], qg);
            i4_pairs<T>(whw[w], qh);
          }
          if (!SACC) {
#pragma unroll
            for (int q = 0; q < 4; ++q) { qg[q] = mul2<T>(qg[q], sgs); qh[q] = mul2<T>(qh[q], shs); }
          }
#pragma unroll
          for (int pp = 0; pp < 2; ++pp) {
            const uint32_t a[4] = {qg[2 * pp], qh[2 * pp], qg[2 * pp + 1], qh[2 * pp + 1]};
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
              const uint4 bw = LAZY ? lds128(xst + aofs[mt][w]) : o.b[LAZY ? 0 : mt][w];
              const uint32_t b0 = pp ? bw.z : bw.x;
              const uint32_t b1 = pp ? bw.w : bw.y;
              if (DBG == 1) {
#pragma unroll
                for (int q = 0; q < 4; ++q) dst[mt][q] += __uint_as_float(a[q] ^ b0);
              } else {
                mma16816<TC>(dst[mt], a, b0, b1);
              }
            }
          }
        } else {
          uint32_t qg[2], qh[2];
          if (OFF != 0.f && Dt<T>::id == FQ_FP16) {
            i8_pairs_off_half(wgw[w], qg);
            i8_pairs_off_half(whw[w], qh);
          } else {
            i8_pairs<T>(wgw[w], qg);
            i8_pairs<T>(whw[w], qh);
          }
          if (!SACC) {
#pragma unroll
            for (int q = 0; q < 2; ++q) { qg[q] = mul2<T>(qg[q], sgs); qh[q] = mul2<T>(qh[q], shs); }
          }
          const uint32_t a[4] = {qg[0], qh[0], qg[1], qh[1]};
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            const uint4 bb = LAZY ? lds128(xst + aofs[mt][w >> 1]) : o.b[LAZY ? 0 : mt][w >> 1];
            mma16816<T>(dst[mt], a, (w & 1) ? bb.z : bb.x, (w & 1) ? bb.w : bb.y);
          }
        }
      }
      if (SACC) {
#pragma unroll
        for (int gi = 0; gi < GS; ++gi)
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            const float(&pp)[4] = part[gi][mt];
            float p0 = pp[0], p1 = pp[1], p2 = pp[2], p3 = pp[3];
            if (NIB && FQ_FOLD2) {
              // S' holds -2^-e * correction: t = 2^-e p - 2^-e corr = 2^-e (p - corr) exactly (power
              // of two), then acc += s * t -- the same two roundings as (s 2^-e) (p - corr), two
              // instructions per output instead of three
              acc[rt][mt][0] = fmaf(o.sg[rt][gi], fmaf(o.iv[mt].x, p0, o.sa[mt][gi].x), acc[rt][mt][0]);
              acc[rt][mt][1] = fmaf(o.sg[rt][gi], fmaf(o.iv[mt].y, p1, o.sa[mt][gi].y), acc[rt][mt][1]);
              acc[rt][mt][2] = fmaf(o.sh[rt][gi], fmaf(o.iv[mt].x, p2, o.sa[mt][gi].x), acc[rt][mt][2]);
              acc[rt][mt][3] = fmaf(o.sh[rt][gi], fmaf(o.iv[mt].y, p3, o.sa[mt][gi].y), acc[rt][mt][3]);
              continue;
            }
            if (OFF != 0.f) {  // remove OFF * sum_k a[tok, k] (tokens 2t, 2t+1 of this MMA tile)
              p0 = fmaf(-OFF, o.sa[mt][gi].x, p0);
              p1 = fmaf(-OFF, o.sa[mt][gi].y, p1);
              p2 = fmaf(-OFF, o.sa[mt][gi].x, p2);
              p3 = fmaf(-OFF, o.sa[mt][gi].y, p3);
            }
            if (NIB) {  // undo the chunk's power-of-two activation scale
              acc[rt][mt][0] = fmaf(o.sg[rt][gi] * o.iv[mt].x, p0, acc[rt][mt][0]);
              acc[rt][mt][1] = fmaf(o.sg[rt][gi] * o.iv[mt].y, p1, acc[rt][mt][1]);
              acc[rt][mt][2] = fmaf(o.sh[rt][gi] * o.iv[mt].x, p2, acc[rt][mt][2]);
              acc[rt][mt][3] = fmaf(o.sh[rt][gi] * o.iv[mt].y, p3, acc[rt][mt][3]);
            } else {
              acc[rt][mt][0] = fmaf(o.sg[rt][gi], p0, acc[rt][mt][0]);
              acc[rt][mt][1] = fmaf(o.sg[rt][gi], p1, acc[rt][mt][1]);
              acc[rt][mt][2] = fmaf(o.sh[rt][gi], p2, acc[rt][mt][2]);
              acc[rt][mt][3] = fmaf(o.sh[rt][gi], p3, acc[rt][mt][3]);
            }
          }
      }
    }
  };
  auto release = [&](int s_) {
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[s_]);
  };
  // (A software-pipelined variant -- stage i+1's operands read and its slot released before stage i
  // is computed -- was measured 40% slower on OPT-175B FC1/FC2 at M <= 8: profiles/r02/decode_pf_rejected.txt.)
  int s = 0;
  uint32_t ph = 0;
  // DS: chunk 1 of a stage uses the second staged scale row iff it starts a new group (groups % 128)
  const int gch = DS ? p.group / KCH : 1;
  int gpos = DS ? (kbeg / KCH) % gch : 0;  // position of the stage's chunk 0 inside its group
  if (DS) {
    for (int i = 0; i < nst; ++i) {
      const int k0 = kbeg + i * KSS;
      mbar_wait(&full_bar[s], ph);
#ifdef FQ_DIAG
      if (i == 0) FQ_TL(2, diag_now());
#endif
      const uint32_t wst = sb + s * CS, xst = sb + SB + s * SS;
      const int r1 = gpos + 1 == gch ? kRowsPerCta * 2 : 0;
      gpos += 2;
      if (gpos >= gch) gpos -= gch;
      if (gpos >= gch) gpos -= gch;
      StageOps o;
      load_ops(wst, xst, o);
      compute(o, xst, k0);
      load_ops(wst + stage_w<BITS>(), xst, o, ROWB, MT * 8 * 16, r1);
      release(s);  // the stage's operands are in registers
      compute(o, xst, k0 + KS);
      if (++s == NSTG) { s = 0; ph ^= 1; }
    }
  } else {
    for (int i = 0; i < nst; ++i) {
      const int k0 = kbeg + i * KS;
      mbar_wait(&full_bar[s], ph);
#ifdef FQ_DIAG
      if (i == 0) FQ_TL(2, diag_now());
#endif
      const uint32_t wst = sb + s * CS, xst = sb + SB + s * SS;
      StageOps o;
      load_ops(wst, xst, o);
      if (EARLY && DBG != 3 && DBG != 4) release(s);  // everything is in registers: hand the slot back
      compute(o, xst, k0);
      if (!EARLY || DBG == 3 || DBG == 4) release(s);
      if (++s == NSTG) { s = 0; ph ^= 1; }
    }
  }

  // ------------------------------------------------------------- epilogue (+ fused A5 fixup)
#ifdef FQ_DIAG
  FQ_TL(3, diag_now());
  FQ_TL(4, 0ull);
  struct DiagExit { __device__ ~DiagExit() { FQ_TL(4, diag_now()); } } diag_exit;
#endif
  auto out_idx = [&](int rt, int mt, int i, int& n, int& tok) {
    n = n0 + ((i >> 1) ? Rh[rt] : Rg[rt]);
    tok = tok0 + mt * 8 + 2 * t + (i & 1);
  };
  auto store_out = [&](int tok, int n, float v) {
    const size_t o = (size_t)(row0 + tok) * N + n;
    if (p.cdt == FQ_FP32) reinterpret_cast<float*>(p.C)[o] = v;
    else reinterpret_cast<T*>(p.C)[o] = Dt<T>::from_f(v);
  };
  const int S_ = p.splits;
  // Fused row-parallel all-reduce ("we must issue an all reduce after each attention
  // and FFN block", §2.1): the rank's final partial of this output tile is pushed into the tile
  // owner's receive slot (rank-indexed), and the last of the `world` ranks to arrive at the owner's
  // counter sums the slots in rank order (deterministic) and writes the tile to every rank's output,
  // then bumps every rank's completion counter (fq_xr_wait waits for it).  No CTA ever waits on
  // another GPU, so the GEMMs of all ranks complete independently.
  const XRPeers* xr = p.xr;
  const int tile = bz * p.gx + bx;
  const int tile_elems = MT * 8 * kRowsPerCta;
  float* xslot = nullptr;
  if (xr) {
    const int owner = tile % xr->world;
    xslot = xr->recv[owner] + ((size_t)tile * xr->world + xr->rank) * tile_elems;
  }
  auto emit = [&](int tok, int n, float v) {  // this rank's final value of output (tok, n)
    if (xslot) xslot[(tok - tok0) * kRowsPerCta + (n - n0)] = v;
    else store_out(tok, n, v);
  };
  auto xr_finish = [&]() {  // consumer warps only; every local value of the tile emitted
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kConsumerWarps));
    const int owner = tile % xr->world;
    if (threadIdx.x == 32) {
      __threadfence_system();
      const int last = atomicAdd_system(xr->arrive[owner] + tile, 1) == xr->world - 1;
      if (last) __threadfence_system();
      s_last = last;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kConsumerWarps));
    if (!s_last) return;
    const int c = threadIdx.x - 32;
    const int n = n0 + c;
    const int ntok = min(M - tok0, MT * 8);
    const float* slots = xr->recv[owner] + (size_t)tile * xr->world * tile_elems;
    if (n < N) {
      for (int j = 0; j < ntok; ++j) {
        float v = 0.f;
        for (int r = 0; r < xr->world; ++r) v += ld_relaxed_sys(slots + (size_t)r * tile_elems + j * kRowsPerCta + c);
        const size_t o = (size_t)(tok0 + j) * N + n;
        for (int d = 0; d < xr->world; ++d) {
          if (p.cdt == FQ_FP32) reinterpret_cast<float*>(xr->out[d])[o] = v;
          else reinterpret_cast<T*>(xr->out[d])[o] = Dt<T>::from_f(v);
        }
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kConsumerWarps));
    if (threadIdx.x == 32) {
      xr->arrive[owner][tile] = 0;  // self-reset (every rank of this call has arrived)
      __threadfence_system();
      for (int d = 0; d < xr->world; ++d) atomicAdd_system(xr->done[d], 1);
    }
  };
  if (S_ == 1) {
#pragma unroll
    for (int rt = 0; rt < 2; ++rt)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          int n, tok;
          out_idx(rt, mt, i, n, tok);
          if (n < N && tok < M) emit(tok, n, acc[rt][mt][i]);
        }
    if (xr) xr_finish();
    return;
  }
  float* part_out = p.ws + (size_t)by * M * N;
#pragma unroll
  for (int rt = 0; rt < 2; ++rt)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int n, tok;
        out_idx(rt, mt, i, n, tok);
        if (n < N && tok < M) __stcg(part_out + (size_t)tok * N + n, acc[rt][mt][i]);
      }
  // bar.sync orders every consumer's partial stores before the counting thread's release fence
  // (cumulativity); its acquire fence + the second bar.sync order the reads of the last CTA.
  asm volatile("bar.sync 1, %0;" ::"n"(32 * kConsumerWarps));
  int* ctr = p.counters + bz * p.gx + bx;
  if (threadIdx.x == 32) {
    __threadfence();
    const int last = (atomicAdd(ctr, 1) == S_ - 1);
    if (last) __threadfence();
    s_last = last;
  }
  asm volatile("bar.sync 1, %0;" ::"n"(32 * kConsumerWarps));
  if (!s_last) return;
  // Fixup: consumer thread c owns column n0 + c (coalesced across the CTA); its tokens are summed
  // over the splits in split order, 4 tokens per round so their loads are in flight together.
  {
    const int c = threadIdx.x - 32;  // 0 .. kRowsPerCta-1
    const int n = n0 + c;
    const int ntok = min(M - tok0, MT * 8);
    if (n < N) {
      for (int j0 = 0; j0 < ntok; j0 += 4) {
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        for (int s = 0; s < S_; ++s) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (j0 + u < ntok) v[u] += __ldcg(p.ws + ((size_t)s * M + tok0 + j0 + u) * N + n);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (j0 + u < ntok) emit(tok0 + j0 + u, n, v[u]);
      }
    }
  }
  if (threadIdx.x == 32) *ctr = 0;  // self-reset for the next call / graph replay
  if (xr) xr_finish();
}

// Completion of a fused row-parallel GEMM on this rank (fq_xr_wait): every output tile has been
// written by its reducing CTA (possibly on another GPU) once `done` reaches the tile count.
// A peer that never arrives (a rank that skipped the call) traps after 5 s instead of hanging the
// device: the error surfaces at the caller's next synchronisation.
__global__ void xr_wait_kernel(int32_t* done, int expected) {
  griddep_launch_dependents();
  if (threadIdx.x == 0) {
    uint64_t t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (ld_acquire_sys(done) < expected) {
      __nanosleep(256);
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 5000000000ull) __trap();
    }
    *done = 0;  // self-reset: no rank can contribute to this rank's next call before it starts
    __threadfence_system();
  }
}

// ---- activation pre-conversion for the nibble path (one launch per GEMM call, M x K elements) --
// Half-warp = one (token, 128-k chunk): 16 lanes x 8 activations.  Output A'[tok][k]: fp16, each
// chunk's 8-element pieces permuted into the decode consumers' fragment order (words (a0,a4),
// (a1,a5)/16, (a2,a6), (a3,a7)/16; cell c -> (c % 4) * 4 + c / 4, XOR (tok & 1) * 4), values
// scaled by 2^e (bf16 input: the chunk max |a| lands in [2^14, 2^15); fp16 input: e = 0).
// S'[chunk][tok] = {1032 * sum_even(a') + 72 * sum_odd(a'), 2^-e, same sum over k < 64, over k >= 64}.
// MODE 1 (group-split consumers, group 64): pieces stay at cell c (XOR (tok & 1) * 4): the consumers'
// word w of thread t is piece 4 w + t there.
template <typename T, int MODE>
__global__ void __launch_bounds__(128) prep_acts_kernel(const T* __restrict__ A, int ntok, int K,
                                                        __half* __restrict__ Ap, float* __restrict__ Sp) {
#ifndef FQ_PREP_EARLY_TRIGGER
#define FQ_PREP_EARLY_TRIGGER 1
#endif
#if FQ_PREP_EARLY_TRIGGER
  // Trigger first: the decode kernel that follows may launch into SM slots the previous GEMM's tail
  // leaves free and start streaming its (constant) weights; it reads A' / S' and writes anything only
  // after its own griddep_wait, i.e. after this grid -- which waits for the previous kernel -- completed.
  griddep_launch_dependents();
  griddep_wait();  // A may be the output of the previous kernel in the stream
#else
  griddep_wait();  // A may be the output of the previous kernel in the stream
  griddep_launch_dependents();
#endif
  const int chunks = K >> 7;
  const int hw = blockIdx.x * 8 + (threadIdx.x >> 4);
  const int l = threadIdx.x & 15;
  if (hw >= ntok * chunks) return;  // whole half-warps exit together
  const unsigned hmask = 0xFFFFu << (threadIdx.x & 16);
  const int tok = hw / chunks, ch = hw - tok * chunks;
  const size_t base = (size_t)tok * K + (size_t)ch * 128;
  const uint4 v = ldg_keep(A + base + l * 8);
  const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
  float f[8];
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
  float inv = 1.f;
  if (Dt<T>::id == FQ_BF16) {
    float mx = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) mx = fmaxf(mx, fabsf(f[e]));
#pragma unroll
    for (int o = 8; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(hmask, mx, o));
    const int E = (int)((__float_as_uint(mx) >> 23) & 0xFF);
    const int F = min(268 - E, 253);  // biased exponent of 2^e, e = 14 - (E - 127)
    const float sc = __uint_as_float((uint32_t)F << 23);
    inv = __uint_as_float((uint32_t)(254 - F) << 23);
#pragma unroll
    for (int e = 0; e < 8; ++e) f[e] *= sc;
  }
  auto h2 = [](float lo, float hi) {
    uint32_t hw2;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(hw2) : "f"(hi), "f"(lo));
    return hw2;
  };
  float sum = fmaf(Nib<__half>::off_even, (f[0] + f[2]) + (f[4] + f[6]),
                   Nib<__half>::off_odd * ((f[1] + f[3]) + (f[5] + f[7])));
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) sum += __shfl_xor_sync(hmask, sum, o);  // 64-k half sums
  const float half_sum = sum, other = __shfl_xor_sync(hmask, sum, 8);
  sum += other;
  const uint4 o = make_uint4(h2(f[0], f[4]), h2(f[1] * 0.0625f, f[5] * 0.0625f), h2(f[2], f[6]),
                             h2(f[3] * 0.0625f, f[7] * 0.0625f));
  const int kl = l * 8, tq = kl >> 5, w16 = (kl & 31) >> 3;
  const int cell = (MODE == 1 ? l : (w16 * 4 + tq)) ^ ((tok & 1) << 2);
  *reinterpret_cast<uint4*>(Ap + base + cell * 8) = o;
  if (l == 0) {
    if (FQ_FOLD2)  // corrections pre-multiplied by -2^-e (exact: power of two)
      *reinterpret_cast<float4*>(Sp + ((size_t)ch * ntok + tok) * 4) =
          make_float4(-sum * inv, inv, -half_sum * inv, -other * inv);
    else
      *reinterpret_cast<float4*>(Sp + ((size_t)ch * ntok + tok) * 4) = make_float4(sum, inv, half_sum, other);
  }
}

// ------------------------------------------------------------------------------------- host side
#ifdef FQ_DIAG
extern "C" int fq_diag_timeline(unsigned long long* host, int nctas, int reset) {
  const int n = nctas < kDiagCtas ? nctas : kDiagCtas;
  if (reset) return (int)cudaMemcpyToSymbol(g_diag_tl, host, (size_t)n * 8 * sizeof(unsigned long long));
  return (int)cudaMemcpyFromSymbol(host, g_diag_tl, (size_t)n * 8 * sizeof(unsigned long long));
}
#endif
static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }
constexpr int kMaxCounters = 16384;
constexpr size_t kCounterBytes = kMaxCounters * sizeof(int);


// Group-split nibble path (int4, group 64, single-problem launches): K % 128 == 0 for the prep.
static bool gs_of(int bits, int group, int K) {
  return FQ_NIB && bits == 4 && group == 64 && K % 128 == 0;
}
static bool nib_of(int bits, int group, int K = -1) {
  return FQ_NIB && bits <= 4 && (group % 128 == 0 || (K >= 0 && gs_of(bits, group, K)));
}

int gemv_max_m(int bits, int group) { return nib_of(bits, group) ? 32 : 16; }

GemvPlan plan_gemv(int M, int K, int N, int bits, int group, int nsm, int splits_override) {
  (void)group;
  GemvPlan p{};
  p.kchunk = bits <= 4 ? 256 : 128;  // split-K granularity (two kernel stages; one stage measured slower on small matrices)
  // 8-token MMA tiles per token tile: 1 (M <= 8), 2 (<= 16), 4 (int4 nibble path, > 16 tokens:
  // every weight is streamed once per 32 tokens)
  p.mt = M <= 8 ? 1 : (M <= 16 || !nib_of(bits, group)) ? 2 : 4;  // MT = 4: group % 128 nibble path only
  p.ktiles = (M + p.mt * 8 - 1) / (p.mt * 8);
  p.rt = 2;
  p.rows_per_cta = kRowsPerCta;
  const int gx = (N + p.rows_per_cta - 1) / p.rows_per_cta;
  const int nchunks = (K + p.kchunk - 1) / p.kchunk;
  const int slots = 2 * nsm;  // 2 CTAs per SM (launch bounds + smem)
  int best_s = 1;
  double best = -1e30;
  const int smax = std::min(nchunks, 64);
  for (int s = 1; s <= smax; ++s) {
    const int klen = ((nchunks + s - 1) / s) * p.kchunk;
    if ((K + klen - 1) / klen != s) continue;
    const double ctas = (double)gx * s * p.ktiles;
    const double waves = ctas / slots;
    const double eff = waves / std::ceil(waves);
    // full last wave first; then as few waves as possible (each CTA pays a pipeline fill) and
    // few splits (partials + fixup).  Measured on B200 (OPT FC1/FC2): 1-2 full waves are best.
    const double score = eff - 0.01 * waves - 0.002 * s;
    if (score > best + 1e-9) { best = score; best_s = s; }
  }
  int s = splits_override > 0 ? splits_override : best_s;
  s = std::max(1, std::min(s, nchunks));
  if ((long long)gx * p.ktiles > kMaxCounters) s = 1;  // counter region is fixed-size
  p.klen = ((nchunks + s - 1) / s) * p.kchunk;
  p.splits = (K + p.klen - 1) / p.klen;
  return p;
}


// Workspace layout (fixed, so buffers can be shared by calls of different shapes):
//   [0, kCounterBytes)  arrival counters (zeroed once by the caller, self-resetting)
//   then split-K fp32 partials [S][M][N] (fully overwritten by every call)
//   then, on the nibble path, the pre-converted activations A' [M][K] fp16 and S' [K/128][M][4].
static size_t prep_bytes(int M, int K) {
  return align256((size_t)M * K * 2) + align256((size_t)(K / 128) * M * 16);
}
size_t gemv_workspace_bytes(const GemvPlan& p, int M, int K, int N, int bits, int group) {
  size_t b = kCounterBytes;
  if (p.splits > 1) b += align256((size_t)p.splits * M * N * sizeof(float));
  if (nib_of(bits, group, K)) b += prep_bytes(M, K);
  return b;
}
size_t gemv_grouped_workspace_bytes(int64_t T, int K, int bits) {
  return kCounterBytes + (bits <= 4 ? prep_bytes((int)T, K) : 0);
}
template <int MODE>
static cudaError_t launch_prep_g(int adt, const void* A, int ntok, int K, void* Ap, void* Sp, cudaStream_t st) {
  const int blocks = (int)(((long long)ntok * (K / 128) + 7) / 8);
  if (blocks == 0) return cudaSuccess;
  if (adt == FQ_BF16)
    return launch_pdl(prep_acts_kernel<__nv_bfloat16, MODE>, blocks, 128, 0, st,
                      reinterpret_cast<const __nv_bfloat16*>(A), ntok, K, reinterpret_cast<__half*>(Ap),
                      reinterpret_cast<float*>(Sp));
  return launch_pdl(prep_acts_kernel<__half, MODE>, blocks, 128, 0, st, reinterpret_cast<const __half*>(A), ntok,
                    K, reinterpret_cast<__half*>(Ap), reinterpret_cast<float*>(Sp));
}
static cudaError_t launch_prep(int adt, const void* A, int ntok, int K, void* Ap, void* Sp, cudaStream_t st,
                               bool gs = false) {
  return gs ? launch_prep_g<1>(adt, A, ntok, K, Ap, Sp, st) : launch_prep_g<0>(adt, A, ntok, K, Ap, Sp, st);
}


template <typename T, int BITS, int MT, int SACC, int DBG, int MAXP>
static cudaError_t launch_dec(const DecBatch<MAXP>& b, int ctas, cudaStream_t st) {
  constexpr int smem = DecStage<BITS, MT, SACC>::SMEM;
  cudaError_t e = ensure_smem_attr<decode_kernel<T, BITS, MT, SACC, DBG, MAXP>>(smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(decode_kernel<T, BITS, MT, SACC, DBG, MAXP>, ctas, dec_threads<FQ_NIB && BITS <= 4 && SACC>(),
                    smem, st, b);
}

template <int MAXP>
static cudaError_t dispatch_dec(int adt, int bits, int mt, int sacc, int dbg, const DecBatch<MAXP>& b,
                                int ctas, cudaStream_t st) {
#ifdef FQ_DIAG
  // diagnostics build only (-DFQ_DIAG, build.build_variant): kernels with parts of the work removed
  if (dbg && adt == FQ_BF16 && bits == 4 && mt == 1 && sacc == 1 && MAXP == 1) {
    if (dbg == 1) return launch_dec<__nv_bfloat16, 4, 1, 1, 1, MAXP>(b, ctas, st);
    if (dbg == 2) return launch_dec<__nv_bfloat16, 4, 1, 1, 2, MAXP>(b, ctas, st);
    if (dbg == 3) return launch_dec<__nv_bfloat16, 4, 1, 1, 3, MAXP>(b, ctas, st);
    if (dbg == 4) return launch_dec<__nv_bfloat16, 4, 1, 1, 4, MAXP>(b, ctas, st);
  }
#else
  (void)dbg;
#endif
#define FQ_DEC_CASE(TT, BB, MM, SS) \
  if (bits == BB && mt == MM && sacc == SS) return launch_dec<TT, BB, MM, SS, 0, MAXP>(b, ctas, st);
  if (adt == FQ_BF16) {
    FQ_DEC_CASE(__nv_bfloat16, 4, 1, 1) FQ_DEC_CASE(__nv_bfloat16, 4, 1, 0)
    FQ_DEC_CASE(__nv_bfloat16, 4, 1, 3) FQ_DEC_CASE(__nv_bfloat16, 4, 2, 3)
    FQ_DEC_CASE(__nv_bfloat16, 4, 2, 1) FQ_DEC_CASE(__nv_bfloat16, 4, 2, 0)
    FQ_DEC_CASE(__nv_bfloat16, 4, 4, 1)
    FQ_DEC_CASE(__nv_bfloat16, 4, 1, 2) FQ_DEC_CASE(__nv_bfloat16, 4, 2, 2)
    FQ_DEC_CASE(__nv_bfloat16, 8, 1, 1) FQ_DEC_CASE(__nv_bfloat16, 8, 1, 0)
    FQ_DEC_CASE(__nv_bfloat16, 8, 2, 1) FQ_DEC_CASE(__nv_bfloat16, 8, 2, 0)
    FQ_DEC_CASE(__nv_bfloat16, 3, 1, 1) FQ_DEC_CASE(__nv_bfloat16, 3, 1, 0)
    FQ_DEC_CASE(__nv_bfloat16, 3, 2, 1) FQ_DEC_CASE(__nv_bfloat16, 3, 2, 0) FQ_DEC_CASE(__nv_bfloat16, 3, 4, 1)
    FQ_DEC_CASE(__nv_bfloat16, 2, 1, 1) FQ_DEC_CASE(__nv_bfloat16, 2, 1, 0)
    FQ_DEC_CASE(__nv_bfloat16, 2, 2, 1) FQ_DEC_CASE(__nv_bfloat16, 2, 2, 0) FQ_DEC_CASE(__nv_bfloat16, 2, 4, 1)
    FQ_DEC_CASE(__nv_bfloat16, 3, 2, 3) FQ_DEC_CASE(__nv_bfloat16, 2, 2, 3)
  } else {
    FQ_DEC_CASE(__half, 4, 1, 1) FQ_DEC_CASE(__half, 4, 1, 0)
    FQ_DEC_CASE(__half, 4, 1, 3) FQ_DEC_CASE(__half, 4, 2, 3)
    FQ_DEC_CASE(__half, 4, 2, 1) FQ_DEC_CASE(__half, 4, 2, 0)
    FQ_DEC_CASE(__half, 4, 4, 1)
    FQ_DEC_CASE(__half, 4, 1, 2) FQ_DEC_CASE(__half, 4, 2, 2)
    FQ_DEC_CASE(__half, 8, 1, 1) FQ_DEC_CASE(__half, 8, 1, 0)
    FQ_DEC_CASE(__half, 8, 2, 1) FQ_DEC_CASE(__half, 8, 2, 0)
    FQ_DEC_CASE(__half, 3, 1, 1) FQ_DEC_CASE(__half, 3, 1, 0)
    FQ_DEC_CASE(__half, 3, 2, 1) FQ_DEC_CASE(__half, 3, 2, 0) FQ_DEC_CASE(__half, 3, 4, 1)
    FQ_DEC_CASE(__half, 2, 1, 1) FQ_DEC_CASE(__half, 2, 1, 0)
    FQ_DEC_CASE(__half, 2, 2, 1) FQ_DEC_CASE(__half, 2, 2, 0) FQ_DEC_CASE(__half, 2, 4, 1)
    FQ_DEC_CASE(__half, 3, 2, 3) FQ_DEC_CASE(__half, 2, 2, 3)
  }
#undef FQ_DEC_CASE
  return cudaErrorInvalidValue;
}

// Fill one batch entry (tensor maps + sizes) for one matrix under plan `pl`.  ws: that problem's
// workspace (counters at offset 0, partials after kCounterBytes).
// nib: A points at the pre-converted A' rows of this problem, Sp at S' column tok_base of a
// [K/128][ntok_all][4] array.
static bool make_dec_prob(DecProb& d, const GemvPlan& pl, int bits, int cdt, const void* A, int M, int K,
                          int N, const void* codes, const void* scales, int group, void* C, void* ws,
                          const void* Sp = nullptr, int ntok_all = 0, int tok_base = 0, bool gs = false,
                          bool ds = false) {
  const uint64_t row_bytes = (uint64_t)K * bits / 8;
  if (!make_tmap_2d(&d.w, codes, 1, row_bytes, (uint64_t)N, row_bytes, wb_row(bits), kWBoxRows,
                    bits >= 4 ? 64 : 0))
    return false;
  const int ks = wb_row(bits) * 8 / bits;  // K per 128-k chunk (one stage unless ds: two)
  if (!make_tmap_2d(&d.a, A, 2, (uint64_t)K, (uint64_t)M, (uint64_t)K * 2, ks * (ds ? 2 : 1), pl.mt * 8, 0))
    return false;
  d.tok_base = tok_base;
  if (Sp && !make_tmap_2d(&d.sm, reinterpret_cast<const char*>(Sp) + (size_t)tok_base * 16, 4, (uint64_t)M * 4,
                          (uint64_t)(K / 128), (uint64_t)ntok_all * 16, pl.mt * 8 * 4, ds ? 2 : 1, 0))
    return false;
  // per-element-scale path (group does not cover a stage): stage the KS / group scale rows by TMA
  // when the group divides the stage (then a power of two >= 16), else read them from global memory
  const int sacc = gs ? 2 : (group % ks == 0 ? 1 : 0);
  d.sc_rows = (!sacc && ks % group == 0) ? ks / group : 0;
  d.sc_shift = d.sc_rows ? __builtin_ctz((unsigned)group) : 0;
  if (!make_tmap_2d(&d.s, scales, 2, (uint64_t)N, (uint64_t)(K / group), (uint64_t)N * 2, kWBoxRows,
                    d.sc_rows ? d.sc_rows : (sacc == 2 || ds ? 2 : 1), 0))
    return false;
  d.scales = scales;
  d.C = C;
  d.M = M; d.K = K; d.N = N; d.group = group; d.cdt = cdt;
  d.klen = pl.klen;
  d.splits = pl.splits;
  d.ktiles = pl.ktiles;
  d.gx = (N + pl.rows_per_cta - 1) / pl.rows_per_cta;
  d.counters = reinterpret_cast<int*>(ws);
  d.ws = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + kCounterBytes);
  return true;
}

#ifndef FQ_DEC_DS
#define FQ_DEC_DS 1
#endif
#ifndef FQ_DEC_DS_MT
#define FQ_DEC_DS_MT 2  // double stages up to two 8-token MMA tiles (MT = 2: 2 stages of 42 KB; -1.5 us at M = 9..16)
#endif
// double stages (kernel SACC == 3): int4 nibble path with one scale group per 128-k chunk, up to
// FQ_DEC_DS_MT 8-token MMA tiles
#ifndef FQ_DEC_DS_LOWBIT
#define FQ_DEC_DS_LOWBIT 1  // int3 / int2 bit streams at 9..16 tokens (measured: -4 / -5 us at M = 16,
#endif                      // +0.5..2 us at M <= 8, where they keep single stages)
static bool ds_of(int bits, int mt, int sacc) {
  const bool lowbit = FQ_DEC_DS_LOWBIT && (bits == 3 || bits == 2) && mt == 2;
  return FQ_DEC_DS && (bits == 4 || lowbit) && sacc == 1 && mt <= FQ_DEC_DS_MT;
}

// scale path: 1 = one scale group per stage, 2 = two 64-k groups (group split), 0 = per element
static int sacc_of(int bits, int group, int K = -1) {
  if (group % (bits <= 4 ? 128 : 64) == 0) return 1;
  return (K >= 0 && gs_of(bits, group, K)) ? 2 : 0;
}

int xr_tile_elems(const GemvPlan& p) { return p.mt * 8 * kRowsPerCta; }
int xr_tiles(const GemvPlan& p, int N) { return ((N + kRowsPerCta - 1) / kRowsPerCta) * p.ktiles; }
cudaError_t run_xr_wait(int32_t* done, int expected, cudaStream_t st) {
  return launch_pdl(xr_wait_kernel, 1, 32, 0, st, done, expected);
}

cudaError_t run_gemv(const GemvPlan& pl, int adt, int cdt, int bits, const void* A, int M, int K,
                     int N, const void* codes, const void* scales, int group, void* C, void* ws,
                     cudaStream_t st, const XRPeers* xr_dev) {
  DecBatch<1> b{};
  // double stages (two 128-k chunks per stage): int4 nibble path, one 8-token MMA tile, groups % 128
  const bool ds = nib_of(bits, group, K) && ds_of(bits, pl.mt, sacc_of(bits, group, K));
  if (nib_of(bits, group, K)) {
    char* pre = reinterpret_cast<char*>(ws) + kCounterBytes +
                (pl.splits > 1 ? align256((size_t)pl.splits * M * N * sizeof(float)) : 0);
    char* Sp = pre + align256((size_t)M * K * 2);
#ifdef FQ_DIAG
    // diagnostics only (FQ_DEC_NOPREP=1): skip the activation pre-conversion (stale A' / S' -- valid
    // only when the same activations were converted by an earlier call): the prep kernel's share of
    // the critical path between back-to-back GEMMs
    static const bool noprep = std::getenv("FQ_DEC_NOPREP") && std::atoi(std::getenv("FQ_DEC_NOPREP"));
    cudaError_t r = noprep ? cudaSuccess : launch_prep(adt, A, M, K, pre, Sp, st, sacc_of(bits, group, K) == 2);
#else
    cudaError_t r = launch_prep(adt, A, M, K, pre, Sp, st, sacc_of(bits, group, K) == 2);
#endif
    if (r != cudaSuccess) return r;
    if (!make_dec_prob(b.p[0], pl, bits, cdt, pre, M, K, N, codes, scales, group, C, ws, Sp, M, 0,
                       sacc_of(bits, group, K) == 2, ds))
      return cudaErrorInvalidValue;
  } else if (!make_dec_prob(b.p[0], pl, bits, cdt, A, M, K, N, codes, scales, group, C, ws)) {
    return cudaErrorInvalidValue;
  }
  b.p[0].cta_begin = 0;
  b.p[0].xr = xr_dev;
  b.nprob = 1;
  const int ctas = b.p[0].gx * pl.splits * pl.ktiles;
#ifdef FQ_DIAG
  const char* dbg_env = std::getenv("FQ_DEC_DEBUG");
  const int dbg = dbg_env ? std::atoi(dbg_env) : 0;
#else
  const int dbg = 0;
#endif
  return dispatch_dec<1>(adt, bits, pl.mt, ds ? 3 : sacc_of(bits, group, K), dbg, b, ctas, st);
}

// ---- MoE batch (kernel A7, decode side): experts listed in `experts` (each with 1 <= M_e <= 16)
// are grouped by (MMA token tiles, scale path) and each group runs as ONE launch over all of its
// experts (<= kMaxBatch per launch; the descriptors travel in the kernel parameter block).
constexpr int kMaxBatch = 48;

cudaError_t run_gemv_grouped(int adt, int cdt, int bits, const void* A, int K, int N,
                             const int64_t* offsets, const int32_t* groups, const void* const* codes,
                             const void* const* scales, void* C, void* ws, int64_t T,
                             const int* experts, int nexp, cudaStream_t st) {
  static_assert(sizeof(DecBatch<kMaxBatch>) < 32000, "kernel parameter block limit");
  // nibble-path experts read A'/S' pre-converted once for all T tokens
  char* pre = reinterpret_cast<char*>(ws) + kCounterBytes;
  char* Sp = pre + align256((size_t)T * K * 2);
  bool any_nib = false;
  for (int ii = 0; ii < nexp; ++ii) any_nib |= nib_of(bits, groups[experts[ii]]);
  if (any_nib) {
    cudaError_t r = launch_prep(adt, A, (int)T, K, pre, Sp, st);
    if (r != cudaSuccess) return r;
  }
  for (int cls = 0; cls < 6; ++cls) {
    const int mt = 1 << (cls >> 1);  // 1, 2, 4 MMA token tiles
    const bool sacc = cls & 1;
    DecBatch<kMaxBatch> b{};
    int ctas = 0;
    for (int ii = 0; ii < nexp; ++ii) {
      const int e = experts[ii];
      const int Me = (int)(offsets[e + 1] - offsets[e]);
      GemvPlan pl = plan_gemv(Me, K, N, bits, groups[e], num_sms());
      // the batch fills the machine by itself: no split-K, so no workspace
      pl.splits = 1;
      pl.klen = ((K + pl.kchunk - 1) / pl.kchunk) * pl.kchunk;
      if (pl.mt != mt || sacc_of(bits, groups[e]) != sacc) continue;
      DecProb& d = b.p[b.nprob];
      const char* Ae = reinterpret_cast<const char*>(A) + (size_t)offsets[e] * K * 2;
      char* Ce = reinterpret_cast<char*>(C) + (size_t)offsets[e] * N * (cdt == FQ_FP32 ? 4 : 2);
      const bool nib = nib_of(bits, groups[e]);
      const void* Ause = nib ? static_cast<const void*>(pre + (size_t)offsets[e] * K * 2) : static_cast<const void*>(Ae);
      if (!make_dec_prob(d, pl, bits, cdt, Ause, Me, K, N, codes[e], scales[e], groups[e], Ce, ws,
                         nib ? Sp : nullptr, (int)T, (int)offsets[e], false, nib && ds_of(bits, mt, sacc)))
        return cudaErrorInvalidValue;
      d.cta_begin = ctas;
      ctas += d.gx * d.splits * d.ktiles;
      if (++b.nprob == kMaxBatch) {
        cudaError_t r = dispatch_dec<kMaxBatch>(adt, bits, mt, ds_of(bits, mt, sacc) ? 3 : sacc, 0, b, ctas, st);
        if (r != cudaSuccess) return r;
        b.nprob = 0;
        ctas = 0;
      }
    }
    if (b.nprob) {
      cudaError_t r = dispatch_dec<kMaxBatch>(adt, bits, mt, ds_of(bits, mt, sacc) ? 3 : sacc, 0, b, ctas, st);
      if (r != cudaSuccess) return r;
    }
  }
  return cudaSuccess;
}

// ---- MoE batch with DEVICE expert offsets (fq_gemm_grouped_dev): every expert is launched with the
// geometry of `Mmax` tokens; each CTA reads its expert's token range from the device and leaves if
// its token tile is empty.  The activation maps span all T rows (tokens are addressed row0 + tok).
cudaError_t run_gemv_grouped_dev(int adt, int cdt, int bits, const void* A, int64_t T, int K, int N,
                                 const int64_t* offs_dev, const int32_t* groups, const void* const* codes,
                                 const void* const* scales, void* C, void* ws, int Mmax, const int* experts,
                                 int nexp, int32_t* status, cudaStream_t st) {
  char* pre = reinterpret_cast<char*>(ws) + kCounterBytes;
  char* Sp = pre + align256((size_t)T * K * 2);
  bool any_nib = false;
  for (int ii = 0; ii < nexp; ++ii) any_nib |= nib_of(bits, groups[experts[ii]]);
  if (any_nib) {
    cudaError_t r = launch_prep(adt, A, (int)T, K, pre, Sp, st);
    if (r != cudaSuccess) return r;
  }
  // Token segments of every expert: [0, 8) on the one-tile kernel class (most experts of a skewed
  // routing are small), then [8, min(bound, decode maximum)) on the class its size needs; the
  // tcgen05 kernel takes whatever exceeds the decode maximum.  A segment's CTAs leave at once when
  // the expert has no tokens there.
  for (int seg = 0; seg < 2; ++seg) {
    for (int cls = 0; cls < 6; ++cls) {
      const int mt = 1 << (cls >> 1);
      const bool sacc = cls & 1;
      DecBatch<kMaxBatch> b{};
      int ctas = 0;
      for (int ii = 0; ii < nexp; ++ii) {
        const int e = experts[ii];
        const int md = std::min(Mmax, gemv_max_m(bits, groups[e]));
        const int t0 = seg == 0 ? 0 : 8, t1 = seg == 0 ? std::min(md, 8) : md;
        if (t1 <= t0) continue;
        GemvPlan pl = plan_gemv(t1 - t0, K, N, bits, groups[e], num_sms());
        pl.splits = 1;
        pl.klen = ((K + pl.kchunk - 1) / pl.kchunk) * pl.kchunk;
        if (pl.mt != mt || sacc_of(bits, groups[e]) != sacc) continue;
        DecProb& d = b.p[b.nprob];
        const bool nib = nib_of(bits, groups[e]);
        if (!make_dec_prob(d, pl, bits, cdt, nib ? static_cast<const void*>(pre) : A, (int)T, K, N, codes[e],
                           scales[e], groups[e], C, ws, nib ? Sp : nullptr, (int)T, 0, false,
                           nib && ds_of(bits, mt, sacc)))
          return cudaErrorInvalidValue;
        d.M = t1 - t0;
        d.tskip = t0;
        d.offs = offs_dev;
        d.e = e;
        d.rows = (int)T;
        d.bound = Mmax;
        d.status = status;
        d.cta_begin = ctas;
        ctas += d.gx * d.ktiles;
        if (++b.nprob == kMaxBatch) {
          cudaError_t r = dispatch_dec<kMaxBatch>(adt, bits, mt, ds_of(bits, mt, sacc) ? 3 : sacc, 0, b, ctas, st);
          if (r != cudaSuccess) return r;
          b.nprob = 0;
          ctas = 0;
        }
      }
      if (b.nprob) {
        cudaError_t r = dispatch_dec<kMaxBatch>(adt, bits, mt, ds_of(bits, mt, sacc) ? 3 : sacc, 0, b, ctas, st);
        if (r != cudaSuccess) return r;
      }
    }
  }
  return cudaSuccess;
}

}  // namespace fq
