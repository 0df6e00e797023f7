// fq_i8.cu — int8-activation x int4-weight path with INTEGER group scales.
//
// The paper's stated future work: "the proposed method does not leverage integer instructions even
// when they are available" (§5) and "using int8 activations and int4 weights with integer
// scales for fine-grained quantization ... has the potential to further enhance the efficiency"
// (§5).  Readings R15-R18:
//   weights      W[n,k] ~ sigma[n] * z[k/g, n] * q[n,k]: sigma fp32 per column, z in [1, 16] an
//                integer per group, q int4 -- so q*z is a signed byte and a whole K-reduction is ONE
//                exact integer dot product (no per-group float fold, unlike the bf16 path);
//   activations  a[m,k] ~ s_a[m] * a_q[m,k], per-token symmetric int8;
//   GEMM         C[m,n] = s_a[m] * sigma[n] * sum_k a_q[m,k] * (q[n,k] * z[k/g,n])   (int32 exact).
//
// Kernels:
//   quantize_intscale_kernel   one CTA per weight column: group maxima -> sigma, z -> codes (offline)
//   quantize_acts_i8_kernel    one CTA per token: row max -> s_a -> int8 codes (every GEMM call)
//   gemm_i8_kernel             tcgen05 "kind::i8" GEMM: the dequant warps turn int4 codes into int8
//                              q*z with one IMAD per 4 codes and write them straight into TMEM as the
//                              MMA's A operand (M = 128 weight rows); B = int8 activations staged by
//                              TMA (K-major SW128); s32 accumulators in TMEM.  The integer tensor-core
//                              MMA does 32 k per instruction (kind::f16: 16), and its per-instruction
//                              cost at N <= 128 is the same (profiles/r02/umma_probe2_i8.txt): twice
//                              the weights per tensor-core cycle of the bf16 path.
#include <cuda.h>

#include <algorithm>
#include <cmath>

#include <cooperative_groups.h>

#include "fq_common.cuh"
#include "fq_internal.h"
#include "fq_tcgen05.cuh"

namespace fq {
namespace i8 {

using namespace tc5;

constexpr int kZ = 16;  // integer scale range [1, kZ] (R15)
#ifndef FQ_I8_DBG
#define FQ_I8_DBG 0  // diagnostics builds only (build_variant): 1 = no MMA, 2 = no unpack / tcgen05.st
#endif

// ------------------------------------------------------------------------------ block reductions
__device__ __forceinline__ float block_max(float v, float* red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float r = 0.f;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r = fmaxf(r, red[i]);
  return r;
}
__device__ __forceinline__ int block_or(int v, int* red) {
  v = __any_sync(0xffffffffu, v) ? 1 : 0;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  int r = 0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r |= red[i];
  return r;
}

template <typename T>
__device__ __forceinline__ void load8(const T* p, float (&f)[8]) {
  if constexpr (sizeof(T) == 4) {
    const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
  } else {
    const uint4 v = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if constexpr (Dt<T>::id == FQ_BF16) {
        f[2 * i] = __uint_as_float(w[i] << 16);
        f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
      } else {
        const float2 h = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
        f[2 * i] = h.x;
        f[2 * i + 1] = h.y;
      }
    }
  }
}

// ---------------------------------------------------------------- weights: integer group scales
// One CTA per column n (row n of W [N, K]).  Pass 1: group maxima (exact) into shared memory;
// sigma = RN_fp32(2 amax_col / 240) (IEEE division, R16); z_j = clamp(ceil((2 amax_j) / (15 sigma)),
// 1, 16) in float64; pass 2 (W re-read from L1/L2): q = clamp(round_half_away(w / (sigma z)), -8, 7)
// in float64 (sigma z exact), packed low nibble first.  Non-finite W: sigma 0, z 1, codes 0, status.
template <typename T>
__global__ void __launch_bounds__(256) quantize_intscale_kernel(const T* __restrict__ W, int K, int N, int group,
                                                                uint8_t* __restrict__ codes, uint8_t* __restrict__ z,
                                                                float* __restrict__ sigma, int32_t* status) {
  extern __shared__ uint32_t s_amax[];  // [G] group maxima as fp32 bits (non-negative: int order)
  __shared__ float red[8];
  __shared__ int redi[8];
  const int n = blockIdx.x;
  const int G = K / group;
  const T* row = W + (size_t)n * K;
  for (int j = threadIdx.x; j < G; j += blockDim.x) s_amax[j] = 0u;
  __syncthreads();
  int bad = 0;
  float cmax = 0.f;
  for (int c = threadIdx.x; c < K / 8; c += blockDim.x) {
    float f[8];
    load8(row + c * 8, f);
    float m = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      bad |= !isfinite(f[i]);
      m = fmaxf(m, fabsf(f[i]));
    }
    atomicMax(&s_amax[(c * 8) / group], __float_as_uint(m));  // chunks of 8 never straddle groups
    cmax = fmaxf(cmax, m);
  }
  cmax = block_max(cmax, red);
  bad = block_or(bad, redi);
  const float sg = bad ? 0.f : __fdiv_rn(2.f * cmax, 240.f);  // 2 amax / ((2^4 - 1) * 16)
  if (threadIdx.x == 0) {
    sigma[n] = sg;
    if (bad && status) atomicOr(status, 1);
  }
  const double s15 = 15.0 * (double)sg;  // exact
  for (int j = threadIdx.x; j < G; j += blockDim.x) {
    int zj = 1;
    if (sg > 0.f) {
      const double r = __ddiv_rn(2.0 * (double)__uint_as_float(s_amax[j]), s15);
      zj = (int)fmin(fmax(ceil(r), 1.0), (double)kZ);
    }
    s_amax[j] = (uint32_t)zj;  // reuse: z per group
    z[(size_t)j * N + n] = (uint8_t)zj;
  }
  __syncthreads();
  uint32_t* out = reinterpret_cast<uint32_t*>(codes + (size_t)n * (K / 2));
  for (int c = threadIdx.x; c < K / 8; c += blockDim.x) {
    uint32_t word = 0;
    if (sg > 0.f) {
      float f[8];
      load8(row + c * 8, f);
      const double S = (double)sg * (double)s_amax[(c * 8) / group];  // exact in float64
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const double y = __ddiv_rn((double)f[i], S);
        const int q = (int)fmin(fmax(round(y), -8.0), 7.0);  // round(): half away from zero
        word |= (uint32_t)(q & 0xF) << (4 * i);
      }
    }
    out[c] = word;
  }
}

// ---------------------------------------------------------------- activations: per-token int8
// One CTA per token m: amax -> s_a = RN_fp32(amax / 127) (IEEE division) -> a_q =
// clamp(round_half_away(fp32(a / s_a)), -127, 127) (R17).  Non-finite row: s_a 0, codes 0, status.
template <typename T>
__global__ void __launch_bounds__(1024) quantize_acts_i8_kernel(const T* __restrict__ A, int K, int8_t* __restrict__ Aq,
                                                               float* __restrict__ sa, int32_t* __restrict__ rowsum,
                                                               int32_t* status) {
  __shared__ float red[32];
  __shared__ int redi[32];
#ifndef FQ_I8_EARLY_TRIGGER
#define FQ_I8_EARLY_TRIGGER 1
#endif
  // The GEMM that follows may launch at once and stream its (constant) weights while this runs; it
  // reads a_q / s_a / rowsum only after its own griddep_wait (this grid complete).
  if (FQ_I8_EARLY_TRIGGER) griddep_launch_dependents();
  griddep_wait();  // A may be the previous kernel's output
  const int m = blockIdx.x;
  const T* row = A + (size_t)m * K;
  float mx = 0.f;
  int bad = 0;
  for (int c = threadIdx.x; c < K / 8; c += blockDim.x) {
    float f[8];
    load8(row + c * 8, f);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      bad |= !isfinite(f[i]);
      mx = fmaxf(mx, fabsf(f[i]));
    }
  }
  mx = block_max(mx, red);
  bad = block_or(bad, redi);
  const float s = bad ? 0.f : __fdiv_rn(mx, 127.f);
  if (threadIdx.x == 0) {
    sa[m] = s;
    if (bad && status) atomicOr(status, 1);
  }
  uint2* out = reinterpret_cast<uint2*>(Aq + (size_t)m * K);
  int sum = 0;
  for (int c = threadIdx.x; c < K / 8; c += blockDim.x) {
    uint32_t w[2] = {0u, 0u};
    if (s > 0.f) {
      float f[8];
      load8(row + c * 8, f);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float q = fminf(fmaxf(roundf(__fdiv_rn(f[i], s)), -127.f), 127.f);  // roundf: half away
        sum += (int)q;
        // k-interleaved word: even k in bytes 0..3, odd k in bytes 4..7 (matches the GEMM's A bytes)
        w[i & 1] |= ((uint32_t)(int)q & 0xFFu) << (8 * (i >> 1));
      }
    }
    out[c] = make_uint2(w[0], w[1]);
  }
  // the code sum of the row (the GEMM's biased-weight correction, see gemm_i8_kernel)
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) redi[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += redi[i];
    rowsum[m] = t;
  }
  if (!FQ_I8_EARLY_TRIGGER) griddep_launch_dependents();
}

// Few tokens (decode): one 8-CTA cluster per token, each CTA a contiguous K/8 slice, the row max and
// the code sum reduced across the cluster through distributed shared memory (no global atomics, no
// zero-initialised scratch) -- the same s_a, codes and rowsum as the one-CTA kernel, with 8x the
// SMs on the row (a 98 KB OPT-175B FC2 row took one SM ~8 us).
constexpr int kActCluster = 8;
template <typename T>
__global__ void __cluster_dims__(kActCluster, 1, 1) __launch_bounds__(256)
    quantize_acts_i8_cluster_kernel(const T* __restrict__ A, int K, int8_t* __restrict__ Aq, float* __restrict__ sa,
                                    int32_t* __restrict__ rowsum, int32_t* status) {
  namespace cg = cooperative_groups;
  __shared__ float red[32];
  __shared__ int redi[32];
  __shared__ float c_max;
  __shared__ int c_bad, c_sum;
  // the GEMM that follows may launch at once (it reads a_q / s_a / rowsum after its griddep_wait)
  griddep_launch_dependents();
  griddep_wait();  // A may be the previous kernel's output
  cg::cluster_group cl = cg::this_cluster();
  const int r = (int)cl.block_rank();
  const int m = blockIdx.x / kActCluster;
  const int slice = K / kActCluster;  // a multiple of 8 (host: K % 64 == 0)
  const T* row = A + (size_t)m * K + (size_t)r * slice;
  float mx = 0.f;
  int bad = 0;
  for (int c = threadIdx.x; c < slice / 8; c += blockDim.x) {
    float f[8];
    load8(row + c * 8, f);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      bad |= !isfinite(f[i]);
      mx = fmaxf(mx, fabsf(f[i]));
    }
  }
  mx = block_max(mx, red);
  bad = block_or(bad, redi);
  if (threadIdx.x == 0) {
    c_max = mx;
    c_bad = bad;
  }
  cl.sync();
  float gmx = 0.f;
  int gbad = 0;
#pragma unroll
  for (int i = 0; i < kActCluster; ++i) {
    gmx = fmaxf(gmx, *cl.map_shared_rank(&c_max, i));
    gbad |= *cl.map_shared_rank(&c_bad, i);
  }
  const float s = gbad ? 0.f : __fdiv_rn(gmx, 127.f);
  uint2* out = reinterpret_cast<uint2*>(Aq + (size_t)m * K + (size_t)r * slice);
  int sum = 0;
  for (int c = threadIdx.x; c < slice / 8; c += blockDim.x) {
    uint32_t w[2] = {0u, 0u};
    if (s > 0.f) {
      float f[8];
      load8(row + c * 8, f);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float q = fminf(fmaxf(roundf(__fdiv_rn(f[i], s)), -127.f), 127.f);  // roundf: half away
        sum += (int)q;
        w[i & 1] |= ((uint32_t)(int)q & 0xFFu) << (8 * (i >> 1));  // k-interleaved word
      }
    }
    out[c] = make_uint2(w[0], w[1]);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) redi[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += redi[i];
    c_sum = t;
  }
  cl.sync();
  if (r == 0 && threadIdx.x == 0) {
    int t = 0;
    for (int i = 0; i < kActCluster; ++i) t += *cl.map_shared_rank(&c_sum, i);
    rowsum[m] = t;
    sa[m] = s;
    if (gbad && status) atomicOr(status, 1);
  }
  cl.sync();  // every CTA's shared memory stays alive until rank 0 has read it
}

// ---------------------------------------------------------------- tcgen05 kind::i8 GEMM
constexpr int BM = 128;     // weight rows per tile (UMMA M, TMEM lanes)
constexpr int BK = 128;     // k per stage: one 128-byte SW128 activation row, 64-byte code rows
constexpr int ZROWS = 4;    // z rows staged per K block (groups of >= 32 k)
constexpr int kGroupWarps = 8;  // dequant warps per group: two per TMEM lane quarter, 64 k each
// DG dequant groups take alternate K blocks (one group's barrier waits and tcgen05.st round trip
// overlap the other's loads and unpacking).  Threads: codes TMA, MMA, 8 DG dequant, activation TMA.
__host__ __device__ constexpr int i8_threads(int dg) { return 32 * (3 + kGroupWarps * dg); }
#ifndef FQ_I8_DG_SMALL
#define FQ_I8_DG_SMALL 2  // token tiles <= 32
#endif
#ifndef FQ_I8_SMALL_CPS
#define FQ_I8_SMALL_CPS 2  // CTAs per SM for token tiles <= 32 (measured: FC1 M=1 102 -> 79 us,
                           // FC2 97 -> 67 us; profiles/r02/i8_two_ctas_per_sm.txt)
#endif
#ifndef FQ_I8_MID_CPS
#define FQ_I8_MID_CPS 2    // CTAs per SM for token tiles of 33..64 (the 64-token variant; measured:
                           // OPT-175B M=64 114 -> 87 us FC1, 111 -> 84 us FC2)
#endif
#ifndef FQ_I8_128_CPS
#define FQ_I8_128_CPS 2    // CTAs per SM for token tiles of 65..128 (FC2 M=96 117 -> 95 us, M=128 124 -> 104)
#endif
#ifndef FQ_I8_DG_LARGE
#define FQ_I8_DG_LARGE 2  // measured (profiles/r02/i8_dequant_groups.txt): M = 64 -10%, M = 2048 -9%
#endif
constexpr int kSmemMax = 227 * 1024 - 2048;

// Two rings per CTA:
//   codes ring (CS stages of 128 rows x 64 B int4 codes + the K block's z rows), released by the
//     dequant warps as soon as the codes are in registers -- its turnover is HBM latency + unpack,
//     never the tensor core, so few bytes of smem keep many code bytes in flight (decode);
//   activation ring (AS stages of bn x 128 B int8 activations) + one TMEM A slot (32 columns) per
//     stage, released by the MMA commit.
// CPS CTAs per SM (2 for decode-sized token tiles: two independent pipelines per SM) split the
// SM's tensor memory and shared memory.
template <int BNMAX, int CPS = 1>
struct Geo {
  static constexpr int TMEM_COLS = 512 / CPS;
  static constexpr int SMEM_MAX = (kSmemMax + 2048) / CPS - 2048;
  static constexpr int ACT_STAGE = BNMAX * BK;                 // int8 [bn][128] SW128 (UMMA B)
  static constexpr int CODE_BYTES = BM * BK / 2;               // int4 [128][64 B] SW64
  static constexpr int Z_OFS = CODE_BYTES;                     // z rows [ZROWS][128] after the codes
  static constexpr int CODE_STAGE = CODE_BYTES + ZROWS * BM;   // 8704 (a multiple of 512)
  static constexpr int AS_TMEM = (TMEM_COLS - BNMAX) / (BK / 4);
  static constexpr int AS_SMEM = (BNMAX >= 256 ? 160 * 1024 : 96 * 1024) / CPS / ACT_STAGE;
  static constexpr int AS0 = AS_TMEM < AS_SMEM ? AS_TMEM : AS_SMEM;
  static constexpr int AS = AS0 > 12 ? 12 : AS0;
  static constexpr int CODE_OFS = AS * ACT_STAGE;
  static constexpr int CS0 = (SMEM_MAX - 1024 - CODE_OFS) / CODE_STAGE;
  static constexpr int CS = CS0 > 20 ? 20 : CS0;
  static constexpr int SMEM = CODE_OFS + CS * CODE_STAGE + 1024;
  static_assert(AS >= 3 && CS >= 4, "stages");
};

struct I8Prob {
  CUtensorMap a;     // a_q [M][K] int8, box [128 B][bn rows], SWIZZLE_128B
  CUtensorMap q;     // codes [N][K/2], box [64 B][128 rows], SWIZZLE_64B
  CUtensorMap z;     // z [G][N] u8, box [128 cols][ZROWS rows]
  const float* sa;   // [M]
  const int32_t* rowsum;  // [M] sum_k a_q[m, k] (bias correction)
  const float* sigma;// [N]
  void* C;
  int M, K, N, group, cdt;
  int bn, m_tiles, n_tiles, gm;
  int splits, kbs;   // split-K: items of kbs K blocks
  int32_t* ws;       // split-K int32 partials [tiles * splits][bn][128]
  int* ctr;          // arrival counters per output tile (self-resetting)
};

__device__ __forceinline__ void tile_coords(int tile, int m_tiles, int n_tiles, int GM, int& mt, int& nt) {
  const int group = tile / (GM * n_tiles);
  const int gm = min(GM, m_tiles - group * GM);
  const int local = tile - group * GM * n_tiles;
  mt = group * GM + local % gm;
  nt = local / gm;
}

__device__ __forceinline__ void mma_i8_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// kind::i8 instruction descriptor: D s32, A u8 (biased weights), B s8 (activations), K-major both,
// M = 128, N = n
__device__ __forceinline__ uint32_t idesc_i8(int n) {
  return (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
  uint32_t r;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(r) : "r"(addr));
  return r;
}

// 16-byte chunk c of code row r in shared memory under SWIZZLE_64B
__device__ __forceinline__ int swz64c(int c, int r) { return c ^ ((r >> 1) & 3); }

// 8 int4 codes (one word, code k + i at nibble i) times the integer scale z -> 8 UNSIGNED bytes
// q*z + 128 in the k-interleaved order (k, k+2, k+4, k+6 | k+1, k+3, k+5, k+7) that
// fq_quantize_acts_i8 also stores the activations in (a_q layout, fq.h), so no byte shuffle is
// needed.  u = q + 8 per byte (mask + XOR in one LOP3); u * z + (128 - 8 z) = q*z + 128 per byte stays
// in [0, 240] (no carry between bytes), so one IMAD scales four codes.  The MMA takes A as u8; the
// bias adds 128 * sum_k a_q[m,k] to every output of token m, which the epilogue removes with the
// activation row sums (exact integers).
__device__ __forceinline__ void i4z_bytes(uint32_t w, uint32_t z, uint32_t cz, uint32_t& o0, uint32_t& o1) {
  o0 = lop3_and_xor(w, 0x0F0F0F0Fu, 0x08080808u) * z + cz;       // k, k+2, k+4, k+6
  o1 = lop3_and_xor(w >> 4, 0x0F0F0F0Fu, 0x08080808u) * z + cz;  // k+1, k+3, k+5, k+7
}

template <int BNMAX, int DG, int CPS>
__global__ void __launch_bounds__(i8_threads(DG), CPS) gemm_i8_kernel(const __grid_constant__ I8Prob p) {
  constexpr int kDqWarps = kGroupWarps * DG;
  constexpr int kThreads = i8_threads(DG);
  using Gm = Geo<BNMAX, CPS>;
  constexpr int CS = Gm::CS, AS = Gm::AS;
  constexpr int kACol = BNMAX;  // A slot a at TMEM columns BNMAX + 32 a
  extern __shared__ __align__(1024) uint8_t dsmem[];
  __shared__ __align__(8) uint64_t cfull[CS], cempty[CS], actfull[AS], slotfull[AS], aempty[AS];
  __shared__ __align__(8) uint64_t acc_full, acc_empty;
  __shared__ uint32_t tmem_base_sh;
  __shared__ int s_last;
  uint8_t* sbase = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsmem) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = p.m_tiles * p.n_tiles * p.splits;
  const int kblocks = p.K / BK;

  if (threadIdx.x == 0) {
    for (int c = 0; c < CS; ++c) {
      mbar_init(&cfull[c], 1);
      mbar_init(&cempty[c], kGroupWarps);
    }
    for (int a = 0; a < AS; ++a) {
      mbar_init(&actfull[a], 1);
      mbar_init(&slotfull[a], kGroupWarps);
      mbar_init(&aempty[a], 1);
    }
    mbar_init(&acc_full, 1);
    mbar_init(&acc_empty, kDqWarps);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&tmem_base_sh, Gm::TMEM_COLS);
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.a);
    prefetch_tmap(&p.q);
    prefetch_tmap(&p.z);
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tmem_base_sh;

  auto item_coords = [&](int item, int& mt, int& nt, int& tt, int& ks, int& kb0, int& kb1) {
    tt = item / p.splits;
    ks = item - tt * p.splits;
    tile_coords(tt, p.m_tiles, p.n_tiles, p.gm, mt, nt);
    kb0 = ks * p.kbs;
    kb1 = min(kblocks, kb0 + p.kbs);
  };

  if (warp == 0) {
    // ------------------------------------------------------------------ codes producer (TMA)
    // weights are constants: no griddep_wait, so the codes stream starts while the previous
    // kernel (the activation quantizer) is still running (programmatic dependent launch)
    if (lane == 0) {
      const uint64_t pol_q = policy_evict_first();
      int c = 0;
      uint32_t ph = 0;
      for (int item = blockIdx.x; item < ntiles; item += gridDim.x) {
        int mt, nt, tt, ks, kb0, kb1;
        item_coords(item, mt, nt, tt, ks, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&cempty[c], ph ^ 1);
          uint8_t* st = sbase + Gm::CODE_OFS + c * Gm::CODE_STAGE;
          mbar_arrive_expect_tx(&cfull[c], Gm::CODE_STAGE);
          tma_load_2d(st, &p.q, &cfull[c], kb * (BK / 2), nt * BM, pol_q);
          tma_load_2d(st + Gm::Z_OFS, &p.z, &cfull[c], nt * BM, (kb * BK) / p.group, pol_q);
          if (++c == CS) { c = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == kThreads / 32 - 1) {
    // ------------------------------------------------------------------ activation producer (TMA)
    if (lane == 0) {
      const uint64_t pol_a = policy_evict_last();
      griddep_wait();  // the activations come from the previous kernel (fq_quantize_acts_i8)
      int a = 0;
      uint32_t ph = 0;
      for (int item = blockIdx.x; item < ntiles; item += gridDim.x) {
        int mt, nt, tt, ks, kb0, kb1;
        item_coords(item, mt, nt, tt, ks, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&aempty[a], ph ^ 1);
          mbar_arrive_expect_tx(&actfull[a], p.bn * BK);
          tma_load_2d(sbase + a * Gm::ACT_STAGE, &p.a, &actfull[a], kb * BK, mt * p.bn, pol_a);
          if (++a == AS) { a = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t sb = smem_u32(sbase);
      const uint32_t idesc = idesc_i8(p.bn);
      int a = 0;
      uint32_t ph = 0, acc_ph = 0;
      for (int item = blockIdx.x; item < ntiles; item += gridDim.x) {
        int mt, nt, tt, ks, kb0, kb1;
        item_coords(item, mt, nt, tt, ks, kb0, kb1);
        mbar_wait(&acc_empty, acc_ph ^ 1);
        fence_after();
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&actfull[a], ph);    // activations landed (TMA)
          mbar_wait(&slotfull[a], ph);   // A operand written to TMEM by the dequant warps
          fence_after();
          const uint64_t bdesc = sw128_desc(sb + a * Gm::ACT_STAGE);
#pragma unroll
          for (int kk = 0; kk < BK / 32; ++kk)
            if (!(FQ_I8_DBG & 1))
              mma_i8_ts(tmem, tmem + kACol + a * (BK / 4) + kk * 8, bdesc + (uint64_t)(kk * 2), idesc,
                        (kb != kb0) || (kk != 0));
          mma_commit(&aempty[a]);        // frees the activation stage and the TMEM A slot
          if (++a == AS) { a = 0; ph ^= 1; }
        }
        mma_commit(&acc_full);
        acc_ph ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------------ dequant + epilogue
    const int dq = warp - 2;
    const int quarter = warp & 3;          // TMEM lane quarter this warp may access
    const int kp = (dq >> 2) & 1;          // which 64 k of a K block this warp dequantizes
    const int grp = dq >> 3;               // dequant group: K blocks with blk % DG == grp
    const int row = quarter * 32 + lane;   // weight row within the tile == TMEM lane
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t sb = smem_u32(sbase);
    uint32_t acc_ph = 0;
    int blk = 0;  // K blocks of this CTA so far (ring position of both rings)
    // groups divide the 128-k block (32 / 64) or are whole blocks (g % 128 == 0): the staged z row of
    // each of this thread's two 32-k chunks is fixed (host-validated)
    const int jr0 = p.group >= BK ? 0 : (kp * 64) / p.group;
    const int jr1 = p.group >= BK ? 0 : (kp * 64 + 32) / p.group;
    const uint32_t codes_row = sb + Gm::CODE_OFS + row * 64;
    const uint32_t c0ofs = swz64c(kp * 2, row) << 4, c1ofs = swz64c(kp * 2 + 1, row) << 4;
    const uint32_t z0ofs = Gm::CODE_OFS + Gm::Z_OFS + jr0 * BM + row;
    const uint32_t z1ofs = Gm::CODE_OFS + Gm::Z_OFS + jr1 * BM + row;
    const uint32_t tcol = tmem + lane_base + kACol + kp * 16;
    for (int item = blockIdx.x; item < ntiles; item += gridDim.x) {
      int mt, nt, tt, ks, kb0, kb1;
      item_coords(item, mt, nt, tt, ks, kb0, kb1);
      int prev = -1;  // (DG == 1) A slot written but not yet published (its tcgen05.st in flight)
      for (int kb = kb0; kb < kb1; ++kb, ++blk) {
        if (DG > 1 && (blk % DG) != grp) continue;
        const int c = blk % CS, a = blk % AS;
        const uint32_t cph = (blk / CS) & 1, aph = (blk / AS) & 1;
        mbar_wait(&cfull[c], cph);
        const uint32_t so = c * Gm::CODE_STAGE;
        const uint4 w0 = lds128(codes_row + so + c0ofs);
        const uint4 w1 = lds128(codes_row + so + c1ofs);
        const uint32_t z0 = lds_u8(sb + so + z0ofs), z1 = lds_u8(sb + so + z1ofs);
        __syncwarp();
        if (lane == 0) mbar_arrive(&cempty[c]);  // codes in registers: the stage goes back to the TMA
        uint32_t out[16];
        const uint32_t cz0 = 0x80808080u - z0 * 0x08080808u, cz1 = 0x80808080u - z1 * 0x08080808u;
        i4z_bytes(w0.x, z0, cz0, out[0], out[1]);
        i4z_bytes(w0.y, z0, cz0, out[2], out[3]);
        i4z_bytes(w0.z, z0, cz0, out[4], out[5]);
        i4z_bytes(w0.w, z0, cz0, out[6], out[7]);
        i4z_bytes(w1.x, z1, cz1, out[8], out[9]);
        i4z_bytes(w1.y, z1, cz1, out[10], out[11]);
        i4z_bytes(w1.z, z1, cz1, out[12], out[13]);
        i4z_bytes(w1.w, z1, cz1, out[14], out[15]);
        // DG == 1: publish the previous A slot (its tcgen05.st had this block's loads and unpacking
        // to complete); then wait until the MMAs that last read this block's slot are done
        if (DG == 1 && prev >= 0) {
          tmem_wait_st();
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&slotfull[prev]);
        }
        mbar_wait(&aempty[a], aph ^ 1);
        fence_after();
        if (FQ_I8_DBG & 2) {
          if (out[0] == 0x12345678u && out[15] == 0x9u) tmem_st16(tcol + a * (BK / 4), out);  // keep the unpack alive
        } else {
          tmem_st16(tcol + a * (BK / 4), out);
        }
        if (DG == 1) {
          prev = a;
        } else {  // the other group covers this group's tcgen05.st round trip
          tmem_wait_st();
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&slotfull[a]);
        }
      }
      if (DG == 1 && prev >= 0) {
        tmem_wait_st();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&slotfull[prev]);
      }
      // ---- epilogue: accumulator row `row` (weight n), tokens [part * TPP, +TPP), part = dq / 4
      mbar_wait(&acc_full, acc_ph);
      acc_ph ^= 1;
      fence_after();
      constexpr int TPP = BNMAX / (2 * DG);
      constexpr int CH = TPP < 16 ? TPP : 16;  // accumulator columns per tcgen05.ld
      const int part_i = dq >> 2;
      const int n = nt * BM + row;
      int32_t* part = p.splits > 1 ? p.ws + (size_t)(tt * p.splits + ks) * p.bn * BM : nullptr;
      const float sg = n < p.N ? __ldg(p.sigma + n) : 0.f;
#pragma unroll 1
      for (int c0 = 0; c0 < TPP && part_i * TPP + c0 < p.bn; c0 += CH) {
        uint32_t v[CH];
        tmem_ldn<CH>(tmem + lane_base + part_i * TPP + c0, v);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < CH; ++i) {
          const int tl = part_i * TPP + c0 + i;  // token within the tile
          if (tl >= p.bn) continue;
          if (part) {
            __stcg(part + tl * BM + row, (int32_t)v[i]);
          } else {
            const int tok = mt * p.bn + tl;
            if (tok < p.M && n < p.N) {
              const int32_t acc = (int32_t)v[i] - 128 * __ldg(p.rowsum + tok);
              const float f = (float)acc * __ldg(p.sa + tok) * sg;
              const size_t o = (size_t)tok * p.N + n;
              if (p.cdt == FQ_FP32) reinterpret_cast<float*>(p.C)[o] = f;
              else if (p.cdt == FQ_BF16) reinterpret_cast<__nv_bfloat16*>(p.C)[o] = __float2bfloat16_rn(f);
              else reinterpret_cast<__half*>(p.C)[o] = __float2half_rn(f);
            }
          }
        }
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty);
      if (part) {
        // last-arriving split of the output tile sums the int32 partials (exact) and scales them
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kDqWarps));
        if (threadIdx.x == 64) {
          __threadfence();
          const int last = atomicAdd(&p.ctr[tt], 1) == p.splits - 1;
          if (last) __threadfence();
          s_last = last;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kDqWarps));
        if (s_last) {
          const int tid = threadIdx.x - 64, r = tid & (BM - 1);
          const int nr = nt * BM + r;
          const int tmax = min(p.bn, p.M - mt * p.bn);
          const int32_t* base = p.ws + (size_t)tt * p.splits * p.bn * BM;
          if (nr < p.N) {
            const float sgr = __ldg(p.sigma + nr);
            constexpr int NPAR = kDqWarps * 32 / BM;  // threads per row
            for (int tl0 = tid / BM; tl0 < tmax; tl0 += 8 * NPAR) {  // 8 tokens' loads in flight
              int32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
              for (int q = 0; q < p.splits; ++q)
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                  const int tl = tl0 + NPAR * u;
                  if (tl < tmax) acc[u] += __ldcg(base + ((size_t)q * p.bn + tl) * BM + r);
                }
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const int tl = tl0 + NPAR * u;
                if (tl >= tmax) break;
                const int tok = mt * p.bn + tl;
                const float f = (float)(acc[u] - 128 * __ldg(p.rowsum + tok)) * __ldg(p.sa + tok) * sgr;
                const size_t o = (size_t)tok * p.N + nr;
                if (p.cdt == FQ_FP32) reinterpret_cast<float*>(p.C)[o] = f;
                else if (p.cdt == FQ_BF16) reinterpret_cast<__nv_bfloat16*>(p.C)[o] = __float2bfloat16_rn(f);
                else reinterpret_cast<__half*>(p.C)[o] = __float2half_rn(f);
              }
            }
          }
          if (threadIdx.x == 64) p.ctr[tt] = 0;  // self-reset
        }
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    fence_after();
    tmem_dealloc(tmem, Gm::TMEM_COLS);
  }
}


// ---------------------------------------------------------------- decode (M <= 16): legacy IMMA
// Decode sizes stream every weight once per call and are bound by HBM, not by the tensor core, so
// the tcgen05 kernel above (one 128-row UMMA per 64 weights x 16 k, N padded to 32) is not needed
// there.  This kernel is the bf16 decode kernel's structure (fq_gemv.cu: TMA producer warp, 8
// consumer warps x 32 weight rows, 256-row CTA tiles, 128-k stages, split-K with a deterministic
// last-arriver fixup) on the integer path: each code word becomes the biased u8 weights q z + 128
// with one LOP3 + one IMAD per 4 codes (as above), and mma.sync m16n8k32 u8 x s8 -> s32 takes 32 k
// per instruction (twice bf16's m16n8k16).  The whole K accumulates exactly in int32 (no per-group
// fold: z is inside the weights); the epilogue removes 128 * rowsum and applies s_a * sigma once.
// MMA k-slot mapping (k-step j of a 128-k stage): thread t's slots 4t..4t+3 hold the even k of the
// 8-k block 4t + j and slots 16+4t..16+4t+3 its odd k -- exactly the k-interleaved words of both the
// code nibbles (low / high nibbles) and fq_quantize_acts_i8's a_q layout.
constexpr int kDecRows = 256;
constexpr int kDecWarps = 8;
constexpr int kDecThreads = 32 * (1 + kDecWarps);
// NC 128-k chunks per stage (2: the code, activation and z TMAs of two chunks share one barrier
// round trip, as in the bf16 kernel's double stages)
template <int MT, int NC>
struct DecI8Geo {
  static constexpr int CODE1 = kDecRows * 64;  // one chunk: [256 rows][64 B] int4, SWIZZLE_64B
  static constexpr int ACT1 = MT * 8 * 128;    // one chunk: [MT*8 tokens][128 B] int8, SWIZZLE_128B
  static constexpr int CODE = NC * CODE1;
  static constexpr int ACT = NC * ACT1;
  static constexpr int ZB = 4 * NC * kDecRows;  // up to 4 NC z rows [.][256] u8 (groups of 32)
  static constexpr int PER = ((CODE + ACT + ZB + 1023) / 1024) * 1024;
  static constexpr int N0 = (115712 - 2048) / PER;
  static constexpr int N = N0 > 8 ? 8 : N0;
  static constexpr int SMEM = N * PER + 1024;
};
struct DecI8Prob {
  CUtensorMap a;  // a_q [M][K] int8, box [128 B][MT*8 rows], SWIZZLE_128B
  CUtensorMap q;  // codes [N][K/2], box [64 B][256 rows], SWIZZLE_64B
  CUtensorMap z;  // z [G][N] u8, box [256 cols][zr rows]
  const float* sa;
  const int32_t* rowsum;
  const float* sigma;
  void* C;
  int32_t* ws;    // split-K int32 partials [splits][M][N]
  int* ctr;       // per column tile, self-resetting
  int M, K, N, group, cdt, zr, gx, splits, klen;
};

__device__ __forceinline__ void imma16832(int (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int MT, int NC>
// two 9-warp CTAs per SM: <= 96 registers (18 warps put 5 on some sub-partition's 16K register bank).
// (Four 8-token tiles for 17..32 tokens were measured: FC2 M = 17..32 82-86 us vs 73-78 us on the
// tcgen05 kernel, FC1 equal -- so the IMMA kernel stops at 16 tokens.)
__global__ void __maxnreg__(96) decode_i8_kernel(const __grid_constant__ DecI8Prob p) {
  using G = DecI8Geo<MT, NC>;
  constexpr int NSTG = G::N;
  constexpr int KST = 128 * NC;  // K per stage
  extern __shared__ __align__(1024) uint8_t dsmem[];
  __shared__ __align__(8) uint64_t full_bar[8], empty_bar[8];
  __shared__ int s_last;
  uint8_t* sbase = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsmem) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bx = (int)blockIdx.x % p.gx, by = (int)blockIdx.x / p.gx;
  const int n0 = bx * kDecRows;
  const int kbeg = by * p.klen, kend = min(p.K, kbeg + p.klen);
  const int nst = (kend - kbeg + KST - 1) / KST;  // K % 128 == 0 (ABI); a past-K chunk is TMA zero fill
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTG; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kDecWarps);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.q);
    prefetch_tmap(&p.z);
    prefetch_tmap(&p.a);
  }
  __syncthreads();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (one lane)
    if (lane == 0) {
      const uint64_t polw = policy_evict_first(), pola = policy_evict_last();
      auto issue_w = [&](int i, int s) {
        uint8_t* st = sbase + s * G::PER;
        const int k0 = kbeg + i * KST;
        mbar_arrive_expect_tx(&full_bar[s], G::CODE + G::ACT + p.zr * kDecRows);
#pragma unroll
        for (int c = 0; c < NC; ++c)
          tma_load_2d(st + c * G::CODE1, &p.q, &full_bar[s], (k0 + 128 * c) / 2, n0, polw);
        tma_load_2d(st + G::CODE + G::ACT, &p.z, &full_bar[s], n0, k0 / p.group, polw);
      };
      auto issue_a = [&](int i, int s) {
#pragma unroll
        for (int c = 0; c < NC; ++c)
          tma_load_2d(sbase + s * G::PER + G::CODE + c * G::ACT1, &p.a, &full_bar[s], kbeg + i * KST + 128 * c, 0, pola);
      };
      // weights and z are constants: requested before the wait for the activation quantizer
      const int npre = min(nst, NSTG);
      for (int i = 0; i < npre; ++i) issue_w(i, i);
      griddep_launch_dependents();
      griddep_wait();
      for (int i = 0; i < npre; ++i) issue_a(i, i);
      int s = npre % NSTG;
      uint32_t ph = npre == NSTG ? 1u : 0u;
      for (int i = npre; i < nst; ++i) {
        mbar_wait(&empty_bar[s], ph ^ 1);
        issue_w(i, s);
        issue_a(i, s);
        if (++s == NSTG) { s = 0; ph ^= 1; }
      }
    }
    return;
  }

  // --------------------------------------------------------------------------- consumers
  const int cw = warp - 1, gq = lane >> 2, t = lane & 3;
  uint32_t wofs[2][2], zofs[2][2];  // [row tile][g / h]: byte offsets in a stage (z: row 0)
#pragma unroll
  for (int rt = 0; rt < 2; ++rt)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int R = cw * 32 + rt * 16 + gq + 8 * h;
      wofs[rt][h] = R * 64 + ((t ^ ((R >> 1) & 3)) << 4);  // SWIZZLE_64B: cell t of row R
      zofs[rt][h] = G::CODE + G::ACT + R;
    }
  uint32_t aofs[MT][2];  // the thread's 32 B (cells 2t, 2t+1) of token mt*8+gq, SWIZZLE_128B
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int tok = mt * 8 + gq;
      aofs[mt][c] = G::CODE + tok * 128 + (((2 * t + c) ^ (tok & 7)) << 4);
    }
  int acc[2][MT][4];
#pragma unroll
  for (int rt = 0; rt < 2; ++rt)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[rt][mt][i] = 0;

  const uint32_t sb = smem_u32(sbase);
  int s = 0;
  uint32_t ph = 0;
  // staged z row of this thread's 32-k block in chunk c: (k0 + 128 c + 32 t) / g - k0 / g; for groups
  // >= 128 that needs k0 mod g, tracked per stage (kmod)
  const int g = p.group;
  int kmod = kbeg % g;
  for (int i = 0; i < nst; ++i) {
    mbar_wait(&full_bar[s], ph);
    const uint32_t st = sb + s * G::PER;
#pragma unroll
    for (int ch = 0; ch < NC; ++ch) {
    const int zrow = g <= 128 ? (128 * ch + 32 * t) / g : (kmod + 128 * ch + 32 * t) / g;
    uint4 w[2][2];
    uint32_t zz[2][2];
    uint4 b[MT][2];
#pragma unroll
    for (int rt = 0; rt < 2; ++rt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        w[rt][h] = lds128(st + ch * G::CODE1 + wofs[rt][h]);
        zz[rt][h] = lds_u8(st + zofs[rt][h] + zrow * kDecRows);
      }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int c = 0; c < 2; ++c) b[mt][c] = lds128(st + ch * G::ACT1 + aofs[mt][c]);
    if (ch == NC - 1) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[s]);  // operands in registers: hand the slot back
    }
#pragma unroll
    for (int rt = 0; rt < 2; ++rt) {
      uint32_t zm[2], bias[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        zm[h] = zz[rt][h];
        bias[h] = (128u - 8u * zm[h]) * 0x01010101u;  // u z + 128 - 8 z = q z + 128 per byte
      }
      const uint32_t wg[4] = {w[rt][0].x, w[rt][0].y, w[rt][0].z, w[rt][0].w};
      const uint32_t wh[4] = {w[rt][1].x, w[rt][1].y, w[rt][1].z, w[rt][1].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        // u = q + 8 per nibble: even k in the low nibbles, odd k in the high nibbles
        const uint32_t elo_g = lop3_and_xor(wg[j], 0x0F0F0F0Fu, 0x08080808u);
        const uint32_t ehi_g = lop3_and_xor(wg[j] >> 4, 0x0F0F0F0Fu, 0x08080808u);
        const uint32_t elo_h = lop3_and_xor(wh[j], 0x0F0F0F0Fu, 0x08080808u);
        const uint32_t ehi_h = lop3_and_xor(wh[j] >> 4, 0x0F0F0F0Fu, 0x08080808u);
        const uint32_t a[4] = {elo_g * zm[0] + bias[0], elo_h * zm[1] + bias[1], ehi_g * zm[0] + bias[0],
                               ehi_h * zm[1] + bias[1]};
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          // block 4t + j of token mt*8 + gq: even-k word 2j, odd-k word 2j + 1 of the thread's 32 B
          const uint4 v = b[mt][j >> 1];
          const uint32_t b0 = (j & 1) ? v.z : v.x, b1 = (j & 1) ? v.w : v.y;
          imma16832(acc[rt][mt], a, b0, b1);
        }
      }
    }
    }  // chunk
    if (g > 128) { kmod += KST; while (kmod >= g) kmod -= g; }
    if (++s == NSTG) { s = 0; ph ^= 1; }
  }

  // ------------------------------------------------------------- epilogue (+ split-K fixup)
  auto store = [&](int tok, int n, int32_t v) {
    const float f = (float)(v - 128 * __ldg(p.rowsum + tok)) * __ldg(p.sa + tok) * __ldg(p.sigma + n);
    const size_t o = (size_t)tok * p.N + n;
    if (p.cdt == FQ_FP32) reinterpret_cast<float*>(p.C)[o] = f;
    else if (p.cdt == FQ_BF16) reinterpret_cast<__nv_bfloat16*>(p.C)[o] = __float2bfloat16_rn(f);
    else reinterpret_cast<__half*>(p.C)[o] = __float2half_rn(f);
  };
  auto out_idx = [&](int rt, int mt, int i, int& n, int& tok) {
    n = n0 + cw * 32 + rt * 16 + gq + ((i >> 1) ? 8 : 0);
    tok = mt * 8 + 2 * t + (i & 1);
  };
  if (p.splits == 1) {
#pragma unroll
    for (int rt = 0; rt < 2; ++rt)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          int n, tok;
          out_idx(rt, mt, i, n, tok);
          if (n < p.N && tok < p.M) store(tok, n, acc[rt][mt][i]);
        }
    return;
  }
  int32_t* part = p.ws + (size_t)by * p.M * p.N;
#pragma unroll
  for (int rt = 0; rt < 2; ++rt)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int n, tok;
        out_idx(rt, mt, i, n, tok);
        if (n < p.N && tok < p.M) __stcg(part + (size_t)tok * p.N + n, acc[rt][mt][i]);
      }
  asm volatile("bar.sync 1, %0;" ::"n"(32 * kDecWarps));
  int* ctr = p.ctr + bx;
  if (threadIdx.x == 32) {
    __threadfence();
    const int last = atomicAdd(ctr, 1) == p.splits - 1;
    if (last) __threadfence();
    s_last = last;
  }
  asm volatile("bar.sync 1, %0;" ::"n"(32 * kDecWarps));
  if (!s_last) return;
  {
    const int n = n0 + (int)threadIdx.x - 32;  // consumer thread = column (coalesced)
    if (n < p.N && p.M <= 4) {  // few tokens: one token at a time (measured faster at M = 1)
      for (int tok = 0; tok < p.M; ++tok) {
        int32_t v = 0;
        for (int sp = 0; sp < p.splits; ++sp) v += __ldcg(p.ws + ((size_t)sp * p.M + tok) * p.N + n);
        store(tok, n, v);
      }
    } else if (n < p.N) {
      // all tokens of one split in flight per round (integer sums: exact in any order)
      int32_t v[MT * 8];
#pragma unroll
      for (int tok = 0; tok < MT * 8; ++tok) v[tok] = 0;
      for (int sp = 0; sp < p.splits; ++sp) {
#pragma unroll
        for (int tok = 0; tok < MT * 8; ++tok)
          if (tok < p.M) v[tok] += __ldcg(p.ws + ((size_t)sp * p.M + tok) * p.N + n);
      }
#pragma unroll
      for (int tok = 0; tok < MT * 8; ++tok)
        if (tok < p.M) store(tok, n, v[tok]);
    }
  }
  if (threadIdx.x == 32) *ctr = 0;  // self-reset for the next call / graph replay
}

}  // namespace i8

// ------------------------------------------------------------------------------------- host side
cudaError_t run_quantize_intscale(int wdt, const void* W, int K, int N, int group, void* codes, void* z,
                                  float* sigma, int32_t* status, cudaStream_t st) {
  const size_t smem = (size_t)(K / group) * 4;
  if (wdt == FQ_BF16)
    i8::quantize_intscale_kernel<__nv_bfloat16><<<N, 256, smem, st>>>(
        reinterpret_cast<const __nv_bfloat16*>(W), K, N, group, reinterpret_cast<uint8_t*>(codes),
        reinterpret_cast<uint8_t*>(z), sigma, status);
  else if (wdt == FQ_FP16)
    i8::quantize_intscale_kernel<__half><<<N, 256, smem, st>>>(reinterpret_cast<const __half*>(W), K, N, group,
                                                               reinterpret_cast<uint8_t*>(codes),
                                                               reinterpret_cast<uint8_t*>(z), sigma, status);
  else
    i8::quantize_intscale_kernel<float><<<N, 256, smem, st>>>(reinterpret_cast<const float*>(W), K, N, group,
                                                              reinterpret_cast<uint8_t*>(codes),
                                                              reinterpret_cast<uint8_t*>(z), sigma, status);
  return cudaGetLastError();
}

cudaError_t run_quantize_acts_i8(int adt, const void* A, int M, int K, void* Aq, float* sa, int32_t* rowsum,
                                 int32_t* status, cudaStream_t st) {
#ifndef FQ_I8_ACT_CLUSTER
#define FQ_I8_ACT_CLUSTER 1
#endif
  // few tokens: one 8-CTA cluster per token (the decode case is latency-bound)
  if (FQ_I8_ACT_CLUSTER && M <= 64 && K % (8 * i8::kActCluster) == 0) {
    const int grid = M * i8::kActCluster;
    if (adt == FQ_BF16)
      return launch_pdl(i8::quantize_acts_i8_cluster_kernel<__nv_bfloat16>, grid, 256, 0, st,
                        reinterpret_cast<const __nv_bfloat16*>(A), K, reinterpret_cast<int8_t*>(Aq), sa, rowsum, status);
    if (adt == FQ_FP16)
      return launch_pdl(i8::quantize_acts_i8_cluster_kernel<__half>, grid, 256, 0, st, reinterpret_cast<const __half*>(A),
                        K, reinterpret_cast<int8_t*>(Aq), sa, rowsum, status);
    return launch_pdl(i8::quantize_acts_i8_cluster_kernel<float>, grid, 256, 0, st, reinterpret_cast<const float*>(A), K,
                      reinterpret_cast<int8_t*>(Aq), sa, rowsum, status);
  }
  // one CTA per token; 1024 threads when few tokens (the decode case is latency-bound), else 256
  const int thr = M < 2 * 148 ? 1024 : 256;
  if (adt == FQ_BF16)
    return launch_pdl(i8::quantize_acts_i8_kernel<__nv_bfloat16>, M, thr, 0, st,
                      reinterpret_cast<const __nv_bfloat16*>(A), K, reinterpret_cast<int8_t*>(Aq), sa, rowsum, status);
  if (adt == FQ_FP16)
    return launch_pdl(i8::quantize_acts_i8_kernel<__half>, M, thr, 0, st, reinterpret_cast<const __half*>(A), K,
                      reinterpret_cast<int8_t*>(Aq), sa, rowsum, status);
  return launch_pdl(i8::quantize_acts_i8_kernel<float>, M, thr, 0, st, reinterpret_cast<const float*>(A), K,
                    reinterpret_cast<int8_t*>(Aq), sa, rowsum, status);
}

static int i8_bn(int M) { return std::min(256, (M + 15) / 16 * 16); }
static int i8_bnmax(int bn) { return bn <= 32 ? 32 : (bn <= 64 && FQ_I8_MID_CPS == 2) ? 64 : bn <= 128 ? 128 : 256; }
static int i8_cps(int bn) {
  return bn <= 32 ? FQ_I8_SMALL_CPS : bn <= 64 ? FQ_I8_MID_CPS : bn <= 128 ? FQ_I8_128_CPS : 1;
}
constexpr size_t kI8CounterBytes = 65536;

// Split-K plan: persistent CTAs walk the (tile, K range) items; pick the split count (items of
// >= 4 K blocks) that best fills the last round, with a small charge per extra split (partials).
static int i8_splits(int M, int K, int N, int* kbs_out) {
  const int bn = i8_bn(M);
  const int tiles = ((M + bn - 1) / bn) * ((N + i8::BM - 1) / i8::BM);
  const int kblocks = K / i8::BK;
  if (tiles >= num_sms() * i8_cps(bn))  // the tiles fill the GPU
    return (kbs_out ? (*kbs_out = kblocks) : 0), 1;
  const int smax = std::max(1, std::min(8, kblocks / 4));
  int best_s = 1;
  double best = 1e300;
  for (int s = 1; s <= smax; ++s) {
    const int kbs = (kblocks + s - 1) / s, se = (kblocks + kbs - 1) / kbs;
    const double rounds = (double)tiles * se / (num_sms() * i8_cps(bn));
    const double eff = rounds / std::ceil(rounds);
    const double cost = (1.0 + 0.03 * (se - 1)) / eff;
    if (cost < best * 0.999) { best = cost; best_s = se; }
  }
  if (tiles > (int)(kI8CounterBytes / sizeof(int))) best_s = 1;
  const int kbs = (kblocks + best_s - 1) / best_s;
  if (kbs_out) *kbs_out = kbs;
  return (kblocks + kbs - 1) / kbs;
}

#ifndef FQ_I8_IMMA
#define FQ_I8_IMMA 1  // decode sizes (M <= 16) on the mma.sync m16n8k32 u8 x s8 kernel
#endif
static bool i8_imma(int M) { return FQ_I8_IMMA && M <= 16; }
static GemvPlan i8_dec_plan(int M, int K, int N, int group) {
  return plan_gemv(M, K, N, 4, group, num_sms());  // same split plan as the bf16 decode kernel
}

size_t gemm_i8_workspace_bytes(int M, int K, int N) {
  if (i8_imma(M)) {
    const GemvPlan pl = i8_dec_plan(M, K, N, 128);
    return pl.splits > 1 ? kI8CounterBytes + (size_t)pl.splits * M * N * sizeof(int32_t) : 256;
  }
  const int s = i8_splits(M, K, N, nullptr);
  if (s == 1) return 256;
  const int bn = i8_bn(M);
  const size_t tiles = (size_t)((M + bn - 1) / bn) * ((N + i8::BM - 1) / i8::BM);
  return kI8CounterBytes + tiles * s * bn * i8::BM * sizeof(int32_t);
}

template <int BNMAX, int DG, int CPS>
static cudaError_t launch_i8(const i8::I8Prob& p, cudaStream_t st) {
  using Gm = i8::Geo<BNMAX, CPS>;
  cudaError_t e = ensure_smem_attr<i8::gemm_i8_kernel<BNMAX, DG, CPS>>(Gm::SMEM);
  if (e != cudaSuccess) return e;
  const int items = p.m_tiles * p.n_tiles * p.splits;
  return launch_pdl(i8::gemm_i8_kernel<BNMAX, DG, CPS>, std::min(items, CPS * num_sms()), i8::i8_threads(DG),
                    Gm::SMEM, st, p);
}

#ifndef FQ_I8_DEC_NC
#define FQ_I8_DEC_NC 2  // 128-k chunks per stage of the IMMA decode kernel
#endif
template <int MT>
static cudaError_t launch_dec_i8(const i8::DecI8Prob& d, int ctas, cudaStream_t st) {
  constexpr int NC = FQ_I8_DEC_NC;
  constexpr int smem = i8::DecI8Geo<MT, NC>::SMEM;
  cudaError_t e = ensure_smem_attr<i8::decode_i8_kernel<MT, NC>>(smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(i8::decode_i8_kernel<MT, NC>, ctas, i8::kDecThreads, smem, st, d);
}

static cudaError_t run_dec_i8(const void* Aq, const float* sa, const int32_t* rowsum, int M, int K, int N,
                              int group, const void* codes, const void* z, const float* sigma, void* C, int cdt,
                              void* ws, size_t ws_bytes, cudaStream_t st) {
  i8::DecI8Prob d{};
  const int mt = M <= 8 ? 1 : 2;
  // z rows staged per stage: every group a stage touches (groups >= the stage: the first two)
  d.zr = group < 128 * FQ_I8_DEC_NC ? 128 * FQ_I8_DEC_NC / group : (FQ_I8_DEC_NC > 1 ? 2 : 1);
  if (!make_tmap_2d(&d.a, Aq, 1, (uint64_t)K, (uint64_t)M, (uint64_t)K, 128, mt * 8, 128)) return cudaErrorInvalidValue;
  if (!make_tmap_2d(&d.q, codes, 1, (uint64_t)K / 2, (uint64_t)N, (uint64_t)K / 2, 64, i8::kDecRows, 64))
    return cudaErrorInvalidValue;
  if (!make_tmap_2d(&d.z, z, 1, (uint64_t)N, (uint64_t)(K / group), (uint64_t)N, i8::kDecRows, d.zr, 0))
    return cudaErrorInvalidValue;
  d.sa = sa;
  d.rowsum = rowsum;
  d.sigma = sigma;
  d.C = C;
  d.M = M; d.K = K; d.N = N; d.group = group; d.cdt = cdt;
  d.gx = (N + i8::kDecRows - 1) / i8::kDecRows;
  const GemvPlan pl = i8_dec_plan(M, K, N, group);
  d.splits = 1;
  d.klen = K;
  const size_t need = kI8CounterBytes + (size_t)pl.splits * M * N * sizeof(int32_t);
  if (pl.splits > 1 && ws && ws_bytes >= need && d.gx <= (int)(kI8CounterBytes / sizeof(int))) {
    d.splits = pl.splits;
    d.klen = pl.klen;
    d.ctr = reinterpret_cast<int*>(ws);
    d.ws = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(ws) + kI8CounterBytes);
  }
  const int ctas = d.gx * d.splits;
  return mt == 1 ? launch_dec_i8<1>(d, ctas, st) : launch_dec_i8<2>(d, ctas, st);
}

cudaError_t run_gemm_i8(const void* Aq, const float* sa, const int32_t* rowsum, int M, int K, int N, int group,
                        const void* codes,
                        const void* z, const float* sigma, void* C, int cdt, void* ws, size_t ws_bytes,
                        cudaStream_t st) {
  if (i8_imma(M)) return run_dec_i8(Aq, sa, rowsum, M, K, N, group, codes, z, sigma, C, cdt, ws, ws_bytes, st);
  i8::I8Prob p{};
  p.bn = i8_bn(M);
  if (!make_tmap_2d(&p.a, Aq, 1, (uint64_t)K, (uint64_t)M, (uint64_t)K, i8::BK, p.bn, 128)) return cudaErrorInvalidValue;
  if (!make_tmap_2d(&p.q, codes, 1, (uint64_t)K / 2, (uint64_t)N, (uint64_t)K / 2, i8::BK / 2, i8::BM, 64))
    return cudaErrorInvalidValue;
  if (!make_tmap_2d(&p.z, z, 1, (uint64_t)N, (uint64_t)(K / group), (uint64_t)N, i8::BM, i8::ZROWS, 0))
    return cudaErrorInvalidValue;
  p.sa = sa;
  p.rowsum = rowsum;
  p.sigma = sigma;
  p.C = C;
  p.M = M; p.K = K; p.N = N; p.group = group; p.cdt = cdt;
  p.m_tiles = (M + p.bn - 1) / p.bn;
  p.n_tiles = (N + i8::BM - 1) / i8::BM;
  p.gm = 8;
  int kbs = 0;
  const int s = i8_splits(M, K, N, &kbs);
  p.splits = 1;
  p.kbs = K / i8::BK;
  if (s > 1 && ws && ws_bytes >= gemm_i8_workspace_bytes(M, K, N)) {
    p.splits = s;
    p.kbs = kbs;
    p.ctr = reinterpret_cast<int*>(ws);
    p.ws = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(ws) + kI8CounterBytes);
  }
  switch (i8_bnmax(p.bn)) {
    case 32: return launch_i8<32, FQ_I8_SMALL_CPS == 2 ? 1 : FQ_I8_DG_SMALL, FQ_I8_SMALL_CPS>(p, st);
    case 64: return launch_i8<64, 1, 2>(p, st);
    case 128: return FQ_I8_128_CPS == 2 ? launch_i8<128, 1, 2>(p, st) : launch_i8<128, FQ_I8_DG_LARGE, 1>(p, st);
    default: return launch_i8<256, FQ_I8_DG_LARGE, 1>(p, st);
  }
}

}  // namespace fq
