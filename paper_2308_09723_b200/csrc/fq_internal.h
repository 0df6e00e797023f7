// fq_internal.h — launchers exported by the kernel translation units to the C-ABI layer.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <utility>

namespace fq {

// Routing / planning overrides of one GEMM call (fq_gemm_opts of include/fq.h; all 0 = planned).
// Routing and split plans are pure functions of (shape, Tune): nothing is read from the process
// environment on the product path.
struct Tune {
  int path = 0;    // 0 auto, 1 decode kernel (A4), 2 tcgen05 kernel (A6)
  int splits = 0;  // 0 planned, else the split-K factor
  int hm = 0;      // A6: 0 planned, 1 / 2 halves of 128 weight rows per tile
  int dqg = 0;     // A6: 0 planned, 1 / 2 dequant warp groups
};

cudaError_t run_quantize(int wdt, int sdt, int bits, const void* W, int K, int N, int group,
                         void* codes, void* scales, int32_t* status, cudaStream_t st,
                         const float* amax_tab = nullptr, int tab_r0 = 0, int tab_span = 0);
// A1 over W [N, K]: flags of ladder levels 1 .. nlev-1 OR-ed into flags[flag_ofs + L - 1]
// (flags may be NULL); colmax (nullable) receives max|W[n, :]| per row n (+inf if non-finite).
cudaError_t run_adapt_flags(int wdt, const void* W, int K, int N, int nlev, int gfin,
                            uint32_t alpha, int32_t* flags, int flag_ofs, float* colmax, int32_t* status,
                            cudaStream_t st);
// Coarse adaptive levels of a K-sharded matrix from the [world][N] table of shard column maxima.
cudaError_t run_adapt_cross(const float* colmax, int world, int N, int nlev_cross, uint32_t alpha,
                            int32_t* flags, cudaStream_t st);

// Fused row-parallel all-reduce (NEXT-1): the peer table every rank's decode GEMM reads (a device
// copy of fq_xr_peers, include/fq.h).
constexpr int kXRMaxWorld = 8;
struct XRPeers {
  int32_t world, rank;
  float* recv[kXRMaxWorld];     // each rank's receive slots [tiles][world][tile elems] fp32
  int32_t* arrive[kXRMaxWorld]; // each rank's per-tile arrival counters [tiles]
  int32_t* done[kXRMaxWorld];   // each rank's completion counter
  void* out[kXRMaxWorld];       // each rank's output C [M, N]
};

// Decode GEMM (mma.sync, kernels A4/A5).
struct GemvPlan {
  int rows_per_cta;   // 128 * RT
  int rt;             // row tiles (16 rows) per warp
  int splits;         // split-K factor S
  int kchunk;         // K elements per chunk (128 int4, 64 int8)
  int ktiles;         // token tiles of 16 (gridDim.z)
  int mt;             // 8-token MMA tiles per token tile (1 or 2)
  int klen;           // K elements per split (multiple of kchunk)
};
GemvPlan plan_gemv(int M, int K, int N, int bits, int group, int num_sms, int splits_override = 0);
// Largest M the decode kernel serves in one pass over the weights (32 on the int4 nibble path, else 16).
int gemv_max_m(int bits, int group);
size_t gemv_workspace_bytes(const GemvPlan& p, int M, int K, int N, int bits, int group);
size_t gemv_grouped_workspace_bytes(int64_t T, int K, int bits);
cudaError_t run_gemv(const GemvPlan& p, int adt, int cdt, int bits, const void* A, int M, int K,
                     int N, const void* codes, const void* scales, int group, void* C, void* ws,
                     cudaStream_t st, const XRPeers* xr_dev = nullptr);
// fused all-reduce: receive-slot elements per output tile, tile count, and the completion wait
int xr_tile_elems(const GemvPlan& p);
int xr_tiles(const GemvPlan& p, int N);
cudaError_t run_xr_wait(int32_t* done, int expected, cudaStream_t st);

// MoE batch of decode problems (experts with 1 <= M_e <= 16), one launch per kernel class.
cudaError_t run_gemv_grouped(int adt, int cdt, int bits, const void* A, int K, int N,
                             const int64_t* offsets, const int32_t* groups, const void* const* codes,
                             const void* const* scales, void* C, void* ws, int64_t T,
                             const int* experts, int nexp, cudaStream_t st);

// MoE batches with DEVICE expert offsets (fq_gemm_grouped_dev): launch geometry from the token
// bound Mmax, per-expert token ranges read on the device.
cudaError_t run_gemv_grouped_dev(int adt, int cdt, int bits, const void* A, int64_t T, int K, int N,
                                 const int64_t* offs_dev, const int32_t* groups, const void* const* codes,
                                 const void* const* scales, void* C, void* ws, int Mmax, const int* experts,
                                 int nexp, int32_t* status, cudaStream_t st);
cudaError_t run_gemm_tc_grouped_dev(int adt, int cdt, int bits, const void* A, int64_t T, int K, int N,
                                    const int64_t* offs_dev, const int32_t* groups, const void* const* codes,
                                    const void* const* scales, void* C, int Mmax, const int* experts, int nexp,
                                    const int* skips, int32_t* status, cudaStream_t st);

// Large-M tensor-core GEMM (tcgen05 + TMEM, kernel A6).
// Split-K when the output tiles cannot fill the SMs: workspace = 64 KiB counters (zero-filled once,
// self-resetting) + fp32 partials; without it (ws == NULL or too small) the kernel runs unsplit.
size_t gemm_tc_workspace_bytes(int M, int K, int N, int bits, const Tune& tune);
cudaError_t run_gemm_tc(int adt, int cdt, int bits, const void* A, int M, int K, int N, const void* codes,
                        const void* scales, int group, void* C, void* ws, size_t ws_bytes, cudaStream_t st,
                        const Tune& tune);
cudaError_t run_gemm_tc_grouped(int adt, int cdt, int bits, const void* A, int K, int N, const int64_t* offsets,
                                const int32_t* groups, const void* const* codes, const void* const* scales,
                                void* C, const int* experts, int nexp, cudaStream_t st);

// int8-activation x int4-weight path with integer group scales (fq_i8.cu).
cudaError_t run_quantize_intscale(int wdt, const void* W, int K, int N, int group, void* codes, void* z,
                                  float* sigma, int32_t* status, cudaStream_t st);
cudaError_t run_quantize_acts_i8(int adt, const void* A, int M, int K, void* Aq, float* sa, int32_t* rowsum,
                                 int32_t* status, cudaStream_t st);
size_t gemm_i8_workspace_bytes(int M, int K, int N);
cudaError_t run_gemm_i8(const void* Aq, const float* sa, const int32_t* rowsum, int M, int K, int N, int group,
                        const void* codes, const void* z, const float* sigma, void* C, int cdt, void* ws,
                        size_t ws_bytes, cudaStream_t st);

int num_sms();

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is a per-device-context setting: remember, per
// kernel instantiation and per device, that it was applied (thread-safe; idempotent on a race).
template <auto Kern>
inline cudaError_t ensure_smem_attr(int bytes) {
  static std::atomic<uint64_t> done{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(Kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

// Launch with the programmatic-stream-serialization attribute (PDL); the kernel must call
// griddep_wait() before touching memory written by earlier kernels in the stream.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// 2-D TMA descriptor (CUtensorMap, 128 bytes, written to `tmap`).  elem_bytes 1/2/4 -> u8/bf16/f32.
bool make_tmap_2d(void* tmap, const void* base, int elem_bytes, uint64_t inner, uint64_t outer,
                  uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, int swizzle_bytes);

}  // namespace fq
