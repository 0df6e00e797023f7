// fq_api.cu — the C ABI (include/fq.h): argument validation, sizing, dispatch to the kernels.
// No compute happens here; every step of the hot path runs in the sm_100a kernels.  Every
// argument (including workspace sizes) is validated before the first launch of a call.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <vector>

#include "../../include/fq.h"
#include "fq_internal.h"

namespace fq {

int num_sms() {
  static std::atomic<int> cached[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return 148;
  std::atomic<int>& c = cached[dev & 63];
  int v = c.load(std::memory_order_relaxed);
  if (v) return v;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
  c.store(v, std::memory_order_relaxed);
  return v;
}

static bool valid_dtype(int d) { return d == FQ_BF16 || d == FQ_FP16 || d == FQ_FP32; }
static bool valid_half(int d) { return d == FQ_BF16 || d == FQ_FP16; }
static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

static fq_status check_wdesc(const fq_wdesc* d) {
  if (!d) return FQ_ERR_INVALID_ARG;
  if (d->reserved != 0 || !valid_half(d->scale_dtype)) return FQ_ERR_INVALID_ARG;
  if (d->bits != 2 && d->bits != 3 && d->bits != 4 && d->bits != 8) return FQ_ERR_UNSUPPORTED;
  if (d->K <= 0 || d->N <= 0 || d->K % 32 || d->N % 8) return FQ_ERR_SHAPE;
  if (d->bits < 4 && d->K % 128) return FQ_ERR_SHAPE;  // int3 / int2 rows: whole 128-k stages
  if (d->K > (int64_t)1 << 20 || d->N > (int64_t)1 << 24) return FQ_ERR_SHAPE;
  if (d->group <= 0 || d->group % 16 || d->K % d->group) return FQ_ERR_SHAPE;
  return FQ_OK;
}

static fq_status to_tune(const fq_gemm_opts* o, Tune& t) {
  t = Tune{};
  if (!o) return FQ_OK;
  for (int i = 0; i < 4; ++i)
    if (o->reserved[i]) return FQ_ERR_INVALID_ARG;
  if (o->path < 0 || o->path > 2 || o->splits < 0 || o->splits > 4096 || o->tc_halves < 0 || o->tc_halves > 2 ||
      o->tc_dqg < 0 || o->tc_dqg > 2)
    return FQ_ERR_INVALID_ARG;
  t.path = o->path;
  t.splits = o->splits;
  t.hm = o->tc_halves;
  t.dqg = o->tc_dqg;
  return FQ_OK;
}

static cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static fq_status from_cuda(cudaError_t e) { return e == cudaSuccess ? FQ_OK : FQ_ERR_CUDA; }

// M <= 16 (32 on the int4 nibble path): memory-bound decode kernel (A4/A5), every weight streamed
// once; larger M: tcgen05 tensor-core kernel (A6).  Tune::path forces a path (tests, A/B).
// A single GEMM (N > 0) of 17..32 tokens on the int4 nibble path goes to A6 when A6's 128-row tiles
// do not fill the SMs (A6 then splits K, or uses two-half tiles): measured at M = 17 / 24 / 32
// (profiles/r01/a6_two_half_tiles.txt) OPT-13B attn-out 34-44 -> 24 us, QKV 42-46 -> 36, FFN2
// 56-69 -> 47-48, OPT-30B attn-out 40-50 -> 32, OPT-175B FC2 146 -> 131 (M = 32); matrices with
// >= 148 tiles (OPT-175B FC1, OPT-13B FFN1, OPT-30B QKV / FFN1) stay on the decode kernel.
static bool use_tc_path(int64_t M, int bits, int group, int64_t N, const Tune& t) {
  if (t.path == 1 || bits < 4) return false;  // int3 / int2: decode kernel only (callers reject larger M)
  if (t.path == 2) return true;
  const int dmax = gemv_max_m(bits, group);
  if (M > dmax) return true;
  // single GEMMs of 17..32 tokens: A6 (two CTAs per SM at <= 64-token tiles) beats the decode
  // kernel's four-token-tile class on every measured shape (profiles/r02/a6_two_ctas_per_sm.txt:
  // OPT-175B FC1 M=24 151 -> 133 us, OPT-13B FFN1 M=32 59 -> 43 us); MoE experts (N == 0 here)
  // of <= 32 tokens stay on the batched decode kernel
  return M > 16 && N > 0;
}

static int ilog2_exact(int64_t x) {  // log2 of a power of two, else -1
  if (x <= 0 || (x & (x - 1))) return -1;
  int l = 0;
  while ((1ll << l) < x) ++l;
  return l;
}

// Row-shard geometry check: world a power of two <= 64 whose K-slices sit on the (K, min_group)
// ladder.  Returns log2(world) or -1.
static int rowshard_levels(int64_t K, int32_t world, int32_t min_group) {
  const int lw = ilog2_exact(world);
  if (lw < 0 || world > 64) return -1;
  const int32_t nlev = fq_adapt_levels(K, min_group);
  if (nlev <= lw) return -1;  // K/world is not a ladder level
  return lw;
}

}  // namespace fq

using namespace fq;

extern "C" {

const char* fq_version(void) { return "fq 0.2.0 (sm_100a)"; }

const char* fq_status_str(fq_status s) {
  switch (s) {
    case FQ_OK: return "FQ_OK";
    case FQ_ERR_INVALID_ARG: return "FQ_ERR_INVALID_ARG";
    case FQ_ERR_SHAPE: return "FQ_ERR_SHAPE";
    case FQ_ERR_UNSUPPORTED: return "FQ_ERR_UNSUPPORTED";
    case FQ_ERR_WORKSPACE: return "FQ_ERR_WORKSPACE";
    case FQ_ERR_CUDA: return "FQ_ERR_CUDA";
  }
  return "FQ_ERR_UNKNOWN";
}

size_t fq_codes_bytes(int64_t K, int64_t N, int32_t bits) {
  if (K <= 0 || N <= 0 || (bits != 2 && bits != 3 && bits != 4 && bits != 8) || (K * bits) % 8) return 0;
  return (size_t)(N * (K * bits / 8));
}

size_t fq_scales_bytes(int64_t K, int64_t N, int32_t group, int32_t sdt) {
  if (K <= 0 || N <= 0 || group <= 0 || K % group || !valid_half(sdt)) return 0;
  return (size_t)((K / group) * N * 2);
}

int32_t fq_adapt_levels(int64_t K, int32_t min_group) {
  if (K <= 0 || min_group <= 0 || K % 16) return 0;
  int32_t n = 1;
  int64_t g = K;
  while (g % 2 == 0 && g / 2 >= min_group && (g / 2) % 16 == 0) {
    g /= 2;
    ++n;
  }
  return n;
}

int32_t fq_adapt_group_at(int64_t K, int32_t min_group, int32_t level) {
  const int32_t n = fq_adapt_levels(K, min_group);
  if (n == 0 || level < 0 || level >= n) return 0;
  return (int32_t)(K >> level);
}

int32_t fq_adapt_decide(int64_t K, int32_t min_group, const int32_t* flags_host) {
  const int32_t n = fq_adapt_levels(K, min_group);
  if (n == 0) return 0;
  int64_t g = K;
  for (int32_t L = 1; L < n; ++L) {
    if (!flags_host || !flags_host[L - 1]) break;
    g = K >> L;
  }
  return (int32_t)g;
}

fq_status fq_adapt_flags(const void* W, int32_t wdt, int64_t K, int64_t N, uint32_t alpha_milli,
                         int32_t min_group, int32_t* flags_dev, int32_t* status_dev,
                         void* stream) {
  if (!W || !flags_dev || !valid_dtype(wdt)) return FQ_ERR_INVALID_ARG;
  if (alpha_milli < 1 || alpha_milli > 1000 || min_group < 16) return FQ_ERR_INVALID_ARG;
  if (K <= 0 || N <= 0 || K % 32 || K > (1 << 20) || N > (1 << 24)) return FQ_ERR_SHAPE;
  const int32_t nlev = fq_adapt_levels(K, min_group);
  if (nlev <= 0 || nlev > 16) return FQ_ERR_SHAPE;
  const int gfin = (int)(K >> (nlev - 1));
  if (gfin % 8) return FQ_ERR_SHAPE;
  if (nlev == 1) return FQ_OK;  // nothing to test
  return from_cuda(run_adapt_flags(wdt, W, (int)K, (int)N, nlev, gfin, alpha_milli, flags_dev, 0, nullptr,
                                   status_dev, as_stream(stream)));
}

fq_status fq_adapt_flags_rowshard(const void* W_shard, int32_t wdt, int64_t K, int64_t N, int32_t world,
                                  int32_t rank, uint32_t alpha_milli, int32_t min_group, int32_t* flags_dev,
                                  float* colmax_dev, int32_t* status_dev, void* stream) {
  if (!W_shard || !colmax_dev || !valid_dtype(wdt)) return FQ_ERR_INVALID_ARG;
  if (alpha_milli < 1 || alpha_milli > 1000 || min_group < 16) return FQ_ERR_INVALID_ARG;
  if (K <= 0 || N <= 0 || K % 32 || K > (1 << 20) || N > (1 << 24)) return FQ_ERR_SHAPE;
  if (rank < 0 || rank >= world) return FQ_ERR_INVALID_ARG;
  const int lw = rowshard_levels(K, world, min_group);
  if (lw < 0) return FQ_ERR_SHAPE;
  const int64_t Ks = K / world;
  if (Ks % 32) return FQ_ERR_SHAPE;
  // the shard's own ladder (from K/world) is the tail of the full ladder, shifted by log2(world)
  const int32_t nlev_s = fq_adapt_levels(Ks, min_group);
  if (nlev_s <= 0 || nlev_s > 16 || fq_adapt_levels(K, min_group) != nlev_s + lw) return FQ_ERR_SHAPE;
  const int gfin = (int)(Ks >> (nlev_s - 1));
  if (gfin % 8) return FQ_ERR_SHAPE;
  return from_cuda(run_adapt_flags(wdt, W_shard, (int)Ks, (int)N, nlev_s, gfin, alpha_milli, flags_dev, lw,
                                   colmax_dev + (size_t)rank * N, status_dev, as_stream(stream)));
}

fq_status fq_adapt_flags_cross(const float* colmax_dev, int64_t K, int64_t N, int32_t world,
                               uint32_t alpha_milli, int32_t min_group, int32_t* flags_dev, void* stream) {
  if (!colmax_dev || !flags_dev) return FQ_ERR_INVALID_ARG;
  if (alpha_milli < 1 || alpha_milli > 1000 || min_group < 16) return FQ_ERR_INVALID_ARG;
  if (K <= 0 || N <= 0 || K % 32 || K > (1 << 20) || N > (1 << 24)) return FQ_ERR_SHAPE;
  const int lw = rowshard_levels(K, world, min_group);
  if (lw < 0) return FQ_ERR_SHAPE;
  if (lw == 0) return FQ_OK;  // one shard: no level spans shards
  return from_cuda(run_adapt_cross(colmax_dev, world, (int)N, lw, alpha_milli, flags_dev, as_stream(stream)));
}

fq_status fq_quantize(const void* W, int32_t wdt, const fq_wdesc* d, void* codes, void* scales,
                      int32_t* status_dev, void* stream) {
  fq_status s = check_wdesc(d);
  if (s != FQ_OK) return s;
  if (!W || !codes || !scales || !valid_dtype(wdt)) return FQ_ERR_INVALID_ARG;
  if (!aligned16(W) || !aligned16(codes)) return FQ_ERR_INVALID_ARG;  // 16-byte loads / bulk copies
  // one CTA holds a K-slice of whole groups in registers (slices of <= 12288 elements where the
  // group allows, else one group): group <= 65536 (16-bit W), 32768 (fp32 W)
  if (d->group > (wdt == FQ_FP32 ? 32768 : 65536)) return FQ_ERR_SHAPE;
  return from_cuda(run_quantize(wdt, d->scale_dtype, d->bits, W, (int)d->K, (int)d->N, d->group,
                                codes, scales, status_dev, as_stream(stream)));
}

fq_status fq_quantize_rowshard(const void* W_shard, int32_t wdt, const fq_wdesc* d, int32_t world, int32_t rank,
                               const float* colmax_dev, void* codes, void* scales, int32_t* status_dev,
                               void* stream) {
  fq_status s = check_wdesc(d);
  if (s != FQ_OK) return s;
  if (!W_shard || !codes || !scales || !valid_dtype(wdt)) return FQ_ERR_INVALID_ARG;
  if (!aligned16(W_shard) || !aligned16(codes)) return FQ_ERR_INVALID_ARG;
  if (rank < 0 || world <= 0 || rank >= world || world > 64 || ilog2_exact(world) < 0) return FQ_ERR_INVALID_ARG;
  if (d->K % world) return FQ_ERR_SHAPE;
  const int64_t Ks = d->K / world;
  if (Ks % 32) return FQ_ERR_SHAPE;
  const int64_t gs = std::min<int64_t>(d->group, Ks);
  if (d->group <= Ks) {
    if (Ks % d->group) return FQ_ERR_SHAPE;
  } else if (d->group % Ks) {
    return FQ_ERR_SHAPE;
  }
  if (gs > (wdt == FQ_FP32 ? 32768 : 65536)) return FQ_ERR_SHAPE;
  if (d->group <= Ks)  // whole groups inside the shard: the plain quantizer on the K-slice
    return from_cuda(run_quantize(wdt, d->scale_dtype, d->bits, W_shard, (int)Ks, (int)d->N, (int)gs, codes,
                                  scales, status_dev, as_stream(stream)));
  if (!colmax_dev) return FQ_ERR_INVALID_ARG;
  const int span = (int)(d->group / Ks);  // shards per group
  const int r0 = rank / span * span;
  return from_cuda(run_quantize(wdt, d->scale_dtype, d->bits, W_shard, (int)Ks, (int)d->N, (int)gs, codes, scales,
                                status_dev, as_stream(stream), colmax_dev, r0, span));
}

static size_t gemm_ws_bytes(int64_t M, const fq_wdesc* d, const Tune& t) {
  if (d->bits < 4 && (t.path == 2 || M > gemv_max_m(d->bits, d->group))) return 0;  // unsupported
  if (use_tc_path(M, d->bits, d->group, d->N, t))
    return gemm_tc_workspace_bytes((int)M, (int)d->K, (int)d->N, d->bits, t);
  const GemvPlan p = plan_gemv((int)M, (int)d->K, (int)d->N, d->bits, d->group, num_sms(), t.splits);
  return gemv_workspace_bytes(p, (int)M, (int)d->K, (int)d->N, d->bits, d->group);
}

size_t fq_gemm_workspace_bytes_ex(int64_t M, const fq_wdesc* d, const fq_gemm_opts* opts) {
  Tune t;
  if (check_wdesc(d) != FQ_OK || M <= 0 || to_tune(opts, t) != FQ_OK) return 0;
  return gemm_ws_bytes(M, d, t);
}

size_t fq_gemm_workspace_bytes(int64_t M, const fq_wdesc* d) { return fq_gemm_workspace_bytes_ex(M, d, nullptr); }

fq_status fq_gemm_ex(const void* A, int32_t adt, int64_t M, const fq_wdesc* d, const void* codes,
                     const void* scales, void* C, int32_t cdt, void* ws, size_t ws_bytes, void* stream,
                     const fq_gemm_opts* opts) {
  fq_status s = check_wdesc(d);
  if (s != FQ_OK) return s;
  Tune t;
  if ((s = to_tune(opts, t)) != FQ_OK) return s;
  if (!valid_half(adt)) return FQ_ERR_INVALID_ARG;
  if (d->scale_dtype != adt) return FQ_ERR_UNSUPPORTED;
  if (cdt != adt && cdt != FQ_FP32) return FQ_ERR_UNSUPPORTED;
  if (M < 0 || M > (1 << 20)) return FQ_ERR_SHAPE;
  if (!codes || !scales) return FQ_ERR_INVALID_ARG;
  if (M == 0) return FQ_OK;  // empty batch (A and C may be NULL): nothing to compute, nothing launched
  if (!A || !C) return FQ_ERR_INVALID_ARG;
  // int3 / int2 (NEXT-3): the decode kernel only (M <= 32 on groups % 128 == 0, else 16)
  if (d->bits < 4 && (t.path == 2 || M > gemv_max_m(d->bits, d->group))) return FQ_ERR_UNSUPPORTED;
  if (use_tc_path(M, d->bits, d->group, d->N, t))
    return from_cuda(run_gemm_tc(adt, cdt, d->bits, A, (int)M, (int)d->K, (int)d->N, codes, scales, d->group, C,
                                 ws, ws_bytes, as_stream(stream), t));
  const GemvPlan p = plan_gemv((int)M, (int)d->K, (int)d->N, d->bits, d->group, num_sms(), t.splits);
  const size_t need = gemv_workspace_bytes(p, (int)M, (int)d->K, (int)d->N, d->bits, d->group);
  if (need > 65536 && (!ws || ws_bytes < need)) return FQ_ERR_WORKSPACE;  // counters-only: may be NULL
  return from_cuda(run_gemv(p, adt, cdt, d->bits, A, (int)M, (int)d->K, (int)d->N, codes, scales,
                            d->group, C, ws, as_stream(stream)));
}

fq_status fq_gemm(const void* A, int32_t adt, int64_t M, const fq_wdesc* d, const void* codes,
                  const void* scales, void* C, int32_t cdt, void* ws, size_t ws_bytes,
                  void* stream) {
  return fq_gemm_ex(A, adt, M, d, codes, scales, C, cdt, ws, ws_bytes, stream, nullptr);
}

size_t fq_gemm_grouped_workspace_bytes(int64_t T, int32_t E, const fq_wdesc* d) {
  (void)E;
  if (check_wdesc(d) != FQ_OK || T < 0) return 0;
  // decode experts: counters + the pre-converted activations of all T tokens (shared region,
  // stream-ordered)
  return gemv_grouped_workspace_bytes(T, (int)d->K, d->bits);
}

fq_status fq_gemm_grouped(const void* A, int32_t adt, int64_t T, const int64_t* offsets_host,
                          int32_t E, const fq_wdesc* d, const int32_t* groups_host,
                          const void* const* codes_host, const void* const* scales_host, void* C,
                          int32_t cdt, void* ws, size_t ws_bytes, void* stream) {
  if (!d || !offsets_host || !groups_host || !codes_host || !scales_host || E <= 0)
    return FQ_ERR_INVALID_ARG;
  if (T > 0 && (!A || !C)) return FQ_ERR_INVALID_ARG;  // T == 0: A and C may be NULL
  if (!valid_half(adt) || d->scale_dtype != adt || (cdt != adt && cdt != FQ_FP32)) return FQ_ERR_UNSUPPORTED;
  if (d->bits < 4) return FQ_ERR_UNSUPPORTED;  // int3 / int2: single GEMMs on the decode kernel only
  if (offsets_host[0] != 0 || offsets_host[E] != T || T < 0) return FQ_ERR_SHAPE;
  for (int32_t e = 0; e < E; ++e) {
    fq_wdesc de = *d;
    de.group = groups_host[e];
    const fq_status s = check_wdesc(&de);
    if (s != FQ_OK) return s;
    if (offsets_host[e + 1] < offsets_host[e]) return FQ_ERR_SHAPE;
    if (!codes_host[e] || !scales_host[e]) return FQ_ERR_INVALID_ARG;
  }
  // classify every expert, then validate the workspace of every class, then launch
  const Tune t{};
  std::vector<int> small, large;
  for (int32_t e = 0; e < E; ++e) {
    const int64_t Me = offsets_host[e + 1] - offsets_host[e];
    if (Me == 0) continue;
    (!use_tc_path(Me, d->bits, groups_host[e], 0, t) ? small : large).push_back(e);
  }
  if (!small.empty() && (!ws || ws_bytes < gemv_grouped_workspace_bytes(T, (int)d->K, d->bits)))
    return FQ_ERR_WORKSPACE;
  const cudaStream_t st = as_stream(stream);
  if (!large.empty()) {  // every large expert in one persistent tcgen05 launch (per <= 48 experts)
    cudaError_t r = run_gemm_tc_grouped(adt, cdt, d->bits, A, (int)d->K, (int)d->N, offsets_host, groups_host,
                                        codes_host, scales_host, C, large.data(), (int)large.size(), st);
    if (r != cudaSuccess) return FQ_ERR_CUDA;
  }
  if (!small.empty())
    return from_cuda(run_gemv_grouped(adt, cdt, d->bits, A, (int)d->K, (int)d->N, offsets_host, groups_host,
                                      codes_host, scales_host, C, ws, T, small.data(), (int)small.size(), st));
  return FQ_OK;
}

// ------------------------------------------------------------------------------------------------
// int8 activations x int4 weights with integer group scales (fq_i8.cu)
static fq_status check_i8_shape(int64_t K, int64_t N, int32_t group) {
  if (K <= 0 || N <= 0 || K % 128 || K > 65536 || N % 16 || N > ((int64_t)1 << 24)) return FQ_ERR_SHAPE;
  if (group <= 0 || group % 32 || K % group) return FQ_ERR_SHAPE;
  if (group % 128 && 128 % group) return FQ_ERR_SHAPE;  // 32, 64 or a multiple of 128
  return FQ_OK;
}

size_t fq_zscales_bytes(int64_t K, int64_t N, int32_t group) {
  if (check_i8_shape(K, N, group) != FQ_OK) return 0;
  return (size_t)((K / group) * N);
}

fq_status fq_quantize_intscale(const void* W, int32_t wdt, int64_t K, int64_t N, int32_t group, void* codes,
                               void* zscales, float* colscale, int32_t* status_dev, void* stream) {
  if (!W || !codes || !zscales || !colscale || !valid_dtype(wdt)) return FQ_ERR_INVALID_ARG;
  const fq_status s = check_i8_shape(K, N, group);
  if (s != FQ_OK) return s;
  return from_cuda(run_quantize_intscale(wdt, W, (int)K, (int)N, group, codes, zscales, colscale, status_dev,
                                         as_stream(stream)));
}

fq_status fq_quantize_acts_i8(const void* A, int32_t adt, int64_t M, int64_t K, void* a_q, float* a_scale,
                              int32_t* a_rowsum, int32_t* status_dev, void* stream) {
  if (!valid_dtype(adt)) return FQ_ERR_INVALID_ARG;
  if (M < 0 || M > (1 << 20) || K <= 0 || K % 8 || K > (1 << 20)) return FQ_ERR_SHAPE;
  if (M == 0) return FQ_OK;
  if (!A || !a_q || !a_scale || !a_rowsum) return FQ_ERR_INVALID_ARG;
  return from_cuda(
      run_quantize_acts_i8(adt, A, (int)M, (int)K, a_q, a_scale, a_rowsum, status_dev, as_stream(stream)));
}

size_t fq_gemm_i8_workspace_bytes(int64_t M, int64_t K, int64_t N) {
  if (M <= 0 || M > (1 << 20) || check_i8_shape(K, N, 32) != FQ_OK) return 0;
  return gemm_i8_workspace_bytes((int)M, (int)K, (int)N);
}

fq_status fq_gemm_i8(const void* a_q, const float* a_scale, const int32_t* a_rowsum, int64_t M, int64_t K,
                     int64_t N, int32_t group, const void* codes, const void* zscales, const float* colscale,
                     void* C, int32_t cdt, void* ws, size_t ws_bytes, void* stream) {
  const fq_status s = check_i8_shape(K, N, group);
  if (s != FQ_OK) return s;
  if (!valid_dtype(cdt)) return FQ_ERR_INVALID_ARG;
  if (M < 0 || M > (1 << 20)) return FQ_ERR_SHAPE;
  if (!codes || !zscales || !colscale) return FQ_ERR_INVALID_ARG;
  if (M == 0) return FQ_OK;
  if (!a_q || !a_scale || !a_rowsum || !C) return FQ_ERR_INVALID_ARG;
  return from_cuda(run_gemm_i8(a_q, a_scale, a_rowsum, (int)M, (int)K, (int)N, group, codes, zscales, colscale, C, cdt, ws,
                               ws_bytes, as_stream(stream)));
}

// ------------------------------------------------------------------------------------------------
// Fused row-parallel GEMM + one-shot all-reduce (decode kernel epilogue)
static_assert(sizeof(fq_xr_peers) == sizeof(XRPeers) && FQ_XR_MAX_WORLD == kXRMaxWorld, "peer table layout");

static fq_status xr_plan(int64_t M, const fq_wdesc* d, GemvPlan& pl) {
  const fq_status s = check_wdesc(d);
  if (s != FQ_OK) return s;
  if (M <= 0 || M > gemv_max_m(d->bits, d->group)) return FQ_ERR_UNSUPPORTED;  // decode kernel only
  pl = plan_gemv((int)M, (int)d->K, (int)d->N, d->bits, d->group, num_sms(), 0);
  return FQ_OK;
}

static fq_status check_peers(const fq_xr_peers* x) {
  if (!x || x->world < 1 || x->world > FQ_XR_MAX_WORLD || x->rank < 0 || x->rank >= x->world)
    return FQ_ERR_INVALID_ARG;
  for (int r = 0; r < x->world; ++r)
    if (!x->recv[r] || !x->arrive[r] || !x->done[r] || !x->out[r]) return FQ_ERR_INVALID_ARG;
  return FQ_OK;
}

size_t fq_xr_recv_bytes(int64_t M, const fq_wdesc* d, int32_t world) {
  GemvPlan pl;
  if (world < 1 || world > FQ_XR_MAX_WORLD || xr_plan(M, d, pl) != FQ_OK) return 0;
  return (size_t)xr_tiles(pl, (int)d->N) * world * xr_tile_elems(pl) * sizeof(float);
}

size_t fq_xr_counter_bytes(int64_t M, const fq_wdesc* d) {
  GemvPlan pl;
  if (xr_plan(M, d, pl) != FQ_OK) return 0;
  return (size_t)xr_tiles(pl, (int)d->N) * sizeof(int32_t);
}

fq_status fq_gemm_allreduce(const void* A, int32_t adt, int64_t M, const fq_wdesc* d, const void* codes,
                            const void* scales, int32_t cdt, const fq_xr_peers* peers_host, const void* peers_dev,
                            void* ws, size_t ws_bytes, void* stream) {
  GemvPlan pl;
  fq_status s = xr_plan(M, d, pl);
  if (s != FQ_OK) return s;
  if ((s = check_peers(peers_host)) != FQ_OK) return s;
  if (!valid_half(adt) || d->scale_dtype != adt || (cdt != adt && cdt != FQ_FP32)) return FQ_ERR_UNSUPPORTED;
  if (!A || !codes || !scales || !peers_dev) return FQ_ERR_INVALID_ARG;
  const size_t need = gemv_workspace_bytes(pl, (int)M, (int)d->K, (int)d->N, d->bits, d->group);
  if (need > 65536 && (!ws || ws_bytes < need)) return FQ_ERR_WORKSPACE;
  return from_cuda(run_gemv(pl, adt, cdt, d->bits, A, (int)M, (int)d->K, (int)d->N, codes, scales, d->group,
                            peers_host->out[peers_host->rank], ws, as_stream(stream),
                            reinterpret_cast<const XRPeers*>(peers_dev)));
}

fq_status fq_xr_wait(const fq_xr_peers* peers_host, int64_t M, const fq_wdesc* d, void* stream) {
  GemvPlan pl;
  fq_status s = xr_plan(M, d, pl);
  if (s != FQ_OK) return s;
  if ((s = check_peers(peers_host)) != FQ_OK) return s;
  return from_cuda(run_xr_wait(peers_host->done[peers_host->rank], xr_tiles(pl, (int)d->N), as_stream(stream)));
}

// ------------------------------------------------------------------------------------------------
// MoE batch with DEVICE expert offsets (SURVEY §8(b) expert_offsets_dev): the router's output stays on
// the device; the host supplies only the static per-expert weights and a token bound.
fq_status fq_gemm_grouped_dev(const void* A, int32_t adt, int64_t T, const int64_t* offsets_dev, int32_t E,
                              const fq_wdesc* d, const int32_t* groups_host, const void* const* codes_host,
                              const void* const* scales_host, void* C, int32_t cdt, int64_t max_tokens,
                              int32_t* status_dev, void* ws, size_t ws_bytes, void* stream) {
  if (!d || !offsets_dev || !groups_host || !codes_host || !scales_host || E <= 0) return FQ_ERR_INVALID_ARG;
  if (!valid_half(adt) || d->scale_dtype != adt || (cdt != adt && cdt != FQ_FP32)) return FQ_ERR_UNSUPPORTED;
  if (d->bits < 4) return FQ_ERR_UNSUPPORTED;
  if (T < 0 || T > (1 << 20) || max_tokens < 0 || max_tokens > (1 << 20)) return FQ_ERR_SHAPE;
  for (int32_t e = 0; e < E; ++e) {
    fq_wdesc de = *d;
    de.group = groups_host[e];
    const fq_status s = check_wdesc(&de);
    if (s != FQ_OK) return s;
    if (!codes_host[e] || !scales_host[e]) return FQ_ERR_INVALID_ARG;
  }
  if (T == 0 || max_tokens == 0) return FQ_OK;  // nothing can be routed: nothing launched
  if (!A || !C) return FQ_ERR_INVALID_ARG;
  // Every expert's first tokens (up to the decode kernel's maximum) run on the batched decode kernel,
  // which streams each expert's weights once; when the bound exceeds that, the tcgen05 kernel takes
  // the remaining tokens of every expert (its tiles beyond an expert's count leave at once), so a
  // skewed routing does not push the many small experts onto tcgen05 tiles sized for the largest.
  std::vector<int> all, large, skips;
  for (int32_t e = 0; e < E; ++e) {
    all.push_back(e);
    const int dmax = gemv_max_m(d->bits, groups_host[e]);
    if (max_tokens > dmax) {
      large.push_back(e);
      skips.push_back(dmax);
    }
  }
  if (!ws || ws_bytes < gemv_grouped_workspace_bytes(T, (int)d->K, d->bits)) return FQ_ERR_WORKSPACE;
  const cudaStream_t st = as_stream(stream);
  cudaError_t r = run_gemv_grouped_dev(adt, cdt, d->bits, A, T, (int)d->K, (int)d->N, offsets_dev, groups_host,
                                       codes_host, scales_host, C, ws, (int)max_tokens, all.data(), (int)all.size(),
                                       status_dev, st);
  if (r != cudaSuccess) return FQ_ERR_CUDA;
  if (!large.empty())
    return from_cuda(run_gemm_tc_grouped_dev(adt, cdt, d->bits, A, T, (int)d->K, (int)d->N, offsets_dev,
                                             groups_host, codes_host, scales_host, C, (int)max_tokens, large.data(),
                                             (int)large.size(), skips.data(), status_dev, st));
  return FQ_OK;
}

}  // extern "C"
