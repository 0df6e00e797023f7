/*
 * fq.h — C ABI of the B200 (sm_100a) FineQuant hot path.
 *
 * FineQuant (arXiv 2308.09723): weight-only, symmetric, linear-absmax, group-wise quantization
 * of a weight matrix to int4 / int8 codes with per-group scales in the activation dtype, the
 * paper's adaptive group-size heuristic, and a fused "dequantize on the fly" GEMM of fp16/bf16
 * activations with those codes.  Citations "P:<line> §x" point into the paper text.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  Shapes.  The paper's weight matrix W has K rows (reduction dim) and N columns (outputs);
 *    "each contiguous block of B elements in a given column has its own scaling factor"
 *    (§4.1).  W is STORED like torch nn.Linear.weight: [N, K] row-major, so paper column n
 *    is the contiguous row n.  G = K / group.
 *  Canonical packed layout (bit-exact contract):
 *    codes  [N, K*bits/8] bytes, K contiguous per column n.
 *           int4: byte (n, k/2) = (q[n,k] & 0xF) | (q[n,k+1] & 0xF) << 4  (k even; two's complement)
 *           int8: byte (n, k)   = (uint8_t) q[n,k]
 *           int3 / int2 (the paper's low-bit variants, reading R19): the
 *           column's little-endian bit stream, code k in bits [b k, b k + b) (two's complement),
 *           byte i = stream bits [8i, 8i + 8) -- int4 and int8 are its b = 4 / 8 cases
 *    scales [G, N] row-major, dtype = scale_dtype (the activation dtype, §4.1).
 *  Memory.  Every tensor argument is a caller-owned DEVICE pointer unless documented as host.
 *    The library never allocates device memory; scratch is the caller's `ws`.
 *  Streams.  `stream` is a cudaStream_t passed as void*; all work is enqueued on it
 *    asynchronously.  NULL = legacy default stream.
 *  Errors.  Argument/shape validation is synchronous and happens before any launch, so a call
 *    that returns != FQ_OK has written nothing.  Launch failures return FQ_ERR_CUDA.  Data-
 *    dependent conditions the host cannot see (non-finite W, fp16 scale overflow) are reported
 *    through the optional device status word (bit 0: non-finite input in a group, bit 1: scale
 *    overflow); affected groups get scale 0 and codes 0.  No C++ exception crosses the ABI.
 *  Thread safety.  All functions are re-entrant and thread-safe.  Process-wide state, all of it
 *    caches of pure functions: the SM count per device (atomics), a per-device "dynamic shared
 *    memory attribute applied" bit per kernel (atomics), and a 256-entry cache of encoded TMA
 *    descriptors keyed by every encoding argument (mutex-protected).  Nothing is read from the
 *    process environment: routing is a pure function of the arguments (and fq_gemm_opts).
 */
#ifndef FQ_H_
#define FQ_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FQ_OK = 0,
  FQ_ERR_INVALID_ARG = 1, /* null pointer, alpha out of range, bad dtype enum */
  FQ_ERR_SHAPE = 2,       /* K/N/M/group inconsistent or misaligned */
  FQ_ERR_UNSUPPORTED = 3, /* bits not in {2,3,4,8}; dtype / path combination without a kernel */
  FQ_ERR_WORKSPACE = 4,   /* ws too small (see fq_gemm_workspace_bytes) */
  FQ_ERR_CUDA = 5         /* a CUDA launch / runtime call failed */
} fq_status;

typedef enum { FQ_BF16 = 0, FQ_FP16 = 1, FQ_FP32 = 2 } fq_dtype;

/* Description of one quantized weight matrix. */
typedef struct {
  int64_t K;           /* reduction dim (paper rows); K % 32 == 0 */
  int64_t N;           /* outputs (paper columns); N % 8 == 0 */
  int32_t bits;        /* 4 or 8 ("int8 or int4 weights"); 3 or 2 (no kernel in the
                          paper): K % 128 == 0, fq_gemm on the decode kernel only (M <= 32
                          for group % 128 == 0, else M <= 16; larger M and fq_gemm_grouped:
                          FQ_ERR_UNSUPPORTED) */
  int32_t group;       /* group size along K; group % 16 == 0 and K % group == 0; group == K is
                          per-column (§3.2.1, App. B) */
  int32_t scale_dtype; /* fq_dtype of the scales: FQ_BF16 or FQ_FP16 (activation dtype) */
  int32_t reserved;    /* must be 0 */
} fq_wdesc;

/* Library version string. */
const char* fq_version(void);
/* Human-readable name of a status code (static storage). */
const char* fq_status_str(fq_status s);

/* Byte sizes of the canonical buffers (0 on invalid arguments).
 * fq_codes_bytes = N*K*bits/8 ; fq_scales_bytes = (K/group)*N*sizeof(scale dtype). */
size_t fq_codes_bytes(int64_t K, int64_t N, int32_t bits);
size_t fq_scales_bytes(int64_t K, int64_t N, int32_t group, int32_t scale_dtype);

/* ---------------------------------------------------------------------------------------------
 * Adaptive fine-grained group size (§3.3).  "we start from the column-wise quantization
 * and compute the range ... We then halve the quantization group size and compute the range of
 * each group.  If for any group [the ratio test fires] we halve the quantization group size
 * again."  Reading (R6): level L >= 1 fires iff some group has
 *   1000 * max|child| < alpha_milli * max|parent|,
 * levels are accepted while they fire; the result is the group of the last accepted level.
 * Ladder (R9): g_0 = K, g_{L+1} = g_L/2 while g_L is even, g_L/2 >= min_group, g_L/2 % 16 == 0.
 * The decision is split in two so that tensor-parallel callers can OR the flags of all shards
 * (all-reduce MAX) between the device pass and the host decision.
 * ------------------------------------------------------------------------------------------- */

/* Number of ladder levels including level 0 (= K); flags arrays have fq_adapt_levels()-1 ints.
 * Returns 0 on invalid arguments. */
int32_t fq_adapt_levels(int64_t K, int32_t min_group);
/* Group size of ladder level `level` (0 = K); 0 on invalid arguments. */
int32_t fq_adapt_group_at(int64_t K, int32_t min_group, int32_t level);

/* Device pass (kernel A1): for W [N, K] (dtype wdt in {BF16, FP16, FP32}), OR-accumulates into
 * flags_dev[L-1] (L = 1 .. levels-1) whether level L fires.  flags_dev must be zeroed by the
 * caller before the first contributing call (several calls on row blocks / shards may
 * accumulate into the same flags).  alpha_milli in [1, 1000].  status_dev (nullable) gets bit 0
 * if W holds a non-finite value. */
fq_status fq_adapt_flags(const void* W, int32_t wdt, int64_t K, int64_t N, uint32_t alpha_milli,
                         int32_t min_group, int32_t* flags_dev, int32_t* status_dev, void* stream);

/* Host decision (A2): flags_host = the (levels-1) flags copied back from the device. */
int32_t fq_adapt_decide(int64_t K, int32_t min_group, const int32_t* flags_host);

/* ---------------------------------------------------------------------------------------------
 * Row-parallel (K-sharded) tensor parallelism, SURVEY §8(c) C-T / §8(e).  The paper serves OPT with
 * tensor parallelism, "an all reduce after each attention and FFN block" (§2.1); out-proj and
 * FC2 are row-parallel, so rank r of `world` holds W_r = W[:, r*K/world : (r+1)*K/world] ([N, K/world]
 * row-major).  One g per matrix (R11) is decided on the FULL-K ladder (P:149 starts from the whole
 * column), and the codes/scales of every shard must be the K-/G-slices of the unsharded result.
 * world must be a power of two <= 64 with K/world on the ladder of (K, min_group) (K/world % 16 == 0).
 * Protocol (every rank; "MAX" = an all-reduce MAX across the ranks of the matrix):
 *   1. zero flags_dev [fq_adapt_levels(K, min_group) - 1] and colmax_dev [world * N] (fp32);
 *   2. fq_adapt_flags_rowshard(W_r, ...): OR-s the flags of every level whose parent group lies in
 *      one shard (group <= K/(2 world)) and writes colmax_dev[r*N + n] = max|W_r[n, :]| (+inf if
 *      W_r[n, :] holds a non-finite value);
 *   3. MAX over ranks of flags_dev and colmax_dev (non-negative fp32 order like their int32 bits, so
 *      one int32 MAX all-reduce of both serves);
 *   4. fq_adapt_flags_cross(colmax_dev, ...): OR-s the flags of the coarse levels 1 .. log2(world)
 *      (groups spanning shards) -- identical on every rank, no further exchange;
 *   5. g = fq_adapt_decide(K, min_group, flags copied to the host);
 *   6. fq_quantize_rowshard(W_r, ..., g, colmax_dev): the shard's codes [N, (K/world)*bits/8] and
 *      scales [Gs, N], Gs = (K/world)/g when g <= K/world (plain fq_quantize of the shard), else
 *      Gs = 1: the one scale row of the group holding the shard, from the group's amax =
 *      max of colmax_dev over the shards of that group.  The shard's fq_wdesc for fq_gemm is then
 *      { K/world, N, bits, min(g, K/world), scale_dtype }.
 * For a fixed group > K/world (e.g. per-column) run steps 1-3 with flags_dev = NULL.
 * ------------------------------------------------------------------------------------------- */
fq_status fq_adapt_flags_rowshard(const void* W_shard, int32_t wdt, int64_t K, int64_t N, int32_t world,
                                  int32_t rank, uint32_t alpha_milli, int32_t min_group, int32_t* flags_dev,
                                  float* colmax_dev, int32_t* status_dev, void* stream);
fq_status fq_adapt_flags_cross(const float* colmax_dev, int64_t K, int64_t N, int32_t world,
                               uint32_t alpha_milli, int32_t min_group, int32_t* flags_dev, void* stream);
/* d describes the FULL matrix (K, N, bits, group = g, scale dtype); colmax_dev may be NULL when
 * d->group <= K/world. */
fq_status fq_quantize_rowshard(const void* W_shard, int32_t wdt, const fq_wdesc* d, int32_t world, int32_t rank,
                               const float* colmax_dev, void* codes, void* scales, int32_t* status_dev,
                               void* stream);

/* ---------------------------------------------------------------------------------------------
 * Quantize + pack (kernel A3), App. A with groups.  A CTA streams K-slices
 * of whole groups of one column (<= 24 KB each) through shared memory; a group longer than that is
 * held by one CTA in registers, so group <= 65536 for 16-bit W and <= 32768 for fp32 W (any K
 * otherwise), else FQ_ERR_SHAPE.  W and codes must be 16-byte aligned, else FQ_ERR_INVALID_ARG.
 *   s[j,n] = RNE_scale_dtype( 2 * max_{k in group j} |W[n,k]| / (2^bits - 1) )   (one rounding)
 *   q[n,k] = clamp( round_half_away( W[n,k] / s[k/group, n] ), -2^(bits-1), 2^(bits-1)-1 ),
 *            q = 0 where s == 0.
 * W: [N, K] device, dtype wdt.  codes/scales: device outputs in the canonical layout.
 * status_dev: nullable device int32, OR-ed with bit 0 (non-finite W) / bit 1 (scale overflow).
 * ------------------------------------------------------------------------------------------- */
fq_status fq_quantize(const void* W, int32_t wdt, const fq_wdesc* d, void* codes, void* scales,
                      int32_t* status_dev, void* stream);

/* ---------------------------------------------------------------------------------------------
 * Fused dequantize + GEMM (kernels A4/A5 for M <= 16, the tcgen05 kernel A6 for larger M;
 * fq_gemm_opts can force either), §4.1:
 *   C[m,n] = sum_k A[m,k] * q[n,k] * s[k/group, n]
 * A: [M, K] row-major, dtype adt in {BF16, FP16}; the scales must have dtype adt.
 * C: [M, N] row-major, dtype cdt in {adt, FP32} (FP32 is a diagnostic mode).
 * M == 0 is an empty batch: validated (A and C may be NULL), nothing launched, FQ_OK.
 * M < 0 or M > 2^20: FQ_ERR_SHAPE.
 * ws/ws_bytes: device scratch of at least fq_gemm_workspace_bytes(M, d) bytes.  Layout: a fixed
 *   64 KiB region of arrival counters at offset 0, then split-K fp32 partials.  The buffer must be
 *   ZERO-FILLED once before its first use; every call leaves the counters zeroed again, so one
 *   buffer (sized for the largest call) can be shared by calls of any shape and graph-captured
 *   without re-clearing.  Calls sharing one ws must be stream-ordered.
 * Accumulation is fp32; results are deterministic (fixed-order split-K reduction).  Both paths
 *   split K over CTAs when the output tiles alone cannot fill the GPU (A4: always planned; A6: when
 *   its 128-row x round_up(M,16)-token tiles are fewer than the SMs, then possibly as 256-row
 *   tiles); a NULL/short ws on the A6 path just disables its split.  The routing and the split plan
 *   are pure functions of (M, K, N, bits, group), so fq_gemm_workspace_bytes is exact for a call.
 * ------------------------------------------------------------------------------------------- */
size_t fq_gemm_workspace_bytes(int64_t M, const fq_wdesc* d);
fq_status fq_gemm(const void* A, int32_t adt, int64_t M, const fq_wdesc* d, const void* codes,
                  const void* scales, void* C, int32_t cdt, void* ws, size_t ws_bytes,
                  void* stream);

/* Routing / plan overrides (tests, measurements).  Zero-initialised = fq_gemm's own plan. */
typedef enum {
  FQ_PATH_AUTO = 0,
  FQ_PATH_DECODE = 1,  /* the decode kernel A4 (any M: token tiles of <= 16/32 re-stream W) */
  FQ_PATH_TC = 2       /* the tcgen05 kernel A6 */
} fq_path;
typedef struct {
  int32_t path;       /* fq_path */
  int32_t splits;     /* > 0: split-K factor (A4: K ranges of whole stage pairs; A6: item count) */
  int32_t tc_halves;  /* A6, tiles of <= 128 tokens: 1 or 2 halves of 128 weight rows per tile */
  int32_t tc_dqg;     /* A6, 16 dequant warps: 1, or 2 groups on alternate K blocks (int4 only) */
  int32_t reserved[4];/* must be 0 */
} fq_gemm_opts;
/* As fq_gemm / fq_gemm_workspace_bytes with explicit overrides (opts NULL = all zero).  Invalid
 * override values are FQ_ERR_INVALID_ARG. */
size_t fq_gemm_workspace_bytes_ex(int64_t M, const fq_wdesc* d, const fq_gemm_opts* opts);
fq_status fq_gemm_ex(const void* A, int32_t adt, int64_t M, const fq_wdesc* d, const void* codes,
                     const void* scales, void* C, int32_t cdt, void* ws, size_t ws_bytes, void* stream,
                     const fq_gemm_opts* opts);

/* ---------------------------------------------------------------------------------------------
 * MoE expert batch (kernel A7).  E experts share K, N, bits and scale dtype (d->group ignored);
 * each expert has its own group size (adaptive per expert, "different model weight
 * matrices"; MoE experts P:166-167).  Tokens are sorted by expert:
 *   rows offsets[e] .. offsets[e+1]-1 of A ([T, K]) use expert e; C is [T, N].
 * offsets_host: HOST array of E+1 int64 (non-decreasing, offsets[0] = 0, offsets[E] = T).
 * codes_host / scales_host: HOST arrays of E DEVICE pointers (canonical layout per expert);
 * groups_host: HOST array of E group sizes (each valid for K).  Experts with 1 <= M_e <= 16 (32
 * on the int4 nibble path) run in one launch per kernel class of the decode kernel (A4, batched);
 * larger experts run the tcgen05 kernel (A6); empty experts launch nothing (T == 0: A and C may be
 * NULL, FQ_OK).  ws: fq_gemm_grouped_workspace_bytes(...) bytes, zero-filled once (same
 * contract as fq_gemm's ws); FQ_ERR_WORKSPACE if too small while decode experts are present --
 * checked, like every other argument, before the first launch.
 * ------------------------------------------------------------------------------------------- */
size_t fq_gemm_grouped_workspace_bytes(int64_t T, int32_t E, const fq_wdesc* d);
fq_status fq_gemm_grouped(const void* A, int32_t adt, int64_t T, const int64_t* offsets_host,
                          int32_t E, const fq_wdesc* d, const int32_t* groups_host,
                          const void* const* codes_host, const void* const* scales_host, void* C,
                          int32_t cdt, void* ws, size_t ws_bytes, void* stream);

/* The same batch with the expert offsets on the DEVICE (SURVEY §8(b) expert_offsets_dev): MoE routing
 * is produced on the GPU, so no D2H copy or host synchronisation is needed per MoE layer.
 * offsets_dev: DEVICE int64 [E+1], non-decreasing, offsets[0] = 0, offsets[E] <= T (read by the
 * kernels; it may be written by the previous kernel on the stream).  T = rows of A and C (capacity).
 * max_tokens: a host-known bound on every expert's token count (e.g. the router's capacity); it picks
 * the kernel (decode kernel A4 when <= 16 / 32, else tcgen05 A6) and the launch geometry.  Experts
 * with more tokens than max_tokens, or offsets outside [0, T], are clamped (their extra rows are not
 * computed) and set bit 2 of status_dev (nullable).  ws: fq_gemm_grouped_workspace_bytes(T, E, d).
 * Empty experts cost one early-exiting CTA per tile of the bound. */
fq_status fq_gemm_grouped_dev(const void* A, int32_t adt, int64_t T, const int64_t* offsets_dev, int32_t E,
                              const fq_wdesc* d, const int32_t* groups_host, const void* const* codes_host,
                              const void* const* scales_host, void* C, int32_t cdt, int64_t max_tokens,
                              int32_t* status_dev, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------------------
 * int8 activations x int4 weights with INTEGER group scales -- the paper's future work: "the
 * proposed method does not leverage integer instructions even when they are available" (§5),
 * "using int8 activations and int4 weights with integer scales for fine-grained quantization"
 * (§5).  Readings R15-R18.  Shapes: K % 128 == 0, K <= 65536, N % 16 == 0,
 * K % group == 0 and group in {32, 64} or group % 128 == 0 (else FQ_ERR_SHAPE).
 *   weights (offline, fq_quantize_intscale), W [N, K] of dtype wdt:
 *     sigma[n] = RN_fp32(2 max_k |W[n,k]| / (15 * 16))                     colscale: fp32 [N]
 *     z[j,n]   = clamp(ceil((2 max_{k in j} |W[n,k]| / 15) / sigma[n]), 1, 16)   zscales: u8 [G, N]
 *     q[n,k]   = clamp(round_half_away(W[n,k] / (sigma[n] z[j,n])), -8, 7)  codes: canonical int4
 *     (z and q decided in float64, where sigma*z is exact); a non-finite column gets sigma 0,
 *     z 1, codes 0 and sets bit 0 of status_dev (nullable).
 *   activations (every call, fq_quantize_acts_i8), A [M, K] of dtype adt (K % 8 == 0):
 *     s_a[m] = RN_fp32(max_k |A[m,k]| / 127)                               a_scale: fp32 [M]
 *     a_q[m,k] = clamp(round_half_away(fp32(A[m,k] / s_a[m])), -127, 127)   a_q: int8 [M, K]
 *     rowsum[m] = sum_k a_q[m,k]                                           a_rowsum: int32 [M]
 *     a_q layout: row-major [M, K] with each aligned 8-element word k-interleaved, even k first:
 *     byte 8j + i holds k = 8j + 2i and byte 8j + 4 + i holds k = 8j + 2i + 1 (i < 4) -- the
 *     order in which the GEMM unpacks int4 codes, so its dequantization needs no byte shuffles.
 *     (IEEE fp32 division); a non-finite row gets s_a 0, codes 0 and sets status bit 0.  The GEMM
 *     feeds the weights to the tensor core as unsigned bytes q*z + 128 and removes 128*rowsum[m].
 *   GEMM (fq_gemm_i8; M <= 16: mma.sync m16n8k32 u8 x s8 decode kernel, else tcgen05 kind::i8):
 *     acc[m,n] = sum_k a_q[m,k] * q[n,k] * z[k/group, n]   (exact int32)
 *     C[m,n]   = fp32(acc) * s_a[m] * sigma[n], rounded to cdt (BF16, FP16 or FP32)   C: [M, N]
 *   ws: fq_gemm_i8_workspace_bytes(M, K, N) bytes, zero-filled once (64 KiB of self-resetting
 *   split-K counters + int32 partials; same contract as fq_gemm's ws); NULL / short disables the
 *   K split.  M == 0: nothing launched, FQ_OK.
 * ------------------------------------------------------------------------------------------- */
size_t fq_zscales_bytes(int64_t K, int64_t N, int32_t group);
fq_status fq_quantize_intscale(const void* W, int32_t wdt, int64_t K, int64_t N, int32_t group, void* codes,
                               void* zscales, float* colscale, int32_t* status_dev, void* stream);
fq_status fq_quantize_acts_i8(const void* A, int32_t adt, int64_t M, int64_t K, void* a_q, float* a_scale,
                              int32_t* a_rowsum, int32_t* status_dev, void* stream);
size_t fq_gemm_i8_workspace_bytes(int64_t M, int64_t K, int64_t N);
fq_status fq_gemm_i8(const void* a_q, const float* a_scale, const int32_t* a_rowsum, int64_t M, int64_t K,
                     int64_t N, int32_t group, const void* codes, const void* zscales, const float* colscale,
                     void* C, int32_t cdt, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------------------
 * Fused row-parallel GEMM + one-shot all-reduce.  Row-parallel layers (out-proj,
 * FC2) end in "an all reduce after each attention and FFN block" (§2.1).  Here the decode GEMM
 * (M <= 16, or <= 32 on the int4 nibble path) of each rank pushes its final fp32 partial of every
 * output tile straight into the tile owner's receive slot over NVLink peer memory (tile t is owned
 * by rank t % world); the last rank to arrive at the owner's counter sums the `world` slots in rank
 * order (deterministic, identical on every rank) and writes the tile to EVERY rank's output.  No
 * kernel waits on another GPU inside the GEMM; fq_xr_wait (one tiny kernel) makes the output ready
 * on this rank's stream.  Larger M (prefill): FQ_ERR_UNSUPPORTED (use an NCCL all-reduce).
 *   d_shard: this rank's K-shard [N, K/world] (codes/scales as fq_quantize_rowshard produces).
 *   peers_host: the table below (host copy, validated); peers_dev: a DEVICE copy of the same bytes
 *     (caller-owned, written once), read by the kernels.  Pointers are device addresses valid in
 *     this process (peer memory mapped via CUDA IPC / symmetric memory, or, for one-GPU tests, plain
 *     buffers of one device).  recv: fq_xr_recv_bytes(M, d_shard, world) bytes per rank; arrive:
 *     fq_xr_counter_bytes(M, d_shard) bytes per rank and done: one int32 per rank, all zero-filled
 *     once and self-resetting; out: [M, N] of dtype cdt (adt or FP32) on every rank.
 *   ws: fq_gemm_workspace_bytes_ex(M, d_shard, {.path = FQ_PATH_DECODE}) bytes (fq_gemm's contract).
 *   Calls of a group must be issued in the same order on every rank, each followed by fq_xr_wait on
 *   the same stream before the outputs are read or the buffers reused.  fq_xr_wait traps (a sticky
 *   CUDA error at the next synchronisation) if the group does not complete within 5 s.
 * ------------------------------------------------------------------------------------------- */
#define FQ_XR_MAX_WORLD 8
typedef struct {
  int32_t world;                       /* 1 .. FQ_XR_MAX_WORLD */
  int32_t rank;                        /* 0 .. world-1 */
  float* recv[FQ_XR_MAX_WORLD];        /* each rank's receive slots */
  int32_t* arrive[FQ_XR_MAX_WORLD];    /* each rank's per-tile arrival counters */
  int32_t* done[FQ_XR_MAX_WORLD];      /* each rank's completion counter */
  void* out[FQ_XR_MAX_WORLD];          /* each rank's output C [M, N] */
} fq_xr_peers;
size_t fq_xr_recv_bytes(int64_t M, const fq_wdesc* d_shard, int32_t world);
size_t fq_xr_counter_bytes(int64_t M, const fq_wdesc* d_shard);
fq_status fq_gemm_allreduce(const void* A, int32_t adt, int64_t M, const fq_wdesc* d_shard, const void* codes,
                            const void* scales, int32_t cdt, const fq_xr_peers* peers_host, const void* peers_dev,
                            void* ws, size_t ws_bytes, void* stream);
fq_status fq_xr_wait(const fq_xr_peers* peers_host, int64_t M, const fq_wdesc* d_shard, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FQ_H_ */
