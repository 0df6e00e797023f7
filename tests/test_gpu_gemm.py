"""GPU parity of the fused dequant-GEMM (kernels A4/A5, and the large-M path) against the fp64
oracle.  Tolerance (BASELINE.json north_star): max |C - C_ref| / sum|a*w| <= 2e-3."""
import os

import numpy as np
import pytest
import torch

from oracle import fq_oracle as O
from synth import activations_bits, gaussian_bits, gaussian_with_outliers_bits, wide_range_activations_bits
from helpers import bits_to_torch, torch_to_f64

pytestmark = pytest.mark.gpu
TOL = 2e-3


@pytest.fixture(scope="module")
def fq():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2308_09723_b200 import fq as m
    return m


@pytest.fixture
def env():
    """Routing / plan overrides for the next run_case calls (fq_gemm_opts, include/fq.h)."""
    o = {}

    def set_(k, v):
        o[k] = v
    set_.opts = o
    yield set_


def _opts(fq, env):
    o = getattr(env, "opts", None) if env is not None else None
    if not o:
        return None
    return fq.make_opts(o.get("path", 0), int(o.get("splits", 0)), int(o.get("hm", 0)), int(o.get("dqg", 0)))


def make_case(M, K, N, bits, group, adt="bf16", seed=0, outliers=0):
    if outliers:
        Wb = gaussian_with_outliers_bits((N, K), 0.02, 1000 + seed, outliers, 0.5, "bf16")
    else:
        Wb = gaussian_bits((N, K), 0.02, 1000 + seed, "bf16")
    Ab = activations_bits(M, K, 2000 + seed, adt)
    return Wb, Ab


def run_case(fq, Wb, Ab, bits, group, adt="bf16", cdt=None, env=None):
    W = bits_to_torch(Wb, "bf16")
    A = bits_to_torch(Ab, adt)
    sdt = {"bf16": torch.bfloat16, "fp16": torch.float16}[adt]
    qw = fq.quantize(W, bits, group, scale_dtype=sdt)
    C = fq.gemm(A, qw, out_dtype={"fp32": torch.float32, None: None}[cdt], opts=_opts(fq, env))
    torch.cuda.synchronize()
    return qw, C


def oracle_ref(Wb, Ab, bits, group, adt, cols=None):
    sf = O.FORMATS[adt]
    r = O.quantize(O.decode_bits(Wb, "bf16"), bits, group, sf)
    return O.gemm(O.decode_bits(Ab, adt), r.q, r.s, group, cols)


@pytest.mark.parametrize("M", [1, 2, 3, 8, 9, 16])
@pytest.mark.parametrize("bits", [4, 8])
def test_tiny_config_parity(fq, M, bits):
    # configs[0]: K=256, N=256, group 64 (+ M sweep of the decode regime)
    Wb, Ab = make_case(M, 256, 256, bits, 64, seed=M)
    _, C = run_case(fq, Wb, Ab, bits, 64)
    Cr, D = oracle_ref(Wb, Ab, bits, 64, "bf16")
    assert O.rel_err(torch_to_f64(C), Cr, D) <= TOL


@pytest.mark.parametrize("group", [16, 32, 48, 64, 96, 128, 256, 1536])
@pytest.mark.parametrize("bits", [4, 8])
def test_group_sizes_multi_tile_ragged(fq, bits, group):
    # several CTA tiles, ragged N tail (N not a multiple of the 256-row CTA tile)
    M, K, N = 5, 1536, 776
    Wb, Ab = make_case(M, K, N, bits, group, seed=group, outliers=2)
    _, C = run_case(fq, Wb, Ab, bits, group)
    Cr, D = oracle_ref(Wb, Ab, bits, group, "bf16")
    assert O.rel_err(torch_to_f64(C), Cr, D) <= TOL


@pytest.mark.parametrize("M,K,N,bits,group", [
    (1, 1088, 264, 4, 64),     # K = 4.25 decode stages (group-split path), ragged N
    (9, 1088, 264, 8, 64),     # int8, two token tiles
    (3, 800, 520, 4, 32),      # per-element-scale path, K tail of 32
    (16, 800, 296, 8, 16),
    (5, 352, 256, 8, 32),      # int8 per-element path (128-k stages), K tail of 96
    (1, 96, 256, 4, 96),       # K shorter than one stage, one group per column
    (24, 1152, 392, 4, 128),   # four token tiles (nibble path), K = 4.5 stages
    (1, 1152, 264, 4, 128),    # double stages (two 128-k chunks): K = 4.5 stages, chunk 1 of the last is past K
    (12, 1152, 520, 4, 128),   # double stages, two MMA token tiles, ragged N
    (40, 1088, 264, 4, 64),    # tcgen05 path, K = 17 blocks of 64
    (200, 800, 136, 8, 32),    # tcgen05 path, K = 12.5 blocks
])
def test_ragged_k_tails(fq, M, K, N, bits, group):
    """K not a multiple of the decode stage (256 / 128 k) or of the A6 K block (64): the partial
    last stage / block must contribute exactly its own k range."""
    Wb, Ab = make_case(M, K, N, bits, group, seed=K + M, outliers=1)
    _, C = run_case(fq, Wb, Ab, bits, group)
    Cr, D = oracle_ref(Wb, Ab, bits, group, "bf16")
    assert O.rel_err(torch_to_f64(C), Cr, D) <= TOL


def test_empty_batches(fq):
    """M == 0 through fq.gemm and T == 0 / all-empty experts through fq.gemm_grouped: empty
    outputs, FQ_OK, nothing launched (the C-ABI accepts the NULL pointers of zero-size tensors)."""
    W = bits_to_torch(gaussian_bits((256, 512), 0.02, 9, "bf16"), "bf16")
    qw = fq.quantize(W, 4, 128)
    A = torch.empty((0, 512), dtype=torch.bfloat16, device="cuda")
    C = fq.gemm(A, qw)
    assert C.shape == (0, 256)
    Cg = fq.gemm_grouped(A, [0, 0, 0], [qw, qw])
    assert Cg.shape == (0, 256)
    torch.cuda.synchronize()


@pytest.mark.parametrize("adt", ["bf16", "fp16"])
@pytest.mark.parametrize("bits", [4, 8])
@pytest.mark.parametrize("cdt", [None, "fp32"])
def test_dtypes(fq, adt, bits, cdt):
    M, K, N = 7, 1024, 512
    Wb, Ab = make_case(M, K, N, bits, 128, adt, seed=3)
    _, C = run_case(fq, Wb, Ab, bits, 128, adt, cdt)
    Cr, D = oracle_ref(Wb, Ab, bits, 128, adt)
    assert O.rel_err(torch_to_f64(C), Cr, D) <= TOL


@pytest.mark.parametrize("adt", ["bf16", "fp16"])
@pytest.mark.parametrize("M", [1, 5, 16])
def test_decode_activation_dynamic_range(fq, M, adt):
    """Activations spanning ~2^-90..2^90 (bf16; fp16: its own range) with zero chunks and a zero
    token: the decode kernel's internal fp16 re-encoding of bf16 activations (per-token, per-chunk
    power-of-two scale) must stay within the tolerance of the exact result."""
    lo, hi, shift = (-60.0, 60.0, 30) if adt == "bf16" else (-8.0, 6.0, 4)
    K, N = 1024, 512
    Wb = gaussian_bits((N, K), 0.02, 1234, "bf16")
    Ab = wide_range_activations_bits(M, K, 4321 + M, adt, lo, hi, shift)
    _, C = run_case(fq, Wb, Ab, 4, 128, adt, "fp32")
    Cr, D = oracle_ref(Wb, Ab, 4, 128, adt)
    assert O.rel_err(torch_to_f64(C), Cr, D) <= TOL  # D == 0 (zero token) requires C == 0 exactly


@pytest.mark.parametrize("splits", [1, 2, 3, 7])
@pytest.mark.parametrize("M", [1, 12])
def test_split_k_paths(fq, env, splits, M):
    env("splits", splits)
    Wb, Ab = make_case(M, 4096, 512, 4, 128, seed=11)
    for _ in range(2):  # second call checks the self-resetting counters
        _, C = run_case(fq, Wb, Ab, 4, 128, env=env)
        Cr, D = oracle_ref(Wb, Ab, 4, 128, "bf16")
        assert O.rel_err(torch_to_f64(C), Cr, D) <= TOL


@pytest.mark.parametrize("M,K,N", [(1, 4096, 512), (16, 4096, 768), (17, 2048, 512), (33, 1536, 1280),
                                   (5, 12288, 2048)])
def test_decode_multi_tile_determinism(fq, env, M, K, N):
    """Decode kernel with split-K fixups over several column and token tiles (M > 16 on the decode
    path): the fixup sums partials in a fixed order, so repeated calls are bit-identical (and the
    self-resetting counters are exercised)."""
    env("path", "decode")
    Wb, Ab = make_case(M, K, N, 4, 128, seed=M + K + N)
    _, C0 = run_case(fq, Wb, Ab, 4, 128, "bf16", "fp32", env=env)
    _, C1 = run_case(fq, Wb, Ab, 4, 128, "bf16", "fp32", env=env)
    assert torch.equal(C0, C1)
    Cr, D = oracle_ref(Wb, Ab, 4, 128, "bf16")
    assert O.rel_err(torch_to_f64(C0), Cr, D) <= TOL


@pytest.mark.parametrize("bits,group", [(4, 16), (4, 32), (4, 64), (8, 16), (8, 32)])
@pytest.mark.parametrize("M", [1, 5, 12])
def test_decode_small_groups_long_k(fq, env, bits, group, M):
    """Groups smaller than the decode stage (scale rows staged by TMA per stage) with one CTA per
    column tile streaming many more stages than its ring holds (FQ_GEMV_SPLITS=1): the scales must
    be consumed before the stage is handed back to the producer."""
    env("path", "decode")
    env("splits", 1)
    Wb, Ab = make_case(M, 4096, 512, bits, group, seed=group + M, outliers=2)
    _, C = run_case(fq, Wb, Ab, bits, group, "bf16", "fp32", env=env)
    Cr, D = oracle_ref(Wb, Ab, bits, group, "bf16")
    assert O.rel_err(torch_to_f64(C), Cr, D) <= TOL


@pytest.mark.parametrize("M,K,N,bits,group", [(32, 4096, 512, 4, 128), (100, 2048, 1280, 4, 64),
                                               (300, 2048, 640, 8, 128), (17, 8192, 256, 4, 16)])
def test_tc_split_k(fq, env, M, K, N, bits, group):
    """A6 with few output tiles splits K over CTAs (fixed-order fp32 fixup): parity with the oracle,
    bit-identical repeated calls, and the same result as the unsplit kernel within rounding."""
    env("path", "tc")
    Wb, Ab = make_case(M, K, N, bits, group, seed=M + N)
    _, C0 = run_case(fq, Wb, Ab, bits, group, "bf16", "fp32", env=env)
    _, C1 = run_case(fq, Wb, Ab, bits, group, "bf16", "fp32", env=env)
    assert torch.equal(C0, C1)
    Cr, D = oracle_ref(Wb, Ab, bits, group, "bf16")
    assert O.rel_err(torch_to_f64(C0), Cr, D) <= TOL
    env("splits", 1)
    _, C2 = run_case(fq, Wb, Ab, bits, group, "bf16", "fp32", env=env)
    assert O.rel_err(torch_to_f64(C2), Cr, D) <= TOL


@pytest.mark.parametrize("dqg", [1, 2])
@pytest.mark.parametrize("hm", [1, 2])
@pytest.mark.parametrize("M,K,N,bits,group,adt", [(32, 4096, 512, 4, 128, "bf16"), (48, 2048, 392, 8, 64, "fp16"),
                                                  (100, 3072, 640, 4, 32, "bf16"), (17, 8192, 136, 4, 16, "bf16"),
                                                  (24, 1536, 264, 4, 48, "fp16"), (64, 2048, 520, 4, 64, "bf16")])
def test_tc_tile_halves_split_k(fq, env, dqg, hm, M, K, N, bits, group, adt):
    """A6 with one- and two-half tiles (128 / 256 weight rows, FQ_TC_HM forces the choice) and one or
    two alternating dequant warp groups (FQ_TC_DQG; int4 only, each thread then covers 64 k and up to
    four group boundaries), under split-K: parity, bit-identical repeated calls, and N tails inside /
    past the second half."""
    env("path", "tc")
    env("hm", hm)
    env("dqg", dqg)
    Wb, Ab = make_case(M, K, N, bits, group, adt, seed=M + K + hm)
    _, C0 = run_case(fq, Wb, Ab, bits, group, adt, "fp32", env=env)
    _, C1 = run_case(fq, Wb, Ab, bits, group, adt, "fp32", env=env)
    assert torch.equal(C0, C1)
    Cr, D = oracle_ref(Wb, Ab, bits, group, adt)
    assert O.rel_err(torch_to_f64(C0), Cr, D) <= TOL


@pytest.mark.parametrize("path", ["decode", "tc"])
def test_identity_exact_fp32_out(fq, env, path):
    """A = I (M = K = 256): C[k, n] = q[n,k] * s[k/g, n] exactly in fp32-output mode — catches any
    nibble-order / k-permutation / scale-index bug with zero tolerance.
    decode path: run as 16 token tiles of the M<=16 kernel (FQ_GEMM_PATH=decode)."""
    env("path", path)
    K = N = 256
    Wb = gaussian_bits((N, K), 0.02, 5)
    # decode kernel: groups that are a multiple of its K chunk (128 int4 / 64 int8) apply the scale
    # in fp32 on exact integer partials -> exact.  Smaller groups, and the tcgen05 kernel always,
    # dequantize q*s to the activation dtype first (one bf16 rounding: the paper's own "dequantize
    # the weights to match the data type of the activation").
    for bits, group, exact in ((4, 128, True), (8, 64, True), (4, 256, True), (8, 256, True),
                               (4, 64, False), (4, 16, False), (8, 16, False)):
        exact = exact and path == "decode"
        W = bits_to_torch(Wb, "bf16")
        qw = fq.quantize(W, bits, group)
        A = torch.eye(K, dtype=torch.bfloat16, device="cuda")
        C = fq.gemm(A, qw, out_dtype=torch.float32, opts=_opts(fq, env))
        r = O.quantize(O.decode_bits(Wb, "bf16"), bits, group, O.BF16)
        ref = O.dequantize(r.q, r.s, group).T
        if exact:
            assert np.array_equal(torch_to_f64(C), ref)
        else:
            assert np.all(np.abs(torch_to_f64(C) - ref) <= np.abs(ref) * 2.0**-8)


def test_integer_exact_special_case(fq):
    """Small-integer A and weights built by the exact round-trip construction with s = 2^e:
    C is exactly representable, so the fused kernel must return it with zero error."""
    rng = np.random.default_rng(17)
    M, K, N, g = 16, 512, 64, 64
    A = rng.integers(-2, 3, size=(M, K)).astype(np.float32)
    q = rng.integers(-7, 8, size=(N, K))
    s = 2.0 ** -6
    Wv = (q * s).astype(np.float32)
    for n in range(N):
        for j in range(K // g):
            Wv[n, j * g] = np.float32(7.5 * s)  # anchor: makes the group scale exactly s
    from synth import f32_to_bf16_bits
    W = bits_to_torch(f32_to_bf16_bits(Wv), "bf16")
    qw = fq.quantize(W, 4, g)
    Ct = fq.gemm(bits_to_torch(f32_to_bf16_bits(A), "bf16"), qw, out_dtype=torch.float32)
    qx = q.copy()
    qx[:, ::g] = 7
    exact = (A.astype(np.int64) @ qx.T.astype(np.int64)) * s
    assert np.array_equal(torch_to_f64(Ct), exact.astype(np.float64))


@pytest.mark.parametrize("M", [17, 64, 200])
def test_large_m(fq, M):
    Wb, Ab = make_case(M, 1024, 384, 4, 128, seed=M)
    _, C = run_case(fq, Wb, Ab, 4, 128)
    Cr, D = oracle_ref(Wb, Ab, 4, 128, "bf16")
    assert O.rel_err(torch_to_f64(C), Cr, D) <= TOL


@pytest.mark.parametrize("shape", [(12288, 49152), (49152, 12288)])
@pytest.mark.parametrize("bits", [4, 8])
@pytest.mark.parametrize("M", [1, 16, 32])
def test_opt175b_full_size_sampled(fq, shape, bits, M):
    """configs[1] at full size in the bench's launch configuration; parity on 64 sampled columns
    computed by the oracle one by one (scales/codes of those columns only)."""
    K, N = shape
    from synth import gaussian_torch
    W = gaussian_torch((N, K), 0.02, 1000 + K)
    A = gaussian_torch((M, K), 1.0, 2000 + K)
    qw = fq.quantize(W, bits, 128)
    C = fq.gemm(A, qw)
    torch.cuda.synchronize()
    cols = np.random.default_rng(0).choice(N, 64, replace=False)
    Wc = W[torch.from_numpy(cols).cuda()].float().cpu().double().numpy()
    r = O.quantize(Wc, bits, 128, O.BF16)
    Cr, D = O.gemm(A.float().cpu().double().numpy(), r.q, r.s, 128)
    assert O.rel_err(torch_to_f64(C)[:, cols], Cr, D) <= TOL
    # the sampled columns' codes/scales are bit-exact as well
    assert np.array_equal(qw.codes[torch.from_numpy(cols).cuda()].cpu().numpy(), O.pack_codes(r.q, bits))
    assert np.array_equal(qw.scales[:, torch.from_numpy(cols).cuda()].cpu().view(torch.int16).numpy().view(np.uint16),
                          r.s_bits)


@pytest.mark.parametrize("M,K,N,bits,group,adt", [
    (256, 256, 256, 4, 64, "bf16"),        # one tile
    (300, 1024, 392, 4, 128, "bf16"),      # ragged M and N tails, several K blocks
    (520, 2048, 640, 8, 128, "bf16"),
    (257, 1536, 264, 4, 48, "bf16"),       # non-power-of-two group (adaptive ladder of 12288)
    (512, 2048, 1024, 4, 32, "fp16"),
    (384, 1024, 512, 8, 1024, "fp16"),     # per-column
    (17, 512, 256, 4, 16, "bf16"),         # smallest M routed to the tcgen05 kernel
    # two-half (256-row) tiles of the <= 64-token variant: N tail inside the second half, and a
    # last tile whose second half lies entirely past N (not loaded)
    (48, 1024, 456, 4, 32, "fp16"),
    (64, 2048, 392, 8, 128, "bf16"),
    (33, 1536, 1160, 4, 64, "bf16"),
])
def test_tc_path_parity(fq, env, M, K, N, bits, group, adt):
    """Large-M tcgen05 kernel (A6) vs the fp64 oracle on full outputs."""
    env("path", "tc")
    Wb, Ab = make_case(M, K, N, bits, group, adt, seed=M + K, outliers=1)
    _, C = run_case(fq, Wb, Ab, bits, group, adt, env=env)
    Cr, D = oracle_ref(Wb, Ab, bits, group, adt)
    assert O.rel_err(torch_to_f64(C), Cr, D) <= TOL


@pytest.mark.parametrize("shape", [(12288, 49152), (49152, 12288)])
@pytest.mark.parametrize("bits", [4, 8])
def test_opt175b_prefill_sampled(fq, shape, bits):
    """configs[2]: OPT-175B prefill GEMM at M=2048 through the tcgen05 kernel, parity on sampled
    outputs (64 columns x 48 token rows) computed by the oracle."""
    K, N = shape
    M = 2048
    from synth import gaussian_torch
    W = gaussian_torch((N, K), 0.02, 3000 + K)
    A = gaussian_torch((M, K), 1.0, 4000 + K)
    qw = fq.quantize(W, bits, 128)
    C = fq.gemm(A, qw)
    torch.cuda.synchronize()
    rng = np.random.default_rng(1)
    cols = rng.choice(N, 64, replace=False)
    rows = rng.choice(M, 48, replace=False)
    Wc = W[torch.from_numpy(cols).cuda()].float().cpu().double().numpy()
    r = O.quantize(Wc, bits, 128, O.BF16)
    Cr, D = O.gemm(A[torch.from_numpy(rows).cuda()].float().cpu().double().numpy(), r.q, r.s, 128)
    assert O.rel_err(torch_to_f64(C)[np.ix_(rows, cols)], Cr, D) <= TOL


@pytest.mark.parametrize("M,K,N,group,splits", [
    (1, 1152, 264, 384, None),   # groups of 3 chunks: chunk 1 of every other stage starts a group
    (5, 1152, 264, 384, 3),      # splits start at k = 512 / 1024: chunk 1 / 2 of a group
    (12, 2304, 520, 768, 2),     # two MMA token tiles, 6-chunk groups, second split starts at chunk 4
    (8, 3840, 256, 640, 4),      # 5-chunk groups (not a power of two), splits start at chunks 8 / 16 / 24
    (16, 2048, 296, 1024, 3),    # 8-chunk groups, splits start at chunks 6 / 12
])
def test_double_stage_group_phase(fq, env, M, K, N, group, splits):
    """Double-stage decode (two 128-k chunks per stage, int4, groups % 128): the scale row of each
    chunk follows the group boundaries whatever the split's first k (P:149 group-wise scales)."""
    env("path", "decode")
    if splits:
        env("splits", splits)
    Wb, Ab = make_case(M, K, N, 4, group, "bf16", seed=M + K + group, outliers=1)
    _, C = run_case(fq, Wb, Ab, 4, group, "bf16", env=env)
    Cr, D = oracle_ref(Wb, Ab, 4, group, "bf16")
    assert O.rel_err(torch_to_f64(C), Cr, D) <= TOL


@pytest.mark.parametrize("M,K,N,bits,group,adt,splits", [
    (1, 256, 256, 4, 128, "bf16", None),
    (3, 1536, 776, 4, 128, "bf16", None),    # ragged N tail
    (16, 4096, 512, 4, 256, "bf16", 3),      # split-K, deterministic fixup
    (9, 2048, 640, 8, 64, "bf16", None),
    (5, 2048, 384, 8, 128, "fp16", 2),
    (12, 1024, 512, 4, 1024, "fp16", None),  # per-column
    (7, 1024, 768, 4, 64, "fp16", None),     # group 64: group-split nibble path
    (13, 2048, 512, 4, 64, "bf16", 3),       # group 64, two MMA token tiles, split-K
])
def test_decode_kernels(fq, env, M, K, N, bits, group, adt, splits):
    """Decode kernel classes (token tiles x scale paths) with and without forced split-K."""
    env("path", "decode")
    if splits:
        env("splits", splits)
    Wb, Ab = make_case(M, K, N, bits, group, adt, seed=M * 7 + K, outliers=1)
    for _ in range(2):
        _, C = run_case(fq, Wb, Ab, bits, group, adt, env=env)
        Cr, D = oracle_ref(Wb, Ab, bits, group, adt)
        assert O.rel_err(torch_to_f64(C), Cr, D) <= TOL
