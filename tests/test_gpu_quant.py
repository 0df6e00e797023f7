"""GPU parity of kernels A1/A3 (adaptive flags, quantize+pack) against the oracle: bit-exact."""
import numpy as np
import pytest
import torch

from oracle import fq_oracle as O
from synth import gaussian_bits, gaussian_with_outliers_bits
from helpers import bits_to_torch, torch_to_bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fq():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2308_09723_b200 import fq as m
    return m


def run_quant(fq, bits_W, wdt, bits, group, sdt):
    W = bits_to_torch(bits_W, wdt)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    qw = fq.quantize(W, bits, group, scale_dtype={"bf16": torch.bfloat16, "fp16": torch.float16}[sdt], status=st)
    torch.cuda.synchronize()
    return qw, int(st.item())


def check_exact(fq, bits_W, wdt, bits, group, sdt):
    qw, st = run_quant(fq, bits_W, wdt, bits, group, sdt)
    ref = O.quantize(O.decode_bits(bits_W, wdt), bits, group, O.FORMATS[sdt])
    assert st == ref.status
    got_s = torch_to_bits(qw.scales)
    assert np.array_equal(got_s, ref.s_bits), f"scale mismatch at {np.argwhere(got_s != ref.s_bits)[:5]}"
    got_c = qw.codes.cpu().numpy()
    exp_c = O.pack_codes(ref.q, bits)
    if not np.array_equal(got_c, exp_c):
        bad = np.argwhere(got_c != exp_c)[:5]
        raise AssertionError(f"codes mismatch at {bad}")


@pytest.mark.parametrize("sdt", ["bf16", "fp16"])
def test_hand_example_gpu(fq, golden, sdt):
    g = golden("quant_hand.txt")
    col = np.array([float(v) for v in g["column"]], dtype=np.float32)
    W = np.zeros((8, 64), dtype=np.float32)
    W[0, :4] = col
    from synth import f32_to_bf16_bits
    qw, st = run_quant(fq, f32_to_bf16_bits(W), "bf16", 4, 64, sdt)
    assert st == 0
    assert int(torch_to_bits(qw.scales)[0, 0]) == int(g[f"{sdt}.scale_bits"][0], 16)
    assert qw.codes[0, :2].cpu().tolist() == [int(v, 16) for v in g[f"{sdt}.bytes"]]


@pytest.mark.parametrize("bits", [4, 8])
@pytest.mark.parametrize("group", [16, 32, 48, 64, 96, 128, 256, 768])
def test_quantize_exact_groups(fq, bits, group):
    W = gaussian_with_outliers_bits((40, 1536), 0.02, 1000 + group, 3, 0.5)
    check_exact(fq, W, "bf16", bits, group, "bf16")


@pytest.mark.parametrize("wdt,sdt", [("bf16", "bf16"), ("fp16", "fp16"), ("bf16", "fp16")])
def test_quantize_nonfinite_zero_groups(fq, wdt, sdt):
    """Non-finite elements and all-zero groups at a 512-wide shape, three (bits, group) pairs."""
    from synth import f32_to_bf16_bits
    W = np.random.default_rng(5).normal(0, 0.02, (24, 512)).astype(np.float32)
    W[1, 3] = np.inf
    W[2, 300] = np.nan
    W[5, 128:256] = 0.0
    bitsW = f32_to_bf16_bits(W) if wdt == "bf16" else W.astype(np.float16).view(np.uint16)
    for bits, group in ((4, 128), (8, 64), (4, 16)):
        check_exact(fq, bitsW, wdt, bits, group, sdt)


@pytest.mark.parametrize("wdt", ["bf16", "fp16", "fp32"])
@pytest.mark.parametrize("sdt", ["bf16", "fp16"])
def test_quantize_exact_dtypes(fq, wdt, sdt):
    W = gaussian_bits((24, 512), 0.02, 7, wdt)
    check_exact(fq, W, wdt, 4, 64, sdt)
    check_exact(fq, W, wdt, 8, 512, sdt)  # per-column


@pytest.mark.parametrize("wdt,K,bits,group", [("bf16", 32768, 4, 128), ("fp16", 49152, 8, 64),
                                               ("bf16", 30720, 4, 15360), ("fp32", 24576, 4, 256)])
def test_quantize_exact_long_columns(fq, wdt, K, bits, group):
    """Columns longer than one CTA's K-slice are quantized by several CTAs (whole groups each);
    a group longer than the slice target keeps one group per CTA."""
    W = gaussian_bits((8, K), 0.02, K + bits, wdt)
    check_exact(fq, W, wdt, bits, group, "bf16")


def test_quantize_exact_tiny_config(fq):
    # configs[0]: M=1, K=256, N=256, int4 group=64, bf16
    W = gaussian_bits((256, 256), 0.02, 1001)
    check_exact(fq, W, "bf16", 4, 64, "bf16")


@pytest.mark.parametrize("wdt", ["bf16", "fp16"])
@pytest.mark.parametrize("group", [16, 32, 256])
@pytest.mark.parametrize("order", ["sorted", "shuffled"])
def test_quantize_all_16bit_patterns(fq, wdt, group, order):
    """Every finite bf16 / fp16 value, in pattern order (groups of neighbouring magnitudes: the
    +-7.5 / 127.5 tie cases) and in a seeded shuffle (each value under many unrelated scales); codes
    and scales must match the oracle bit for bit at every bit width.  group 16 runs the per-column
    kernel, 32 / 256 the warp-per-unit kernel."""
    allb = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    allb = allb[np.isfinite(O.decode_bits(allb, wdt))]
    if order == "shuffled":
        allb = np.random.default_rng(group).permutation(allb)
    K = 1024 + 512  # one full and one partial 1024-element unit per column
    n = ((allb.size + K - 1) // K + 7) // 8 * 8
    buf = np.zeros(n * K, dtype=np.uint16)
    buf[: allb.size] = allb
    W = buf.reshape(n, K)
    for bits in (4, 8, 3, 2):
        check_exact(fq, W, wdt, bits, group, wdt)


@pytest.mark.parametrize("wdt", ["bf16", "fp16"])
def test_quantize_exact_ties_both_signs(fq, wdt):
    """Groups whose scale is exact (amax = (2^b - 1)/2 * 2^-e, so s = 2^-e) holding every
    half-integer multiple (k + 1/2) s of both signs: each is an exact tie of |x|/s that App. A's
    rounding (read as round-half-away, DESIGN R3) must send away from zero, plus the integer
    multiples and -0.  Codes and scales must match the oracle bit for bit."""
    for bits in (4, 8):
        qmax = (1 << (bits - 1))
        e = 6
        halves = [(k + 0.5) * 2.0 ** -e for k in range(-qmax, qmax)]  # -(qmax - 1/2) s .. (qmax - 1/2) s
        ints = [k * 2.0 ** -e for k in range(-qmax + 1, qmax)]
        vals = np.array(halves + ints + [-0.0], dtype=np.float32)
        group = 64 if bits == 4 else 512
        K = 1024
        rows = []
        for r in range(8):
            row = np.resize(np.random.default_rng(r).permutation(vals), K).astype(np.float32)
            for g0 in range(0, K, group):  # plant the anchor amax = (qmax - 1/2) s in every group
                row[g0 + r % group] = (qmax - 0.5) * 2.0 ** -e * (1 if r % 2 else -1)
            rows.append(row)
        W = np.stack(rows)
        if wdt == "bf16":
            from synth import f32_to_bf16_bits
            bitsW = f32_to_bf16_bits(W)
        else:
            bitsW = W.astype(np.float16).view(np.uint16)
        check_exact(fq, bitsW, wdt, bits, group, wdt)


@pytest.mark.parametrize("group", [16, 64])
def test_quantize_fp32_near_ties(fq, group):
    """fp32 W (24 significant bits) one ulp either side of every half-integer multiple (k + 1/2) s
    under non-power-of-two scales s: |x| / s sits within ~2^-23 of a tie, so round_half_away must be
    decided exactly (the oracle divides in float64).  Both kernels: group 16 / 64."""
    rows = []
    for bits in (4, 8):
        qmax = 1 << (bits - 1)
        for m in (3.0, 5.0, 1.96875 * 64, 1.5 * 128, 127.0):  # bf16-exact scale mantissas
            s = m * 2.0 ** -12
            vals = []
            for k in range(-qmax, qmax):
                t = np.float32((k + 0.5) * s)
                vals += [np.nextafter(t, np.float32(np.inf)), np.nextafter(t, np.float32(-np.inf)), t]
            vals = np.array(vals, dtype=np.float32)
            K = ((vals.size + group - 2) // (group - 1)) * group
            K = (K + 1023) // 1024 * 1024
            row = np.zeros(K, dtype=np.float32)
            per = group - 1
            for g0, v0 in zip(range(0, K, group), range(0, vals.size, per)):
                chunk = vals[v0:v0 + per]
                row[g0:g0 + chunk.size] = chunk
                row[g0 + group - 1] = np.float32((qmax - 0.5) * s)  # anchor: amax -> this s
            rows.append((bits, row))
    for bits in (4, 8):
        W = np.stack([r for b, r in rows if b == bits])
        W = np.concatenate([W, np.zeros(((8 - W.shape[0] % 8) % 8, W.shape[1]), np.float32)])
        check_exact(fq, W.view(np.uint32), "fp32", bits, group, "bf16")


@pytest.mark.parametrize("wdt", ["bf16", "fp16"])
@pytest.mark.parametrize("group", [16, 64, 1024])
def test_quantize_subnormal_fp16_scales(fq, wdt, group):
    """Groups with amax from 1e-9 to 1e-3 under fp16 scales: below amax ~ 2^-14 (2^b - 1) / 2 the
    scale is an fp16 subnormal with few significant bits, so |x| / s can leave the code range on
    either side and must be clamped at both ends (and ties still decided exactly)."""
    rng = np.random.default_rng(group)
    N, K = 64, 2048
    amax = 10.0 ** rng.uniform(-9, -3, size=(N, K // group))
    W = rng.uniform(-1, 1, size=(N, K)) * np.repeat(amax, group, axis=1)
    if wdt == "bf16":
        from synth import f32_to_bf16_bits
        bitsW = f32_to_bf16_bits(W.astype(np.float32))
    else:
        bitsW = W.astype(np.float16).view(np.uint16)
    for bits in (4, 8, 3, 2):
        check_exact(fq, bitsW, wdt, bits, group, "fp16")


def test_zero_and_nonfinite_status(fq):
    from synth import f32_to_bf16_bits
    W = np.zeros((8, 64), dtype=np.float32)
    W[1, 3] = np.inf
    W[2, 40] = np.nan
    W[3, 5] = 0.25
    check_exact(fq, f32_to_bf16_bits(W), "bf16", 4, 32, "bf16")
    W2 = np.full((8, 64), 1e6, dtype=np.float32)
    check_exact(fq, W2.view(np.uint32), "fp32", 4, 32, "fp16")  # fp16 scale overflow -> status 2


@pytest.mark.parametrize("K,N,alpha,outliers", [(128, 8, 500, 0), (128, 8, 500, 1), (4096, 64, 500, 2),
                                                (12288, 32, 300, 1), (7168, 16, 800, 3)])
def test_adapt_flags_match_oracle(fq, K, N, alpha, outliers):
    if outliers:
        Wb = gaussian_with_outliers_bits((N, K), 0.01, K + N, outliers, 1.0)
    else:
        Wb = gaussian_bits((N, K), 1.0, K + N)
    Wd = O.decode_bits(Wb, "bf16")
    exp_flags = O.adapt_flags(Wd, alpha, 16)
    W = bits_to_torch(Wb, "bf16")
    nlev = fq.fq_adapt_levels(K, 16)
    flags = torch.zeros(nlev - 1, dtype=torch.int32, device="cuda")
    fq.fq_adapt_flags(W, alpha, 16, flags)
    got = [bool(f) for f in flags.cpu().tolist()]
    assert got == exp_flags
    assert fq.adapt_group(W, alpha, 16) == O.adapt_group_size(Wd, alpha, 16)
