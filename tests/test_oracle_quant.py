"""Pins for the oracle's formats, quantizer and packing (CPU only).

Each pin is fixed by something other than the oracle itself: numpy/torch IEEE casts, the
hand-worked example of tests/golden/quant_hand.txt (App. A), exact rational
arithmetic, closed-form round-trip constructions and the App. A error bound.
"""
import math
from fractions import Fraction

import numpy as np
import pytest
import torch

from oracle import fq_oracle as O
from synth import gaussian_bits


# ---------------------------------------------------------------- formats
def test_round_to_bf16_matches_torch_cast_on_fp32_patterns():
    rng = np.random.default_rng(0)
    u = rng.integers(0, 2**32, size=2_000_000, dtype=np.uint64).astype(np.uint32)
    f = u.view(np.float32)
    f = f[np.isfinite(f)]
    ref = torch.from_numpy(f.copy()).to(torch.bfloat16).to(torch.float64).numpy()
    got = O.round_to_format(f.astype(np.float64), O.BF16)
    assert np.array_equal(got, ref)


def test_round_to_fp16_matches_numpy_cast_on_doubles():
    rng = np.random.default_rng(1)
    x = rng.standard_normal(1_000_000) * np.exp2(rng.integers(-30, 18, 1_000_000))
    ref = x.astype(np.float16).astype(np.float64)
    got = O.round_to_format(x, O.FP16)
    assert np.array_equal(got, ref)


def test_round_to_format_hand_values():
    # ties to even at 1 + 2^-8 (bf16 keeps 7 fraction bits)
    assert O.round_to_format(np.array([1 + 2**-8]), O.BF16)[0] == 1.0
    assert O.round_to_format(np.array([1 + 3 * 2**-8]), O.BF16)[0] == 1 + 2**-6
    # smallest bf16 subnormal 2^-133; half of it ties to 0 (even)
    assert O.round_to_format(np.array([2.0**-133]), O.BF16)[0] == 2.0**-133
    assert O.round_to_format(np.array([2.0**-134]), O.BF16)[0] == 0.0
    assert O.round_to_format(np.array([65520.0]), O.FP16)[0] == math.inf
    assert O.round_to_format(np.array([65519.0]), O.FP16)[0] == 65504.0


def test_round_half_away_edges():
    y = np.array([0.49999999999999994, 0.5, -0.5, 1.5, 2.5, -2.5, 7.5, -7.5, -7.4999999])
    assert O.round_half_away(y).tolist() == [0, 1, -1, 2, 3, -3, 8, -8, -7]


# ---------------------------------------------------------------- hand example (golden)
@pytest.mark.parametrize("fmt", ["bf16", "fp16"])
def test_hand_example(golden, fmt):
    g = golden("quant_hand.txt")
    col = np.array([float(v) for v in g["column"]])
    F = O.FORMATS[fmt]
    for K in (4, 64):  # K=64: zero padded (ABI minimum); amax and codes are unchanged
        W = np.zeros((1, K))
        W[0, :4] = col
        r = O.quantize(W, 4, K, F)
        assert r.s[0, 0] == float(g[f"{fmt}.scale"][0])
        assert r.s_bits[0, 0] == int(g[f"{fmt}.scale_bits"][0], 16)
        assert r.q[0, :4].tolist() == [int(v) for v in g[f"{fmt}.codes"]]
        assert np.all(r.q[0, 4:] == 0)
        packed = O.pack_codes(r.q, 4)
        assert packed[0, :2].tolist() == [int(v, 16) for v in g[f"{fmt}.bytes"]]
    if fmt == "bf16":
        deq = O.dequantize(r.q, r.s, 64)[0, :4]
        assert deq.tolist() == [float(v) for v in g["bf16.dequant"]]
        A = np.zeros((1, 64))
        A[0, :4] = 1.0
        C, _ = O.gemm(A, r.q, r.s, 64)
        assert C[0, 0] == float(g["bf16.gemm_ones"][0])


# ---------------------------------------------------------------- exact rational brute force
def _rne_fraction(x: Fraction, p: int, emin: int) -> Fraction:
    """Round a positive rational to p significant bits (ties to even) with integer arithmetic."""
    if x == 0:
        return Fraction(0)
    e = x.numerator.bit_length() - x.denominator.bit_length()
    if Fraction(2) ** e > x:
        e -= 1
    e = max(e, emin)
    quantum = Fraction(2) ** (e - (p - 1))
    n = x / quantum
    fl = n.numerator // n.denominator
    rem = n - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    return fl * quantum


def _round_half_away_fraction(y: Fraction) -> int:
    a = abs(y)
    fl = a.numerator // a.denominator
    if a - fl >= Fraction(1, 2):
        fl += 1
    return fl if y >= 0 else -fl


@pytest.mark.parametrize("bits,fmt", [(4, "bf16"), (8, "bf16"), (4, "fp16"), (8, "fp16")])
def test_quantize_vs_exact_rationals(bits, fmt):
    F = O.FORMATS[fmt]
    W = O.decode_bits(gaussian_bits((6, 256), 0.02, 11, "bf16"), "bf16")
    W[0, 5] = 0.5  # an outlier in one group
    r = O.quantize(W, bits, 32, F)
    lo, hi = -(1 << (bits - 1)), (1 << (bits - 1)) - 1
    for n in range(W.shape[0]):
        for j in range(W.shape[1] // 32):
            grp = [Fraction(float(v)) for v in W[n, j * 32:(j + 1) * 32]]
            amax = max(abs(v) for v in grp)
            s = _rne_fraction(2 * amax / ((1 << bits) - 1), F.p, F.emin)
            assert Fraction(float(r.s[j, n])) == s
            for i, v in enumerate(grp):
                qq = 0 if s == 0 else min(hi, max(lo, _round_half_away_fraction(v / s)))
                assert int(r.q[n, j * 32 + i]) == qq


def test_ties_exactly_on_half_steps_bf16():
    """Exhaustive over every finite bf16 value x, for several bf16 scales s: the oracle's code
    equals the exact rational decision (half away from zero, then clamp)."""
    allbits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    xs = O.decode_bits(allbits, "bf16")
    xs = xs[np.isfinite(xs)]
    for s in (0.53515625, 2.0**-7, 0.0078125 * 3, 1.5, 0.013671875):
        y = xs / s
        sel = np.abs(y) < 9          # in-range codes (others clamp)
        x_sel = xs[sel]
        # the oracle's code decision: float64 quotient + round_half_away
        got = O.round_half_away(x_sel / s)
        for x, qv in zip(x_sel[::7], got[::7]):
            assert qv == _round_half_away_fraction(Fraction(float(x)) / Fraction(s))


# ---------------------------------------------------------------- closed-form round trip
@pytest.mark.parametrize("bits", [4, 8])
def test_representable_round_trip(bits):
    """Groups built as {anchor +-((2^b-1)/2) s} U {q s : |q| <= 2^(b-1)-1} with s having few
    significant bits: 2*amax/(2^b-1) == s exactly, codes == q, anchor -> +hi / -(hi+1)."""
    rng = np.random.default_rng(5)
    half = ((1 << bits) - 1) / 2
    hi = (1 << (bits - 1)) - 1
    g = 64
    N, G = 7, 4
    q = rng.integers(-hi, hi + 1, size=(N, G * g))
    s = np.empty((G, N))
    for n in range(N):
        for j in range(G):
            if bits == 4:
                s[j, n] = rng.choice([9, 11, 13, 15]) * 2.0 ** int(rng.integers(-12, -4))
            else:
                s[j, n] = 2.0 ** int(rng.integers(-14, -6))
    W = q * np.repeat(s.T, g, axis=1)
    anchors = rng.integers(0, g, size=(N, G))
    signs = rng.choice([-1, 1], size=(N, G))
    exp_q = q.copy()
    for n in range(N):
        for j in range(G):
            k = j * g + anchors[n, j]
            W[n, k] = signs[n, j] * half * s[j, n]
            exp_q[n, k] = hi if signs[n, j] > 0 else -hi - 1
    # all values are exact bf16 values
    assert np.array_equal(O.round_to_format(W, O.BF16), W)
    r = O.quantize(W, bits, g, O.BF16)
    assert np.array_equal(r.s, s)
    assert np.array_equal(r.q, exp_q)


# ---------------------------------------------------------------- App. A error bound / invariants
@pytest.mark.parametrize("bits,group", [(4, 16), (4, 64), (8, 128), (4, 256)])
def test_error_bound_and_ranges(bits, group):
    W = O.decode_bits(gaussian_bits((16, 512), 0.02, 21), "bf16")
    r = O.quantize(W, bits, group, O.BF16)
    lo, hi = -(1 << (bits - 1)), (1 << (bits - 1)) - 1
    assert r.q.min() >= lo and r.q.max() <= hi
    deq = O.dequantize(r.q, r.s, group)
    sfull = np.repeat(r.s.T, group, axis=1)
    err = np.abs(W - deq)
    clamped = (r.q == hi) & (W / sfull > hi + 0.5 - 1e-12)
    assert np.all(err[~clamped] <= sfull[~clamped] / 2)
    # clamped positive extreme: |x - hi s| <= s (0.5 + (2^b-1)/2 * 2^-8)
    assert np.all(err[clamped] <= sfull[clamped] * (0.5 + ((1 << bits) - 1) / 2 * 2.0**-8))
    # monotone refinement: child scale <= parent scale
    r2 = O.quantize(W, bits, group * 2, O.BF16)
    assert np.all(r.s <= np.repeat(r2.s, 2, axis=0))


def test_zero_group_and_status():
    W = np.zeros((2, 64))
    W[1, 0] = 1.0
    r = O.quantize(W, 4, 32, O.BF16)
    assert r.s[0, 0] == 0 and r.s[1, 0] == 0 and np.all(r.q[0] == 0)
    assert r.status == 0
    W[0, 3] = np.nan
    assert O.quantize(W, 4, 32, O.BF16).status == 1
    W2 = np.full((1, 32), 1e6)  # fp16 scale 2e6/15 overflows
    r3 = O.quantize(W2, 4, 32, O.FP16)
    assert r3.status == 2 and np.all(r3.q == 0) and r3.s[0, 0] == 0


@pytest.mark.parametrize("bits", [4, 8])
def test_pack_unpack_round_trip(bits):
    rng = np.random.default_rng(3)
    lo, hi = -(1 << (bits - 1)), (1 << (bits - 1)) - 1
    q = rng.integers(lo, hi + 1, size=(5, 96)).astype(np.int8)
    p = O.pack_codes(q, bits)
    assert p.shape == (5, 96 * bits // 8)
    assert np.array_equal(O.unpack_codes(p, bits, 96), q)
