"""Pins for the oracle's int8-activation x int4-weight path with integer group scales
(§5; readings R15-R19 in DESIGN.md), CPU only.

Pinned by: the hand-worked fixture tests/golden/intscale_hand.txt; numpy float32 arithmetic (IEEE
correctly rounded division) for the fp32 scale and quotient decisions; exact rational arithmetic
(fractions) for the ceil / integer decisions taken in float64; the exact round-trip construction
(anchors at 7.5 sigma z); brute-force Python loops for the integer GEMM.
"""
from fractions import Fraction

import numpy as np
import pytest

from oracle import fq_oracle as O
from synth import activations_bits, gaussian_bits, gaussian_with_outliers_bits


def _f(v):
    return [float(x) for x in v]


def test_hand_fixture(golden):
    g = golden("intscale_hand.txt")
    W = np.array([_f(g["w.column"])])
    grp = int(g["w.group"][0])
    r = O.quantize_intscale(W, 4, grp)
    sig_bits = int(g["w.sigma_bits"][0], 0)
    assert np.float32(r.sigma[0]).view(np.uint32) == sig_bits
    assert r.z[:, 0].tolist() == [int(x) for x in g["w.z"]]
    assert r.q[0].tolist() == [int(x) for x in g["w.codes"]]
    A = np.array([_f(g["a.row"])])
    a = O.quantize_acts_i8(A)
    assert a.s_a[0] == float(g["a.scale"][0])
    assert a.a_q[0].tolist() == [int(x) for x in g["a.codes"]]
    C, D, acc = O.gemm_i8(a.a_q, a.s_a, r.q, r.z, r.sigma, grp)
    assert int(acc[0, 0]) == int(g["gemm.acc"][0])
    sigma = float(np.uint32(sig_bits).view(np.float32))
    assert C[0, 0] == int(g["gemm.acc"][0]) * sigma  # 14 x 24 bits: exact in float64


def test_sigma_and_act_scale_equal_ieee_fp32_division():
    # R16 / R17: the float64 quotient rounded once more to fp32 equals the IEEE fp32 division
    # (numpy float32 arithmetic) -- no double rounding for /120 and /127
    Wb = gaussian_bits((512, 256), 0.02, 5)
    W = O.decode_bits(Wb, "bf16")
    r = O.quantize_intscale(W, 4, 64)
    amax_col = np.abs(W).max(axis=1).astype(np.float32)
    want = (np.float32(2) * amax_col) / np.float32(240)
    assert np.array_equal(r.sigma.astype(np.float32), want)
    A = O.decode_bits(activations_bits(300, 512, 6), "bf16")
    a = O.quantize_acts_i8(A)
    want_a = np.abs(A).max(axis=1).astype(np.float32) / np.float32(127)
    assert np.array_equal(a.s_a.astype(np.float32), want_a)


def test_z_and_codes_equal_exact_rational_decisions():
    # the ceil (z) and integer (q) decisions taken in float64 equal the exact rational ones
    Wb = gaussian_with_outliers_bits((24, 256), 0.02, 11, 3, 0.5)
    W = O.decode_bits(Wb, "bf16")
    g = 32
    r = O.quantize_intscale(W, 4, g)
    for n in range(W.shape[0]):
        sig = Fraction(float(r.sigma[n]))
        for j in range(W.shape[1] // g):
            blk = [Fraction(float(x)) for x in W[n, j * g:(j + 1) * g]]
            amax = max(abs(x) for x in blk)
            ratio = 2 * amax / (15 * sig) if sig else Fraction(0)
            zc = -((-ratio.numerator) // ratio.denominator)  # exact ceil
            z = min(16, max(1, zc))
            assert int(r.z[j, n]) == z
            S = sig * z
            for i, x in enumerate(blk):
                y = x / S if S else Fraction(0)
                t = abs(y)
                m = t.numerator // t.denominator
                if t - m >= Fraction(1, 2):
                    m += 1
                qv = max(-8, min(7, m if y >= 0 else -m))
                assert int(r.q[n, j * g + i]) == qv


def test_round_trip_construction():
    # W = sigma z q exactly (sigma = 2^e, q in [-7, 7]) plus one anchor -7.5 sigma z per group; one
    # group per column has z = 16, so amax_col = 120 sigma and sigma, z, q are recovered exactly
    rng = np.random.default_rng(3)
    N, K, g = 32, 256, 32
    G = K // g
    e = -9
    sig = 2.0 ** e
    W = np.zeros((N, K))
    zs = rng.integers(1, 17, size=(G, N))
    zs[rng.integers(0, G, size=N), np.arange(N)] = 16
    qs = rng.integers(-7, 8, size=(N, K))
    for n in range(N):
        for j in range(G):
            z = zs[j, n]
            W[n, j * g:(j + 1) * g] = sig * z * qs[n, j * g:(j + 1) * g]
            a = rng.integers(0, g)
            W[n, j * g + a] = -7.5 * sig * z
            qs[n, j * g + a] = -8
    assert np.array_equal(O.round_to_format(W, O.BF16), W)  # bf16-exact construction
    r = O.quantize_intscale(W, 4, g)
    assert np.all(r.sigma == sig)
    assert np.array_equal(r.z.astype(np.int64), zs)
    assert np.array_equal(r.q.astype(np.int64), qs)


def test_act_round_trip_construction():
    rng = np.random.default_rng(4)
    M, K = 16, 128
    q = rng.integers(-127, 128, size=(M, K))
    q[np.arange(M), rng.integers(0, K, size=M)] = 127 * rng.choice([-1, 1], size=M)
    sc = 2.0 ** rng.integers(-20, 10, size=M)
    A = q * sc[:, None]
    a = O.quantize_acts_i8(A)
    assert np.array_equal(a.s_a, sc)
    assert np.array_equal(a.a_q.astype(np.int64), q)


def test_act_quant_invariants_and_edges():
    A = O.decode_bits(activations_bits(64, 384, 9), "bf16")
    A[3] = 0.0
    a = O.quantize_acts_i8(A)
    assert a.a_q.min() >= -127 and a.a_q.max() <= 127
    assert a.s_a[3] == 0 and np.all(a.a_q[3] == 0)
    rows = np.arange(64) != 3
    err = np.abs(A[rows] - a.a_q[rows] * a.s_a[rows, None])
    # half a step, plus the fp32 rounding of s_a and of the quotient (|a / s_a| <= 127.000..)
    assert np.all(err <= a.s_a[rows, None] * (0.5 + 128 * 2.0**-23))
    am = np.abs(A[rows]).argmax(axis=1)
    assert np.all(np.abs(a.a_q[rows][np.arange(63), am]) == 127)
    B = A.copy()
    B[5, 7] = np.nan
    assert O.quantize_acts_i8(B).status == 1


def test_intscale_invariants():
    W = O.decode_bits(gaussian_with_outliers_bits((64, 512), 0.02, 21, 4, 0.8), "bf16")
    r = O.quantize_intscale(W, 4, 64)
    assert r.z.min() >= 1 and r.z.max() <= 16 and np.all(r.z.max(axis=0) == 16)
    S = r.sigma[None, :] * r.z  # effective group scale >= App. A's fine scale (ceil) ...
    fine = 2 * O.group_amax(W, 64) / 15
    assert np.all((S >= fine) | (r.z == 16))
    assert np.all(S >= fine * (1 - 2.0**-23))  # ... up to sigma's fp32 rounding where z is clamped
    assert r.q.min() >= -8 and r.q.max() <= 7
    Wd = r.q * np.repeat(S.T, 64, axis=1)
    inner = (r.q > -8) & (r.q < 7)
    assert np.all(np.abs(W - Wd)[inner] <= np.repeat(S.T, 64, axis=1)[inner] / 2 * (1 + 1e-12))


def test_intscale_nonfinite_and_zero_columns():
    W = O.decode_bits(gaussian_bits((4, 128), 0.02, 2), "bf16")
    W[1, 5] = np.inf
    W[2] = 0.0
    r = O.quantize_intscale(W, 4, 32)
    assert r.status == 1
    assert r.sigma[1] == 0 and np.all(r.q[1] == 0) and np.all(r.z[:, 1] == 1)
    assert r.sigma[2] == 0 and np.all(r.q[2] == 0) and np.all(r.z[:, 2] == 1)
    assert r.sigma[0] > 0 and r.sigma[3] > 0


def test_gemm_i8_brute_force():
    rng = np.random.default_rng(8)
    M, N, K, g = 3, 5, 64, 16
    a = rng.integers(-127, 128, size=(M, K)).astype(np.int8)
    q = rng.integers(-8, 8, size=(N, K)).astype(np.int8)
    z = rng.integers(1, 17, size=(K // g, N)).astype(np.uint8)
    sa = rng.random(M) + 0.5
    sg = rng.random(N) * 1e-3
    C, D, acc = O.gemm_i8(a, sa, q, z, sg, g)
    for m in range(M):
        for n in range(N):
            s = 0
            d = 0
            for k in range(K):
                t = int(a[m, k]) * int(q[n, k]) * int(z[k // g, n])
                s += t
                d += abs(t)
            assert int(acc[m, n]) == s
            assert C[m, n] == pytest.approx(s * sa[m] * sg[n], rel=1e-15, abs=0)
            assert D[m, n] == pytest.approx(d * sa[m] * sg[n], rel=1e-15, abs=0)
