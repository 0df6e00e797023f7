"""Pins for the oracle GEMM C = A . dequant(Q)^T (§4.1) and its tolerance metric."""
import itertools
import math

import numpy as np

from oracle import fq_oracle as O
from synth import activations_bits, gaussian_bits


def test_integer_exact_special_case():
    """A small integers, q from the round-trip construction, s = 2^e:  C = (A @ q^T) * 2^e exactly."""
    rng = np.random.default_rng(17)
    M, K, N, g = 5, 256, 12, 64
    A = rng.integers(-3, 4, size=(M, K)).astype(np.float64)
    q = rng.integers(-7, 8, size=(N, K))
    e = -6
    s = np.full((K // g, N), 2.0**e)
    C, D = O.gemm(A, q, s, g)
    exact = (A.astype(np.int64) @ q.T.astype(np.int64)).astype(np.float64) * 2.0**e
    assert np.array_equal(C, exact)
    assert np.array_equal(D, (np.abs(A).astype(np.int64) @ np.abs(q).T.astype(np.int64)) * 2.0**e)


def test_one_hot_and_identity():
    W = O.decode_bits(gaussian_bits((16, 128), 0.02, 3), "bf16")
    r = O.quantize(W, 4, 32, O.BF16)
    deq = O.dequantize(r.q, r.s, 32)
    C, _ = O.gemm(np.eye(128), r.q, r.s, 32)
    assert np.array_equal(C, deq.T)            # C[k, n] = q[n, k] s[k/g, n]
    A = np.zeros((1, 128))
    A[0, 77] = 1
    C1, _ = O.gemm(A, r.q, r.s, 32)
    assert np.array_equal(C1[0], deq[:, 77])


def test_brute_force_loops_tiny():
    A = O.decode_bits(activations_bits(2, 32, 4), "bf16")
    W = O.decode_bits(gaussian_bits((3, 32), 0.02, 5), "bf16")
    r = O.quantize(W, 4, 16, O.BF16)
    C, D = O.gemm(A, r.q, r.s, 16)
    for m, n in itertools.product(range(2), range(3)):
        acc = 0.0
        dacc = 0.0
        for k in range(32):
            p = A[m, k] * float(r.q[n, k]) * r.s[k // 16, n]
            acc = math.fsum([acc, p])
            dacc += abs(p)
        assert abs(C[m, n] - acc) <= 1e-15 * dacc
        assert abs(D[m, n] - dacc) <= 1e-15 * dacc


def test_linearity_and_cols_subset():
    A = O.decode_bits(activations_bits(3, 256, 6), "bf16")
    B = O.decode_bits(activations_bits(3, 256, 7), "bf16")
    W = O.decode_bits(gaussian_bits((20, 256), 0.02, 8), "bf16")
    r = O.quantize(W, 8, 128, O.BF16)
    C1, D1 = O.gemm(A, r.q, r.s, 128)
    C2, _ = O.gemm(B, r.q, r.s, 128)
    C3, _ = O.gemm(2 * A - 3 * B, r.q, r.s, 128)
    assert np.allclose(C3, 2 * C1 - 3 * C2, rtol=0, atol=1e-12 * np.abs(D1).max() * 5)
    cols = np.array([0, 5, 19])
    Cs, Ds = O.gemm(A, r.q, r.s, 128, cols)
    assert np.array_equal(Cs, C1[:, cols]) and np.array_equal(Ds, D1[:, cols])


def test_rel_err_semantics():
    C = np.array([[1.0, 0.0]])
    D = np.array([[2.0, 0.0]])
    assert abs(O.rel_err(np.array([[1.002, 0.0]]), C, D) - 0.001) < 1e-15
    assert O.rel_err(np.array([[1.0, 1e-30]]), C, D) == math.inf


def test_grouped_matches_per_expert():
    A = O.decode_bits(activations_bits(7, 64, 9), "bf16")
    off = np.array([0, 3, 3, 7])
    ex = []
    for e in range(3):
        W = O.decode_bits(gaussian_bits((8, 64), 0.02, 30 + e), "bf16")
        r = O.quantize(W, 4, 16 * (e + 1) if 64 % (16 * (e + 1)) == 0 else 64, O.BF16)
        ex.append((r.q, r.s, 64 // r.s.shape[0]))
    C, D = O.gemm_grouped(A, off, ex)
    C0, _ = O.gemm(A[0:3], *ex[0])
    C2, _ = O.gemm(A[3:7], *ex[2])
    assert np.array_equal(C[0:3], C0) and np.array_equal(C[3:7], C2)
