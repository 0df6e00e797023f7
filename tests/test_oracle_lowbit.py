"""Pins for the oracle's int3 / int2 packing and quantization (CPU only).

The paper evaluates int3 weights (tab:optiml-mt) but ships no kernel or layout
for them; the packed layout is SPEC.md:96's little-endian bit stream.  Pins: the
hand-packed bytes of tests/golden/int3_hand.txt, the independent int4 / int8 packers (the bit
stream at b = 4 / 8 must reproduce them), the round-trip law, and App. A at b = 3 by hand.
"""
import numpy as np
import pytest

from oracle import fq_oracle as O
from synth import gaussian_bits


def _ints(v):
    return [int(x, 0) for x in v]


@pytest.mark.parametrize("b", [2, 3])
def test_bitstream_hand_bytes(golden, b):
    g = golden("int3_hand.txt")
    q = np.array([_ints(g[f"int{b}.codes"])], dtype=np.int8)
    want = _ints(g[f"int{b}.bytes"])
    got = O.pack_codes(q, b)
    assert got.tolist() == [want]
    assert O.unpack_codes(got, b, q.shape[1]).tolist() == q.tolist()


@pytest.mark.parametrize("b", [4, 8])
def test_bitstream_equals_nibble_and_byte_packers(b):
    # the general little-endian stream at b = 4 / 8 is the canonical int4 (low nibble first) /
    # int8 layout, which pack_codes implements by an independent formula
    rng = np.random.default_rng(b)
    q = rng.integers(-(1 << (b - 1)), 1 << (b - 1), size=(7, 64)).astype(np.int8)
    assert np.array_equal(O.pack_bitstream(q, b), O.pack_codes(q, b))
    assert np.array_equal(O.unpack_bitstream(O.pack_codes(q, b), b, 64), q)


@pytest.mark.parametrize("b", [2, 3])
def test_bitstream_round_trip_and_size(b):
    rng = np.random.default_rng(10 + b)
    for K in (8, 64, 136):
        q = rng.integers(-(1 << (b - 1)), 1 << (b - 1), size=(5, K)).astype(np.int8)
        p = O.pack_codes(q, b)
        assert p.shape == (5, K * b // 8)  # SPEC.md:138 ceil(rows*b/8) bytes per column
        assert np.array_equal(O.unpack_codes(p, b, K), q)


def test_int3_bit_positions_one_hot():
    # a single code -1 (all ones) at position k sets exactly stream bits 3k..3k+2
    for k in range(8):
        q = np.zeros((1, 8), dtype=np.int8)
        q[0, k] = -1
        p = O.pack_codes(q, 3)
        bits = [(p[0, i // 8] >> (i % 8)) & 1 for i in range(24)]
        assert [i for i, v in enumerate(bits) if v] == [3 * k, 3 * k + 1, 3 * k + 2]


def test_int3_quantize_hand(golden):
    g = golden("int3_hand.txt")
    W = np.array([[float(v) for v in g["int3q.column"]]])
    r = O.quantize(W, 3, 8, O.BF16)
    assert r.s[0, 0] == float(g["int3q.scale"][0])
    assert int(r.s_bits[0, 0]) == int(g["int3q.scale_bits"][0], 0)
    assert r.q[0].tolist() == _ints(g["int3q.codes"])
    assert O.pack_codes(r.q, 3)[0].tolist() == _ints(g["int3q.bytes"])


@pytest.mark.parametrize("b", [2, 3])
def test_lowbit_quantize_invariants(b):
    # App. A error bound |x - q s| <= s/2 except the clamped positive extreme; codes in range
    W = O.decode_bits(gaussian_bits((16, 256), 0.02, 77 + b), "bf16")
    r = O.quantize(W, b, 64, O.BF16)
    lo, hi = -(1 << (b - 1)), (1 << (b - 1)) - 1
    assert r.q.min() >= lo and r.q.max() <= hi
    Wd = O.dequantize(r.q, r.s, 64)
    s_full = np.repeat(r.s.T, 64, axis=1)
    inner = (r.q > lo) & (r.q < hi)
    assert np.all(np.abs(W - Wd)[inner] <= s_full[inner] / 2 * (1 + 1e-12))
