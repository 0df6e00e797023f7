"""Pins for the adaptive group-size oracle (§3.3, reading R6).

Paper parity is UNPINNED (no worked example in the paper; its inequality is ambiguous).  The
pins are SPEC.md's [DERIVED] fixtures and its invariants."""
import numpy as np
import pytest

from oracle import fq_oracle as O
from synth import gaussian_bits, gaussian_with_outliers_bits


def W_of(bits):
    return O.decode_bits(bits, "bf16")


def test_ladders():
    assert O.adapt_ladder(4096) == [4096, 2048, 1024, 512, 256, 128, 64, 32, 16]
    assert O.adapt_ladder(12288) == [12288, 6144, 3072, 1536, 768, 384, 192, 96, 48]
    assert O.adapt_ladder(128, 64) == [128, 64]
    assert O.adapt_ladder(96) == [96, 48]


def test_spec_fixture_gaussian_stays_per_column():
    # Gaussian 128x8 (K=128 rows, N=8 columns), alpha=0.5 -> per-column
    W = W_of(gaussian_bits((8, 128), 1.0, 7))
    assert O.adapt_group_size(W, 500, 16) == 128


def test_spec_fixture_outlier_goes_to_min_group():
    # N(0, 0.01) with one planted 1.0 outlier -> halves down to min_group 16
    W = W_of(gaussian_with_outliers_bits((8, 128), 0.01, 8, 1, 1.0))
    rep = O.adapt_report(W, 500, 16)
    assert rep.group == 16
    assert all(lv.accepted for lv in rep.levels)


def test_spec_fixture_zero_matrix():
    assert O.adapt_group_size(np.zeros((8, 128)), 500, 16) == 128


def test_invariants_monotone_in_alpha_and_in_ladder():
    for seed in range(6):
        W = W_of(gaussian_with_outliers_bits((16, 512), 0.02, 100 + seed, 1 + seed % 3, 0.05 + 0.05 * seed))
        prev = None
        for a in (50, 200, 400, 600, 800, 950):
            g = O.adapt_group_size(W, a, 16)
            assert g in O.adapt_ladder(512, 16)
            if prev is not None:
                assert g <= prev   # larger alpha -> finer (or equal) groups
            prev = g
            assert g == O.adapt_group_size(W, a, 16)  # determinism


def test_outlier_sensitivity():
    # an outlier >= 10x column absmax strictly decreases g (or hits the floor), alpha>=0.2
    W = W_of(gaussian_bits((8, 256), 0.02, 55))
    for a in (200, 500, 800):
        g0 = O.adapt_group_size(W, a, 16)
        W2 = W.copy()
        W2[3, 77] = 10 * np.abs(W).max()
        g1 = O.adapt_group_size(W2, a, 16)
        assert g1 < g0 or g1 == 16


def test_scale_shrink_witness():
    # an accepted halving has a child scale < alpha * parent scale (up to bf16 rounding)
    W = W_of(gaussian_with_outliers_bits((8, 256), 0.02, 9, 1, 0.8))
    rep = O.adapt_report(W, 500, 16)
    ladder = O.adapt_ladder(256, 16)
    for lv in rep.levels:
        if lv.accepted:
            sp = O.quantize(W, 4, ladder[lv.level - 1], O.BF16).s
            sc = O.quantize(W, 4, ladder[lv.level], O.BF16).s
            par = np.repeat(sp, 2, axis=0)
            assert np.any(sc < 0.5 * par * (1 + 2.0**-7))


def test_decide_and_tp_or_of_column_shards():
    W = W_of(gaussian_with_outliers_bits((32, 1024), 0.02, 10, 2, 0.3))
    flags = O.adapt_flags(W, 500, 16)
    assert O.adapt_decide(flags, 1024, 16) == O.adapt_group_size(W, 500, 16)
    # column shards (rows of our [N, K] storage): OR of shard flags == unsharded flags
    for t in (2, 4, 8):
        shard_flags = [O.adapt_flags(W[i * 32 // t:(i + 1) * 32 // t], 500, 16) for i in range(t)]
        ored = [any(f[L] for f in shard_flags) for L in range(len(flags))]
        assert ored == flags


def test_alpha_range_rejected():
    with pytest.raises(ValueError):
        O.adapt_report(np.zeros((2, 64)), 0, 16)
    with pytest.raises(ValueError):
        O.adapt_report(np.zeros((2, 64)), 1001, 16)


def _hand_column(quarters):
    col = []
    for a in quarters:
        col += [a] + [(-1) ** (i + 1) * a / 2 for i in range(1, 16)]
    return np.array([col], dtype=np.float64)


@pytest.mark.parametrize("name", ["prefix", "pairing"])
def test_hand_fixtures_levels(golden, name):
    """tests/golden/adapt_hand.txt (hand-derived, PAPER.md:147-149 + R6/R7): per-level flags, min
    ratios and counts, and the accepted-prefix decision.  Fixture 'prefix' fails a deepest-fired-level
    rule; fixture 'pairing' fails a child-to-parent pairing other than j // 2."""
    g = golden("adapt_hand.txt")
    W = _hand_column([float(x) for x in g[f"{name}_quarters"]])
    assert np.max(np.abs(W)) == 1.0
    rep = O.adapt_report(W, 500, 16)
    assert [lv.group for lv in rep.levels] == [32, 16]
    assert [int(lv.flag) for lv in rep.levels] == [int(x) for x in g[f"{name}_flags"]]
    assert [lv.min_ratio for lv in rep.levels] == [float(x) for x in g[f"{name}_min_ratio"]]
    assert [lv.count_below for lv in rep.levels] == [int(x) for x in g[f"{name}_count_below"]]
    assert rep.group == int(g[f"{name}_group"][0])
    assert O.adapt_group_size(W, 500, 16) == rep.group
    assert O.adapt_decide(O.adapt_flags(W, 500, 16), 64, 16) == rep.group


def test_hand_fixture_pairing_in_multicolumn_matrix(golden):
    """The same two columns side by side: flags OR over columns (L1 from 'pairing', L2 from 'prefix'),
    so L1 and L2 both fire -> 16.  Either column alone stops earlier."""
    g = golden("adapt_hand.txt")
    W = np.vstack([_hand_column([float(x) for x in g["prefix_quarters"]]),
                   _hand_column([float(x) for x in g["pairing_quarters"]])])
    assert O.adapt_flags(W, 500, 16) == [True, True]
    assert O.adapt_group_size(W, 500, 16) == 16
