"""GPU parity at the benchmarked sizes, in the launch configurations bench.py times.

* configs[2] (OPT-175B prefill, tcgen05 A6): M = 2048 .. 8192 and ragged raster groups (tiles of 256
  tokens are rastered in groups of 8 token tiles: M = 2304 leaves a last group of one tile, M = 2064
  a last tile of 16 tokens), sampled outputs covering every token tile and so every raster group.
* configs[3] (MoE batch: 64 experts [16384 x 4096], int4 adaptive, outliers planted in e % 4 == 0 ->
  g in {16, 4096}): uniform M_e = 16 / 64 / 256 and Zipf routing, sampled columns of every expert.
* A6 with 256-token tiles and 16-element groups in one GEMM.

The oracle computes the sampled outputs one by one from the same bytes (codes/scales of the sampled
columns are compared bit-exact first).  Tolerance: north_star 2e-3 of sum |a w|."""
import numpy as np
import pytest
import torch

from oracle import fq_oracle as O
from synth import gaussian_torch, zipf_routing, uniform_routing
from helpers import torch_to_f64

pytestmark = pytest.mark.gpu
TOL = 2e-3
FC1, FC2 = (12288, 49152), (49152, 12288)


@pytest.fixture(scope="module")
def fq():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2308_09723_b200 import fq as m
    return m


def to_f64(t):
    return t.float().cpu().double().numpy()


def check_sampled(fq, qw, W, A, C, rows, cols, bits, group):
    idx = torch.from_numpy(np.asarray(cols)).cuda()
    r = O.quantize(to_f64(W[idx]), bits, group, O.BF16)
    assert np.array_equal(qw.codes[idx].cpu().numpy(), O.pack_codes(r.q, bits)), "codes"
    assert np.array_equal(qw.scales[:, idx].cpu().view(torch.int16).numpy().view(np.uint16), r.s_bits), "scales"
    Ar = to_f64(A[torch.from_numpy(np.asarray(rows)).cuda()])
    Cr, D = O.gemm(Ar, r.q, r.s, group)
    err = O.rel_err(torch_to_f64(C)[np.ix_(rows, cols)], Cr, D)
    assert err <= TOL, err


def tile_rows(M, bn=256, per_tile=3, seed=0):
    """Rows from every token tile (first, last and one random row of each): every raster group
    and the ragged last tile are sampled."""
    rng = np.random.default_rng(seed)
    rows = []
    for t0 in range(0, M, bn):
        t1 = min(M, t0 + bn)
        rows += [t0, t1 - 1] + list(rng.integers(t0, t1, size=max(0, per_tile - 2)))
    return np.unique(np.array(rows))


@pytest.mark.parametrize("shape", [FC1, FC2])
@pytest.mark.parametrize("M,bits", [(4096, 4), (8192, 4), (8192, 8), (2304, 4), (2064, 8)])
def test_opt175b_prefill_large_m(fq, shape, M, bits):
    K, N = shape
    W = gaussian_torch((N, K), 0.02, 5000 + K)
    A = gaussian_torch((M, K), 1.0, 6000 + M)
    qw = fq.quantize(W, bits, 128)
    C = fq.gemm(A, qw)
    torch.cuda.synchronize()
    rng = np.random.default_rng(M + K)
    # columns from the first, the last and random 128-row weight tiles
    cols = np.unique(np.concatenate([[0, 127, N - 1], rng.choice(N, 45, replace=False)]))
    check_sampled(fq, qw, W, A, C, tile_rows(M), cols, bits, 128)
    del W, A, C, qw
    torch.cuda.empty_cache()


@pytest.mark.parametrize("M,K,N,group", [(256, 4096, 1024, 16), (512, 2048, 640, 16), (256, 12288, 512, 48)])
def test_a6_full_token_tiles_small_groups(fq, M, K, N, group):
    """256-token A6 tiles with groups much smaller than the 64-k stage (several scale rows per
    stage, up to 4 group boundaries per thread), full outputs."""
    W = gaussian_torch((N, K), 0.02, 700 + group)
    A = gaussian_torch((M, K), 1.0, 800 + M)
    qw = fq.quantize(W, 4, group)
    C = fq.gemm(A, qw, out_dtype=torch.float32)
    torch.cuda.synchronize()
    r = O.quantize(to_f64(W), 4, group, O.BF16)
    Cr, D = O.gemm(to_f64(A), r.q, r.s, group)
    assert O.rel_err(torch_to_f64(C), Cr, D) <= TOL


# ---------------------------------------------------------------------------------------- MoE
E_MOE, K_MOE, N_MOE = 64, 4096, 16384


@pytest.fixture(scope="module")
def moe_experts(fq):
    """configs[3] experts exactly as bench.py builds them (seeded on the device), quantized with
    the adaptive group size; returns (quantized experts, weights of 4 columns per expert)."""
    experts, Wcols, cols = [], [], []
    rng = np.random.default_rng(31)
    for e in range(E_MOE):
        W = gaussian_torch((N_MOE, K_MOE), 0.01 if e % 4 == 0 else 0.02, 7000 + e)
        if e % 4 == 0:
            W[e % N_MOE, (37 * e) % K_MOE] = 1.0
        q = fq.quantize(W, 4, None, alpha_milli=500, min_group=16)
        # adaptive decision checked against the oracle on a subset (the full fp64 pass over a
        # 16384 x 4096 matrix takes seconds)
        if e in (0, 1, 4, 7):
            assert q.group == O.adapt_group_size(to_f64(W), 500, 16), e
        assert q.group == (16 if e % 4 == 0 else K_MOE), (e, q.group)
        c = np.unique(np.concatenate([[e % N_MOE], rng.choice(N_MOE, 5, replace=False)]))
        Wcols.append(to_f64(W[torch.from_numpy(c).cuda()]))
        cols.append(c)
        experts.append(q)
        del W
    torch.cuda.empty_cache()
    return experts, Wcols, cols


@pytest.mark.parametrize("routing", ["uniform16", "uniform64", "uniform256", "zipf64"])
def test_moe_configs3_batch(fq, moe_experts, routing):
    experts, Wcols, cols = moe_experts
    if routing.startswith("uniform"):
        off = uniform_routing(E_MOE, int(routing[7:]))
    else:
        off = zipf_routing(E_MOE, E_MOE * 64, seed=3000)
    T = int(off[-1])
    A = gaussian_torch((T, K_MOE), 1.0, 3000 + T)
    C = fq.gemm_grouped(A, off, experts)
    torch.cuda.synchronize()
    Ad = to_f64(A)
    Cd = torch_to_f64(C)
    for e, q in enumerate(experts):
        lo, hi = int(off[e]), int(off[e + 1])
        if hi == lo:
            continue
        c = cols[e]
        r = O.quantize(Wcols[e], 4, q.group, O.BF16)
        idx = torch.from_numpy(c).cuda()
        assert np.array_equal(q.codes[idx].cpu().numpy(), O.pack_codes(r.q, 4)), e
        assert np.array_equal(q.scales[:, idx].cpu().view(torch.int16).numpy().view(np.uint16), r.s_bits), e
        Cr, D = O.gemm(Ad[lo:hi], r.q, r.s, q.group)
        err = O.rel_err(Cd[lo:hi][:, c], Cr, D)
        assert err <= TOL, (e, hi - lo, q.group, err)
