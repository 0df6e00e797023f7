"""GPU parity of the int8-activation x int4-weight path with integer group scales (
PAPER.md:397-399 §5; readings R15-R18) against the oracle on the same seeded bytes.

* fq_quantize_intscale: codes, integer group scales z and column scales sigma bit-exact;
* fq_quantize_acts_i8: int8 codes and per-token scales bit-exact;
* fq_gemm_i8 (tcgen05 kind::i8): the oracle's integer accumulation is exact, so the GPU output must
  equal C_ref = acc * s_a * sigma up to fp32 rounding (3 roundings of 2^-24) plus the output
  rounding (bf16: 2^-9 relative); the north_star metric (2e-3 of sum |a w|) is checked as well.
Shapes cover every kernel variant (token tiles of <= 32 / 128 / 256), ragged token / weight tiles,
split-K, groups from 32 to K, and OPT-175B FC1 / FC2 at full size on sampled outputs."""
import numpy as np
import pytest
import torch

from oracle import fq_oracle as O
from synth import activations_bits, gaussian_bits, gaussian_torch, gaussian_with_outliers_bits, \
    wide_range_activations_bits
from helpers import bits_to_torch, torch_to_f64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fq():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2308_09723_b200 import fq as m
    return m


def check_weights(qw, r, cols=None):
    c = slice(None) if cols is None else torch.from_numpy(np.asarray(cols)).cuda()
    assert np.array_equal(qw.codes[c].cpu().numpy(), O.pack_codes(r.q, 4)), "codes"
    assert np.array_equal(qw.zscales[:, c].cpu().numpy(), r.z), "integer scales"
    assert np.array_equal(qw.colscale[c].cpu().numpy(), r.sigma.astype(np.float32)), "column scales"


def unperm(a_q):
    """fq_quantize_acts_i8's k-interleaved words (fq.h) back to row-major k order."""
    a = a_q.cpu().numpy()
    M, K = a.shape
    return a.reshape(M, K // 8, 2, 4).transpose(0, 1, 3, 2).reshape(M, K)


def check_out(C, Cr, D, cdt):
    Cg = torch_to_f64(C)
    bound = (2.0 ** -8 if cdt != torch.float32 else 2.0 ** -21) * np.abs(Cr)
    bad = np.abs(Cg - Cr) > bound + 1e-30
    assert not bad.any(), (np.argwhere(bad)[:5], Cg[bad][:5], Cr[bad][:5])
    assert O.rel_err(Cg, Cr, D) <= 2e-3


@pytest.mark.parametrize("wdt", ["bf16", "fp16", "fp32"])
@pytest.mark.parametrize("K,N,group", [(256, 64, 32), (1024, 272, 64), (4096, 128, 128), (2048, 96, 2048)])
def test_quantize_intscale_bit_exact(fq, wdt, K, N, group):
    Wb = gaussian_with_outliers_bits((N, K), 0.02, 100 + K + N, 3, 0.6, dtype=wdt)
    W = bits_to_torch(Wb, wdt)
    qw = fq.quantize_intscale(W, group)
    torch.cuda.synchronize()
    r = O.quantize_intscale(O.decode_bits(Wb, wdt), 4, group)
    check_weights(qw, r)


def test_quantize_intscale_nonfinite_and_zero_columns(fq):
    Wb = gaussian_bits((32, 512), 0.02, 3)
    W = bits_to_torch(Wb, "bf16")
    W[4, 9] = float("inf")
    W[7, 100] = float("nan")
    W[11] = 0
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    qw = fq.quantize_intscale(W, 64, status=st)
    torch.cuda.synchronize()
    Wd = torch_to_f64(W.float())
    r = O.quantize_intscale(Wd, 4, 64)
    assert r.status == 1 and int(st.item()) & 1
    check_weights(qw, r)


@pytest.mark.parametrize("adt", ["bf16", "fp16", "fp32"])
@pytest.mark.parametrize("M,K", [(1, 128), (7, 4096), (64, 12288), (3, 1000), (65, 256), (16, 49152)])
def test_quantize_acts_bit_exact(fq, adt, M, K):
    Ab = activations_bits(M, K, 40 + M, dtype=adt)
    A = bits_to_torch(Ab, adt)
    a_q, sa, rs = fq.quantize_acts_i8(A)
    torch.cuda.synchronize()
    r = O.quantize_acts_i8(O.decode_bits(Ab, adt))
    assert np.array_equal(unperm(a_q), r.a_q)
    assert np.array_equal(sa.cpu().numpy(), r.s_a.astype(np.float32))
    assert np.array_equal(rs.cpu().numpy(), r.rowsum)


def test_quantize_acts_wide_range_and_edges(fq):
    Ab = wide_range_activations_bits(12, 1024, 8)
    A = bits_to_torch(Ab, "bf16")
    A[5, 17] = float("nan")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    a_q, sa, rs = fq.quantize_acts_i8(A, status=st)
    torch.cuda.synchronize()
    r = O.quantize_acts_i8(torch_to_f64(A.float()))
    assert r.status == 1 and int(st.item()) & 1
    assert np.array_equal(unperm(a_q), r.a_q)
    assert np.array_equal(sa.cpu().numpy(), r.s_a.astype(np.float32))
    assert np.array_equal(rs.cpu().numpy(), r.rowsum)


CASES = [
    # (M, K, N, group): token-tile variants 32 / 128 / 256, ragged tiles, split-K (few tiles, long K)
    (1, 256, 128, 32), (5, 1024, 144, 64), (3, 768, 128, 384), (16, 4096, 256, 128), (17, 512, 400, 32), (32, 8192, 128, 128),
    (33, 1024, 272, 256), (64, 2048, 384, 64), (100, 4096, 128, 4096), (128, 1024, 1024, 128),
    (129, 512, 256, 32), (200, 6144, 512, 128), (256, 2048, 640, 64), (300, 1024, 384, 128),
    (640, 4096, 256, 128), (1000, 512, 1152, 512),
    # decode sizes on the mma.sync m16n8k32 u8 x s8 kernel: two token tiles, ragged column tile,
    # 32- / 64-k groups (4 / 2 staged z rows), split-K with long K, groups of 3 stages
    (9, 2048, 784, 32), (12, 12288, 1024, 64), (2, 4096, 4096, 256), (8, 3072, 400, 384), (13, 1024, 16, 128),
    # two-chunk stages: K % 256 == 128 (the last stage's second chunk is past K), groups straddling stages
    (4, 1152, 272, 128), (11, 1920, 400, 384), (1, 2432, 512, 32),
]


@pytest.mark.parametrize("cdt", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("M,K,N,group", CASES)
def test_gemm_i8_parity(fq, M, K, N, group, cdt):
    Wb = gaussian_with_outliers_bits((N, K), 0.02, 7 * K + N, 2, 0.3)
    Ab = activations_bits(M, K, 3 * M + K)
    W = bits_to_torch(Wb, "bf16")
    A = bits_to_torch(Ab, "bf16")
    qw = fq.quantize_intscale(W, group)
    C = fq.gemm_i8(A, qw, out_dtype=cdt)
    torch.cuda.synchronize()
    r = O.quantize_intscale(O.decode_bits(Wb, "bf16"), 4, group)
    a = O.quantize_acts_i8(O.decode_bits(Ab, "bf16"))
    check_weights(qw, r)
    Cr, D, _ = O.gemm_i8(a.a_q, a.s_a, r.q, r.z, r.sigma, group)
    check_out(C, Cr, D, cdt)


def test_gemm_i8_repeat_bit_identical_and_empty(fq):
    W = gaussian_torch((512, 8192), 0.02, 1)
    A = gaussian_torch((16, 8192), 1.0, 2)
    qw = fq.quantize_intscale(W, 128)
    C1 = fq.gemm_i8(A, qw)
    C2 = fq.gemm_i8(A, qw)
    torch.cuda.synchronize()
    assert torch.equal(C1, C2)
    E = fq.gemm_i8(torch.empty((0, 8192), dtype=torch.bfloat16, device="cuda"), qw)
    assert E.shape == (0, 512)


@pytest.mark.parametrize("shape", [(12288, 49152), (49152, 12288)])
@pytest.mark.parametrize("M", [1, 16, 64, 2048])
def test_gemm_i8_opt175b_sampled(fq, shape, M):
    K, N = shape
    W = gaussian_torch((N, K), 0.02, 900 + K)
    A = gaussian_torch((M, K), 1.0, 901 + M)
    qw = fq.quantize_intscale(W, 128)
    C = fq.gemm_i8(A, qw)
    torch.cuda.synchronize()
    rng = np.random.default_rng(M)
    cols = np.unique(np.concatenate([[0, 127, N - 1], rng.choice(N, 40, replace=False)]))
    rows = np.unique(np.concatenate([[0, M - 1], rng.integers(0, M, size=min(M, 30))]))
    idx = torch.from_numpy(cols).cuda()
    r = O.quantize_intscale(torch_to_f64(W[idx].float()), 4, 128)
    check_weights(qw, r, cols)
    a = O.quantize_acts_i8(torch_to_f64(A.float()))
    Cr, D, _ = O.gemm_i8(a.a_q[rows], a.s_a[rows], r.q, r.z, r.sigma, 128)
    check_out(C[torch.from_numpy(rows).cuda()][:, idx], Cr, D, torch.bfloat16)
    del W, A, C, qw
    torch.cuda.empty_cache()
