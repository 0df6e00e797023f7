"""GPU parity of the int3 / int2 weights (the paper's int3 rows PAPER.md:332-346 and
2-bit weights, for which the paper ships no kernel; layout reading R19 = SPEC's bit stream)
against the oracle: codes (bit stream) and scales bit-exact, GEMM outputs within the north_star
tolerance 2e-3 of sum |a w|, on every decode-kernel class (1 / 2 / 4 token tiles, group-per-stage
and per-element-scale paths), ragged N tails, both activation dtypes, and OPT-175B FC1 / FC2 at full
size on sampled outputs.  Includes the paper's mixed configuration: attention int3 (64) with
everything else int4 (64), tab:optiml-mt."""
import numpy as np
import pytest
import torch

from oracle import fq_oracle as O
from synth import activations_bits, gaussian_bits, gaussian_torch, gaussian_with_outliers_bits
from helpers import bits_to_torch, torch_to_f64

pytestmark = pytest.mark.gpu
TOL = 2e-3


@pytest.fixture(scope="module")
def fq():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2308_09723_b200 import fq as m
    return m


def check_quant(qw, Wd, bits, group, fmt=O.BF16):
    r = O.quantize(Wd, bits, group, fmt)
    assert np.array_equal(qw.codes.cpu().numpy(), O.pack_codes(r.q, bits)), "codes"
    assert np.array_equal(qw.scales.cpu().view(torch.int16).numpy().view(np.uint16), r.s_bits), "scales"
    return r


@pytest.mark.parametrize("bits", [3, 2])
@pytest.mark.parametrize("wdt", ["bf16", "fp16", "fp32"])
@pytest.mark.parametrize("K,N,group", [(128, 64, 16), (384, 264, 64), (4096, 128, 128), (1024, 72, 1024)])
def test_quantize_lowbit_bit_exact(fq, bits, wdt, K, N, group):
    Wb = gaussian_with_outliers_bits((N, K), 0.02, 300 + K + bits, 2, 0.4, dtype=wdt)
    W = bits_to_torch(Wb, wdt)
    qw = fq.quantize(W, bits, group)
    torch.cuda.synchronize()
    check_quant(qw, O.decode_bits(Wb, wdt), bits, group)


CASES = [
    # (M, K, N, group): one / two / four 8-token MMA tiles, group per stage (g % 128) and
    # per-element scales (g = 32 / 64), ragged N tails, split-K
    (1, 128, 256, 128), (1, 4096, 264, 64), (3, 1024, 512, 32), (8, 2048, 520, 128), (9, 1024, 256, 64),
    (16, 8192, 256, 256), (17, 2048, 512, 128), (32, 4096, 264, 4096),
]


@pytest.mark.parametrize("bits", [3, 2])
@pytest.mark.parametrize("adt", ["bf16", "fp16"])
@pytest.mark.parametrize("M,K,N,group", CASES)
def test_gemm_lowbit_parity(fq, bits, adt, M, K, N, group):
    Wb = gaussian_bits((N, K), 0.02, 11 * K + N + bits)
    Ab = activations_bits(M, K, 5 * M + K, adt)
    W = bits_to_torch(Wb, "bf16")
    A = bits_to_torch(Ab, adt)
    sdt = {"bf16": torch.bfloat16, "fp16": torch.float16}[adt]
    qw = fq.quantize(W, bits, group, scale_dtype=sdt)
    C = fq.gemm(A, qw)
    Cf = fq.gemm(A, qw, out_dtype=torch.float32)
    torch.cuda.synchronize()
    r = check_quant(qw, O.decode_bits(Wb, "bf16"), bits, group, O.FORMATS[adt])
    Cr, D = O.gemm(O.decode_bits(Ab, adt), r.q, r.s, group)
    assert O.rel_err(torch_to_f64(C), Cr, D) <= TOL
    assert O.rel_err(torch_to_f64(Cf), Cr, D) <= TOL


def test_lowbit_unsupported_paths(fq):
    W = gaussian_torch((256, 1024), 0.02, 1)
    q3 = fq.quantize(W, 3, 64)
    A = gaussian_torch((17, 1024), 1.0, 2)  # 17 tokens on the per-element-scale path: > 16
    with pytest.raises(fq.FQError) as e:
        fq.gemm(A, q3)
    assert e.value.status == fq.FQ_ERR_UNSUPPORTED
    with pytest.raises(fq.FQError) as e:
        fq.gemm(gaussian_torch((64, 1024), 1.0, 3), fq.quantize(W, 2, 128))
    assert e.value.status == fq.FQ_ERR_UNSUPPORTED


@pytest.mark.parametrize("bits", [3, 2])
@pytest.mark.parametrize("shape", [(12288, 49152), (49152, 12288)])
@pytest.mark.parametrize("M", [1, 16])
def test_lowbit_opt175b_sampled(fq, bits, shape, M):
    K, N = shape
    W = gaussian_torch((N, K), 0.02, 1700 + K)
    A = gaussian_torch((M, K), 1.0, 1701 + M)
    qw = fq.quantize(W, bits, 128)
    C = fq.gemm(A, qw)
    torch.cuda.synchronize()
    rng = np.random.default_rng(M + bits)
    cols = np.unique(np.concatenate([[0, 255, N - 1], rng.choice(N, 40, replace=False)]))
    idx = torch.from_numpy(cols).cuda()
    r = O.quantize(torch_to_f64(W[idx].float()), bits, 128, O.BF16)
    assert np.array_equal(qw.codes[idx].cpu().numpy(), O.pack_codes(r.q, bits))
    assert np.array_equal(qw.scales[:, idx].cpu().view(torch.int16).numpy().view(np.uint16), r.s_bits)
    Cr, D = O.gemm(torch_to_f64(A.float()), r.q, r.s, 128)
    assert O.rel_err(torch_to_f64(C[:, idx]), Cr, D) <= TOL
    del W, A, C, qw
    torch.cuda.empty_cache()


def test_mixed_int3_attention_int4_others(fq):
    """tab:optiml-mt row "int3 (64) | int4 (64)": an OPT-30B-shaped layer slice with the attention
    projections at int3 g64 and the FFN at int4 g64 (a per-matrix bits choice), decode M = 4."""
    h = 7168
    M = 4
    x = bits_to_torch(activations_bits(M, h, 77), "bf16")
    mats = {"qkv": (3 * h, h, 3), "out": (h, h, 3), "fc1": (4 * h // 8, h, 4), "fc2": (h // 8, 4 * h, 4)}
    for i, (name, (n, k, bits)) in enumerate(mats.items()):
        Wb = gaussian_bits((n, k), 0.02, 900 + i)
        W = bits_to_torch(Wb, "bf16")
        qw = fq.quantize(W, bits, 64)
        A = x if k == h else bits_to_torch(activations_bits(M, k, 78), "bf16")
        C = fq.gemm(A, qw)
        torch.cuda.synchronize()
        r = check_quant(qw, O.decode_bits(Wb, "bf16"), bits, 64)
        Cr, D = O.gemm(torch_to_f64(A.float()), r.q, r.s, 64)
        assert O.rel_err(torch_to_f64(C), Cr, D) <= TOL, name
