"""GPU parity of the MoE expert batch (kernel A7): per-expert adaptive group size (§3.3,
one g per expert matrix), tokens sorted by expert, experts of every size class in one call."""
import numpy as np
import pytest
import torch

from oracle import fq_oracle as O
from synth import activations_bits, gaussian_bits, gaussian_with_outliers_bits, zipf_routing
from helpers import bits_to_torch, torch_to_f64

pytestmark = pytest.mark.gpu
TOL = 2e-3


@pytest.fixture(scope="module")
def fq():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2308_09723_b200 import fq as m
    return m


def build_experts(fq, E, K, N, bits, seed0=1000):
    """Experts with e % 4 == 0 get a planted outlier -> adaptive group = min_group."""
    Wbs, qws, ref = [], [], []
    for e in range(E):
        if e % 4 == 0:
            Wb = gaussian_with_outliers_bits((N, K), 0.01, seed0 + e, 1, 1.0)
        else:
            Wb = gaussian_bits((N, K), 0.02, seed0 + e)
        W = bits_to_torch(Wb, "bf16")
        qw = fq.quantize(W, bits, None, alpha_milli=500, min_group=16)  # adaptive
        Wd = O.decode_bits(Wb, "bf16")
        g = O.adapt_group_size(Wd, 500, 16)
        assert qw.group == g
        r = O.quantize(Wd, bits, g, O.BF16)
        assert np.array_equal(qw.codes.cpu().numpy(), O.pack_codes(r.q, bits))
        Wbs.append(Wb)
        qws.append(qw)
        ref.append((r.q, r.s, g))
    return qws, ref


@pytest.mark.parametrize("bits", [4, 8])
def test_moe_mixed_sizes(fq, bits):
    E, K, N = 10, 512, 384
    counts = [0, 1, 3, 8, 9, 16, 17, 40, 2, 5]  # empty, decode classes, and tcgen05-sized experts
    off = np.zeros(E + 1, dtype=np.int64)
    off[1:] = np.cumsum(counts)
    qws, ref = build_experts(fq, E, K, N, bits)
    Ab = activations_bits(int(off[-1]), K, 2000)
    A = bits_to_torch(Ab, "bf16")
    C = fq.gemm_grouped(A, off, qws)
    torch.cuda.synchronize()
    Cr, D = O.gemm_grouped(O.decode_bits(Ab, "bf16"), off, ref)
    assert O.rel_err(torch_to_f64(C), Cr, D) <= TOL
    # fp32 output mode
    C32 = fq.gemm_grouped(A, off, qws, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert O.rel_err(torch_to_f64(C32), Cr, D) <= TOL


def test_moe_zipf_routing_many_experts(fq):
    """64 experts (> one launch's batch capacity), Zipf-skewed routing of 64 x 4 tokens."""
    E, K, N = 64, 256, 256
    off = zipf_routing(E, 256, seed=3000)
    qws, ref = build_experts(fq, E, K, N, 4, seed0=5000)
    Ab = activations_bits(int(off[-1]), K, 2001)
    A = bits_to_torch(Ab, "bf16")
    C = fq.gemm_grouped(A, off, qws)
    torch.cuda.synchronize()
    Cr, D = O.gemm_grouped(O.decode_bits(Ab, "bf16"), off, ref)
    assert O.rel_err(torch_to_f64(C), Cr, D) <= TOL
