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


# ------------------------------------------------------------------ device expert offsets (§8(b))
def _dev_case(fq, counts, K, N, bits, max_tokens, seed, T_extra=5):
    E = len(counts)
    off = np.zeros(E + 1, dtype=np.int64)
    off[1:] = np.cumsum(counts)
    qws, ref = build_experts(fq, E, K, N, bits, seed0=seed)
    T = int(off[-1]) + T_extra  # capacity rows beyond the routed tokens: never written
    Ab = activations_bits(T, K, seed + 1)
    A = bits_to_torch(Ab, "bf16")
    # the offsets are produced on the device by the previous op on the stream (a router's cumsum)
    cnt = torch.tensor(counts, dtype=torch.int64, device="cuda")
    off_dev = torch.zeros(E + 1, dtype=torch.int64, device="cuda")
    off_dev[1:] = torch.cumsum(cnt, 0)
    # fp32 output for the tolerance check (a dominant same-sign term makes bf16 output rounding alone
    # exceed 2e-3 of sum |a w|, SURVEY §8(c) error budget); the bf16 output must be its rounding
    C = torch.full((T, N), 7.0, dtype=torch.float32, device="cuda")
    Cb = torch.full((T, N), 7.0, dtype=torch.bfloat16, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    fq.gemm_grouped_dev(A, off_dev, qws, max_tokens, out=C, status=st)
    fq.gemm_grouped_dev(A, off_dev, qws, max_tokens, out=Cb)
    torch.cuda.synchronize()
    assert torch.equal(Cb, C.to(torch.bfloat16))
    return off, qws, ref, Ab, C, st


@pytest.mark.parametrize("bits", [4, 8])
@pytest.mark.parametrize("counts,max_tokens", [
    ([0, 1, 3, 8, 2, 16, 5, 0], 16),                 # decode kernel (A4), empty experts
    ([0, 20, 7, 32, 1, 0, 30, 12], 32),               # int4: nibble decode path up to 32; int8: tcgen05
    ([0, 40, 130, 3, 64, 0, 200, 17], 256),           # tcgen05 (A6) with tiles beyond some experts
])
def test_moe_device_offsets(fq, bits, counts, max_tokens):
    K, N = 512, 384
    off, qws, ref, Ab, C, st = _dev_case(fq, counts, K, N, bits, max_tokens, 7000 + max_tokens)
    assert int(st.item()) == 0
    R = int(off[-1])
    Cr, D = O.gemm_grouped(O.decode_bits(Ab[:R], "bf16"), off, ref)
    assert O.rel_err(torch_to_f64(C[:R]), Cr, D) <= TOL
    assert torch.all(C[R:] == 7.0)  # capacity rows past offsets[E] untouched


def test_moe_device_offsets_over_bound(fq):
    """An expert with more tokens than the bound: its first max_tokens rows are computed, the rest
    untouched, status bit 2 set; the other experts are unaffected."""
    K, N = 256, 256
    counts = [3, 12, 5]
    off, qws, ref, Ab, C, st = _dev_case(fq, counts, K, N, 4, 8, 7100)
    assert int(st.item()) & 4
    R = int(off[-1])
    Cr, D = O.gemm_grouped(O.decode_bits(Ab[:R], "bf16"), off, ref)
    ok = np.ones(R, dtype=bool)
    ok[3 + 8:3 + 12] = False  # expert 1 rows beyond the bound
    Cg = torch_to_f64(C[:R])
    assert O.rel_err(Cg[ok], Cr[ok], D[ok]) <= TOL
    assert torch.all(C[3 + 8:3 + 12] == 7.0)
