"""Back-to-back GEMMs with no host synchronisation: each GEMM's output is the next one's input, one
matrix is quantized in the middle of the chain, and the split-K workspace is shared by every call.

The decode kernel and its activation pre-conversion are launched with programmatic dependent launch
and trigger their dependents at CTA start (the next GEMM pre-streams its weights while the previous
one finishes); this checks that every read of a previous kernel's output and every workspace write
stays ordered behind the dependency wait.  Each link is compared with the fp64 oracle applied to the
GPU's own input of that link (so bf16 rounding of the intermediates does not compound), the
mid-chain quantization bit-exactly with the oracle, and a second run of the chain bit-for-bit with
the first.  Tolerance: BASELINE.json north_star, 2e-3 of sum|a*w|."""
import numpy as np
import pytest
import torch

from oracle import fq_oracle as O
from synth import activations_bits, gaussian_bits
from helpers import bits_to_torch, torch_to_f64

pytestmark = pytest.mark.gpu
TOL = 2e-3
K = N = 2048  # square, so outputs chain; 8 column tiles -> the decode plan splits K (shared workspace)
LINKS = 4
GROUP = 128


@pytest.fixture(scope="module")
def fq():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2308_09723_b200 import fq as m
    return m


@pytest.fixture(scope="module")
def weights():
    Wb = [gaussian_bits((N, K), 0.03, 7100 + i, "bf16") for i in range(LINKS)]
    refs = [O.quantize(O.decode_bits(w, "bf16"), 4, GROUP, O.BF16) for w in Wb]
    return Wb, refs


def run_chain(fq, Wb, M, seed):
    """Quantize links 0..2 up front, link 3 inside the chain; return inputs, outputs, last q."""
    qs = [fq.quantize(bits_to_torch(Wb[i], "bf16"), 4, GROUP) for i in range(LINKS - 1)]
    torch.cuda.synchronize()
    W3 = bits_to_torch(Wb[LINKS - 1], "bf16")
    x = bits_to_torch(activations_bits(M, K, seed, "bf16"), "bf16")
    xs, ys = [], []
    for i in range(LINKS):
        if i == LINKS - 1:
            qs.append(fq.quantize(W3, 4, GROUP))  # enqueued right behind GEMM i-1, no sync
        y = fq.gemm(x, qs[i])
        xs.append(x)
        ys.append(y)
        x = y
    torch.cuda.synchronize()
    return xs, ys, qs[-1]


@pytest.mark.parametrize("M", [1, 5, 8, 16, 24, 64])
def test_chain_links_match_oracle(fq, weights, M):
    Wb, refs = weights
    xs, ys, q3 = run_chain(fq, Wb, M, 7200 + M)
    r3 = refs[LINKS - 1]
    assert np.array_equal(q3.codes.cpu().numpy(), O.pack_codes(r3.q, 4)), "mid-chain codes"
    assert np.array_equal(q3.scales.cpu().view(torch.int16).numpy().view(np.uint16), r3.s_bits), "mid-chain scales"
    for i in range(LINKS):
        Cr, D = O.gemm(torch_to_f64(xs[i]), refs[i].q, refs[i].s, GROUP)
        err = O.rel_err(torch_to_f64(ys[i]), Cr, D)
        assert err <= TOL, f"link {i} M={M}: {err}"


@pytest.mark.parametrize("M", [1, 16])
def test_chain_is_deterministic(fq, weights, M):
    Wb, _ = weights
    _, y1, _ = run_chain(fq, Wb, M, 7300)
    _, y2, _ = run_chain(fq, Wb, M, 7300)
    for a, b in zip(y1, y2):
        assert torch.equal(a.view(torch.int16), b.view(torch.int16))
