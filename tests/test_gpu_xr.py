"""Fused row-parallel GEMM + one-shot all-reduce (§2.1 "we must issue an all
reduce after each attention and FFN block") on ONE GPU: every rank of a group runs on the same
device (xr_group_local: the peer table holds plain device addresses), each rank's decode GEMM
pushes its partial tiles to the tile owners and the last arriver reduces and broadcasts.  All
ranks' GEMMs are issued before any rank waits, as separate GPUs would run them concurrently.

Checks: every rank's output is bit-identical; it equals the rank-ordered fp32 sum of the ranks'
own partial GEMMs exactly (same kernel, same order); it matches the oracle's UNSHARDED product
within the north_star tolerance; repeated calls (self-resetting counters) are bit-identical."""
import numpy as np
import pytest
import torch

from oracle import fq_oracle as O
from synth import activations_bits, gaussian_bits
from helpers import bits_to_torch, torch_to_f64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fq():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2308_09723_b200 import fq as m
    return m


def run_group(fq, ranks, As, qws, M):
    d = qws[0].desc
    nb = fq.fq_gemm_workspace_bytes_ex(M, d, fq.make_opts("decode"))
    wss = [torch.zeros(max(nb, 256), dtype=torch.uint8, device="cuda")
           for _ in ranks]
    for r, R in enumerate(ranks):  # every rank's GEMM first ...
        fq.fq_gemm_allreduce(As[r], M, d, qws[r].codes, qws[r].scales, fq._DT[R.out.dtype], R.peers, R.peers_dev,
                             wss[r])
    for R in ranks:                # ... then every rank's completion wait
        fq.fq_xr_wait(R.peers, M, d)
    torch.cuda.synchronize()
    return [R.out.clone() for R in ranks]


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("M,K,N,bits,group", [(1, 8192, 1024, 4, 128), (5, 4096, 1000, 4, 64),
                                              (16, 16384, 768, 4, 128), (24, 8192, 512, 4, 128),
                                              (3, 4096, 512, 8, 128)])
def test_fused_allreduce_parity(fq, world, M, K, N, bits, group):
    Wb = gaussian_bits((N, K), 0.02, 4000 + K + N)
    Ab = activations_bits(M, K, 4100 + M)
    W = bits_to_torch(Wb, "bf16")
    A = bits_to_torch(Ab, "bf16")
    Ks = K // world
    qws = [fq.quantize(W[:, r * Ks:(r + 1) * Ks].contiguous(), bits, group) for r in range(world)]
    As = [A[:, r * Ks:(r + 1) * Ks].contiguous() for r in range(world)]
    for dt in (torch.float32, torch.bfloat16):
        ranks = fq.xr_group_local(world, M, qws[0].desc, dt)
        outs = run_group(fq, ranks, As, qws, M)
        for o in outs[1:]:
            assert torch.equal(o, outs[0])
        again = run_group(fq, ranks, As, qws, M)
        assert torch.equal(again[0], outs[0])
        if dt == torch.float32:
            ref = None
            for r in range(world):
                p = fq.gemm(As[r], qws[r], out_dtype=torch.float32, opts=fq.make_opts("decode"))
                ref = p if ref is None else ref + p
            torch.cuda.synchronize()
            assert torch.equal(outs[0], ref)
    # the unsharded oracle product
    r_full = O.quantize(O.decode_bits(Wb, "bf16"), bits, group, O.BF16)
    Cr, D = O.gemm(O.decode_bits(Ab, "bf16"), r_full.q, r_full.s, group)
    assert O.rel_err(torch_to_f64(outs[0]), Cr, D) <= 2e-3


def test_fused_allreduce_rejects_prefill_and_bad_tables(fq):
    d = fq.make_wdesc(4096, 512, 4, 128, fq.FQ_BF16)
    assert fq.fq_xr_recv_bytes(64, d, 2) == 0          # M beyond the decode kernel
    assert fq.fq_xr_recv_bytes(16, d, 9) == 0          # world > 8
    pt = fq.fq_xr_peers()
    pt.world, pt.rank = 2, 2                            # rank out of range
    dummy = torch.zeros(16, dtype=torch.uint8, device="cuda")
    A = torch.zeros((4, 4096), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(fq.FQError) as e:
        fq.fq_gemm_allreduce(A, 4, d, dummy, dummy, fq.FQ_BF16, pt, dummy, None)
    assert e.value.status == fq.FQ_ERR_INVALID_ARG
