"""GPU parity of tensor-parallel sharding (A8) on one device: every shard of t = 2/4/8 is
quantized and multiplied by the libfq kernels; column shards' codes/scales must be the bit-exact
slices of the unsharded ones, and the sum of the row shards' partials must match the unsharded
fp64 oracle within 2e-3.  The NCCL all-reduce itself runs in bench.py under
torchrun; here a world-size-1 NCCL group drives TPOptLayer end to end."""
import os
import socket

import numpy as np
import pytest
import torch

from oracle import fq_oracle as O
from synth import activations_bits, gaussian_bits
from helpers import bits_to_torch, torch_to_f64

pytestmark = pytest.mark.gpu
TOL = 2e-3


@pytest.fixture(scope="module")
def fq():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2308_09723_b200 import fq as m
    return m


@pytest.mark.parametrize("t", [2, 4, 8])
@pytest.mark.parametrize("M", [1, 16, 64])
def test_column_and_row_shards(fq, t, M):
    from paper_2308_09723_b200.tp import shard_bounds, check_row_group
    K, N, bits, g = 2048, 1024, 4, 128
    Wb = gaussian_bits((N, K), 0.02, 77)
    Ab = activations_bits(M, K, 78)
    W = bits_to_torch(Wb, "bf16")
    A = bits_to_torch(Ab, "bf16")
    full = fq.quantize(W, bits, g)
    # column shards: slices of the unsharded codes/scales, bit-exact
    for r in range(t):
        lo, hi = shard_bounds(N, t, r)
        sh = fq.quantize(W[lo:hi].contiguous(), bits, g)
        assert torch.equal(sh.codes, full.codes[lo:hi])
        assert torch.equal(sh.scales, full.scales[:, lo:hi])
    # row shards: partials over K slices, summed
    check_row_group(K, t, g)
    acc = torch.zeros(M, N, dtype=torch.float32, device="cuda")
    for r in range(t):
        lo, hi = shard_bounds(K, t, r, 32)
        sh = fq.quantize(W[:, lo:hi].contiguous(), bits, g)
        assert torch.equal(sh.codes, full.codes[:, lo * bits // 8:hi * bits // 8])
        acc += fq.gemm(A[:, lo:hi].contiguous(), sh, out_dtype=torch.float32)
    r_ = O.quantize(O.decode_bits(Wb, "bf16"), bits, g, O.BF16)
    Cr, D = O.gemm(O.decode_bits(Ab, "bf16"), r_.q, r_.s, g)
    assert O.rel_err(torch_to_f64(acc), Cr, D) <= TOL


def test_opt_layer_world1_nccl(fq):
    """TPOptLayer on a 1-rank NCCL group (the t=1 configuration of configs[4], scaled down)."""
    import torch.distributed as dist
    from paper_2308_09723_b200.tp import ShardSpec, TPLinearFQ, TPOptLayer
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1)
    h, M = 512, 4
    mats = {}
    seeds = dict(qkv=11, out=12, fc1=13, fc2=14)
    for name, (n, k) in dict(qkv=(3 * h, h), out=(h, h), fc1=(4 * h, h), fc2=(h, 4 * h)).items():
        mats[name] = bits_to_torch(gaussian_bits((n, k), 0.02, seeds[name]), "bf16")
    kinds = dict(qkv="col", out="row", fc1="col", fc2="row")
    lin = {k: TPLinearFQ(v, ShardSpec(kinds[k], v.shape[1], v.shape[0], 1, 0)) for k, v in mats.items()}
    layer = TPOptLayer(lin["qkv"], lin["out"], lin["fc1"], lin["fc2"])
    x = bits_to_torch(activations_bits(M, h, 5), "bf16")
    y = layer.forward(x)
    torch.cuda.synchronize()
    # reference: the same chain through the oracle (bf16 rounding between layers as in the layer)
    def deq(t):
        return O.decode_bits(t.cpu().view(torch.int16).numpy().view(np.uint16), "bf16")
    def ref_gemm(xx, w):
        r = O.quantize(deq(w), 4, 128, O.BF16)
        return O.gemm(xx, r.q, r.s, 128)
    q, _ = ref_gemm(deq(x), mats["qkv"])
    q = O.round_to_format(q, O.BF16)[:, :h]
    y1, _ = ref_gemm(q, mats["out"])
    y1 = O.round_to_format(y1, O.BF16)
    f, _ = ref_gemm(y1, mats["fc1"])
    f = O.round_to_format(f, O.BF16)
    yr, D = ref_gemm(f, mats["fc2"])
    # bf16 roundings of intermediates differ between the two chains: compare at a looser bound
    assert O.rel_err(torch_to_f64(y), yr, D) <= 1e-2
    dist.destroy_process_group()
