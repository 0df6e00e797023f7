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


def _simulate_rowshard(fq, W, t, adaptive=True, group=None, alpha=500, min_group=16):
    """Run tp.rowshard_protocol's steps for all t ranks on one GPU, with a torch max over the
    ranks' buffers standing in for the int32 MAX all-reduce (plumbing only)."""
    from paper_2308_09723_b200.tp import shard_bounds
    N, K = W.shape
    ops = fq.KERNEL_OPS
    nflags = max(0, fq.fq_adapt_levels(K, min_group) - 1)
    shards, bufs = [], []
    for r in range(t):
        lo, hi = shard_bounds(K, t, r, 32)
        Ws = W[:, lo:hi].contiguous()
        buf, flags, colmax = ops.alloc(nflags, t, N, W.device)
        ops.shard_pass(Ws, K, t, r, alpha, min_group, flags, colmax)
        shards.append(Ws)
        bufs.append((buf, flags, colmax))
    red = torch.stack([b[0] for b in bufs]).amax(dim=0)
    gs = []
    for buf, flags, colmax in bufs:
        buf.copy_(red)
        if adaptive:
            ops.cross(colmax, K, N, t, alpha, min_group, flags)
            gs.append(ops.decide(K, min_group, flags))
    g = gs[0] if adaptive else group
    assert all(x == g for x in gs), gs
    qws = [fq.quantize_rowshard(shards[r], K, t, r, 4 if group is None else 4, g, bufs[r][2]) for r in range(t)]
    return g, shards, qws, bufs


@pytest.mark.parametrize("t", [1, 2, 4, 8])
@pytest.mark.parametrize("name", ["gauss", "outlier", "step2", "step4", "step8"])
def test_rowshard_adaptive_bitexact(fq, t, name):
    """Row-parallel adaptive quantization: the group size decided from
    K-shards equals the unsharded one, every shard's codes/scales are the K-/G-slices of the
    unsharded quantization (bit-exact, including groups wider than a shard), and the sum of the
    shards' partial GEMMs matches the unsharded fp64 oracle within 2e-3."""
    from test_tp import _rowshard_matrices
    from synth import f32_to_bf16_bits
    from paper_2308_09723_b200.tp import shard_bounds
    Wd = _rowshard_matrices()[name]
    N, K = Wd.shape
    Wb = f32_to_bf16_bits(Wd.astype(np.float32))
    assert np.array_equal(O.decode_bits(Wb, "bf16"), Wd)
    W = bits_to_torch(Wb, "bf16")
    g, shards, qws, _ = _simulate_rowshard(fq, W, t)
    g_ref = O.adapt_group_size(Wd, 500, 16)
    assert g == g_ref
    ref = O.quantize(Wd, 4, g, O.BF16)
    ks = K // t
    for r, qw in enumerate(qws):
        lo, hi = shard_bounds(K, t, r, 32)
        assert qw.group == min(g, ks)
        assert np.array_equal(qw.codes.cpu().numpy(), O.pack_codes(ref.q[:, lo:hi], 4)), f"codes r={r}"
        srow = ref.s_bits[lo // g:(hi + g - 1) // g] if g <= ks else ref.s_bits[lo // g:lo // g + 1]
        assert np.array_equal(qw.scales.cpu().view(torch.int16).numpy().view(np.uint16), srow), f"scales r={r}"
    Ab = activations_bits(5, K, 91)
    A = bits_to_torch(Ab, "bf16")
    acc = torch.zeros(5, N, dtype=torch.float32, device="cuda")
    for r, qw in enumerate(qws):
        lo, hi = shard_bounds(K, t, r, 32)
        acc += fq.gemm(A[:, lo:hi].contiguous(), qw, out_dtype=torch.float32)
    Cr, D = O.gemm(O.decode_bits(Ab, "bf16"), ref.q, ref.s, g)
    assert O.rel_err(torch_to_f64(acc), Cr, D) <= TOL


@pytest.mark.parametrize("t", [2, 8])
@pytest.mark.parametrize("group", [2048, 512])
def test_rowshard_fixed_wide_group(fq, t, group):
    """Fixed groups wider than a shard (per-column g = K, and K/4 at t = 8): scales from the MAX-
    reduced shard column maxima, bit-exact with the unsharded quantization."""
    from paper_2308_09723_b200.tp import shard_bounds
    Wb = gaussian_bits((64, 2048), 0.02, 93)
    W = bits_to_torch(Wb, "bf16")
    _, shards, qws, _ = _simulate_rowshard(fq, W, t, adaptive=False, group=group)
    ref = O.quantize(O.decode_bits(Wb, "bf16"), 4, group, O.BF16)
    for r, qw in enumerate(qws):
        lo, hi = shard_bounds(2048, t, r, 32)
        assert np.array_equal(qw.codes.cpu().numpy(), O.pack_codes(ref.q[:, lo:hi], 4))
        j = lo // group
        nrow = max(1, (hi - lo) // group)
        assert np.array_equal(qw.scales.cpu().view(torch.int16).numpy().view(np.uint16), ref.s_bits[j:j + nrow])


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
    y, mid = layer.forward(x, return_all=True)
    torch.cuda.synchronize()

    # every GEMM of the chain against the oracle on the SAME input the layer fed it (the layer's own
    # bf16 intermediates), at the north-star tolerance 2e-3
    def deq(t):
        return O.decode_bits(t.cpu().view(torch.int16).numpy().view(np.uint16), "bf16")

    def check(inp, name, out):
        r = O.quantize(deq(mats[name]), 4, 128, O.BF16)
        Cr, D = O.gemm(deq(inp), r.q, r.s, 128)
        assert O.rel_err(torch_to_f64(out), Cr, D) <= TOL, name
    check(x, "qkv", mid["qkv"])
    check(mid["attn"], "out", mid["out"])
    check(mid["out"], "fc1", mid["fc1"])
    check(mid["fc1"], "fc2", mid["fc2"])
    assert torch.equal(y, mid["fc2"])
    dist.destroy_process_group()
