"""Tensor-parallel plumbing (A8) on CPU with the gloo backend, world_size 2 (and 4).

The sharding / all-reduce logic of paper_2308_09723_b200.tp is exercised with the oracle GEMM
injected as the compute (the CUDA kernels need a GPU; their sharded parity is in
test_gpu_tp.py).  Checks: column shards' codes/scales are the slices of the unsharded ones
(bit-exact), the row-parallel all-reduced result equals the unsharded GEMM, and the adaptive
decision agrees on all shards after OR-ing the level flags.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fq_oracle as O
from synth import gaussian_bits, gaussian_with_outliers_bits, activations_bits


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2308_09723_b200.tp import shard_bounds, check_row_group, tp_forward
        K, N, M, bits, g = 512, 256, 3, 4, 64
        Wb1 = gaussian_bits((N, K), 0.02, 1001)        # column-parallel (paper columns = rows here)
        Wb2 = gaussian_bits((K, N), 0.02, 1002)        # row-parallel: [N2=K, K2=N]
        W1 = O.decode_bits(Wb1, "bf16")
        W2 = O.decode_bits(Wb2, "bf16")
        A = O.decode_bits(activations_bits(M, K, 2001), "bf16")
        # column shard of W1 (output columns), row shard of W2 (its K = N of W1)
        c0, c1 = shard_bounds(N, world, rank)
        r0, r1 = shard_bounds(N, world, rank, 32)
        assert (c0, c1) == (r0, r1)
        check_row_group(N, world, g)
        q1 = O.quantize(W1[c0:c1], bits, g, O.BF16)
        q2 = O.quantize(W2[:, r0:r1], bits, g, O.BF16)
        full1 = O.quantize(W1, bits, g, O.BF16)
        full2 = O.quantize(W2, bits, g, O.BF16)
        ok_codes = np.array_equal(q1.q, full1.q[c0:c1]) and np.array_equal(q1.s, full1.s[:, c0:c1])
        ok_codes &= np.array_equal(q2.q, full2.q[:, r0:r1]) and np.array_equal(q2.s, full2.s[r0 // g:r1 // g])

        def gemm_fn(x, shard):
            qq, g_ = shard
            C, _ = O.gemm(x.numpy(), qq.q, qq.s, g_)
            return torch.from_numpy(C)

        def allreduce(t):
            dist.all_reduce(t, op=dist.ReduceOp.SUM)

        out = tp_forward(torch.from_numpy(A), [(q1, g), (q2, g)], gemm_fn, allreduce, ["col", "row"],
                         world, rank)
        ref1, _ = O.gemm(A, full1.q, full1.s, g)
        ref, D = O.gemm(ref1, full2.q, full2.s, g)
        err = O.rel_err(out.numpy(), ref, D)

        # adaptive decision: OR of shard flags (all-reduce MAX) == unsharded flags
        Wa = O.decode_bits(gaussian_with_outliers_bits((64, 1024), 0.01, 77, 1, 1.0), "bf16")
        lo, hi = shard_bounds(64, world, rank)
        f = torch.tensor([int(x) for x in O.adapt_flags(Wa[lo:hi], 500, 16)], dtype=torch.int32)
        dist.all_reduce(f, op=dist.ReduceOp.MAX)
        ok_adapt = [bool(x) for x in f.tolist()] == O.adapt_flags(Wa, 500, 16)
        q.put((rank, bool(ok_codes), float(err), bool(ok_adapt)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_tp_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_codes, err, ok_adapt in res:
        assert ok_codes, f"rank {rank}: shard codes are not slices of the unsharded codes"
        assert err <= 1e-12, f"rank {rank}: TP result differs from unsharded ({err})"
        assert ok_adapt, f"rank {rank}: adaptive flags disagree"


def test_shard_validation():
    from paper_2308_09723_b200.tp import shard_bounds, check_row_group
    assert shard_bounds(49152, 8, 3) == (18432, 24576)
    with pytest.raises(ValueError):
        shard_bounds(100, 8, 0)
    check_row_group(49152, 8, 128)
    with pytest.raises(ValueError):
        check_row_group(12288, 8, 12288)  # per-column groups cannot be row-sharded
