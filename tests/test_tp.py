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
    check_row_group(12288, 8, 12288)      # per-column groups: each shard holds a slice of the group
    with pytest.raises(ValueError):
        check_row_group(12288, 8, 1024)   # 1536-element shards and 1024-element groups do not nest


class _NumpyOps:
    """CPU stand-ins for the device steps of tp.rowshard_protocol (test infrastructure): the shard
    pass is the oracle's adaptive pass on the shard matrix (whose ladder is the tail of the full
    ladder) plus its column maxima; the cross step evaluates the coarse levels on the table."""

    @staticmethod
    def alloc(nflags, world, N, device):
        buf = torch.zeros(nflags + world * N, dtype=torch.int32)
        return buf, buf[:nflags], buf[nflags:].view(torch.float32)

    @staticmethod
    def shard_pass(W_shard, K, world, rank, alpha_milli, min_group, flags, colmax):
        Wn = W_shard.numpy()
        N = Wn.shape[0]
        lw = world.bit_length() - 1
        for lvl, f in enumerate(O.adapt_flags(Wn, alpha_milli, min_group), start=1):
            if f:
                flags[lvl + lw - 1] = 1
        colmax[rank * N:(rank + 1) * N] = torch.from_numpy(np.abs(Wn).max(axis=1)).float()

    @staticmethod
    def cross(colmax, K, N, world, alpha_milli, min_group, flags):
        tab = colmax.view(world, N).double().numpy()
        lw = world.bit_length() - 1
        for L in range(1, lw + 1):
            span = world >> L
            for j in range(1 << L):
                ch = tab[j * span:(j + 1) * span].max(axis=0)
                pa = tab[(j // 2) * 2 * span:(j // 2 + 1) * 2 * span].max(axis=0)
                if np.any(1000.0 * ch < alpha_milli * pa):
                    flags[L - 1] = 1

    @staticmethod
    def decide(K, min_group, flags):
        return O.adapt_decide([bool(x) for x in flags.tolist()], K, min_group)


def _rowshard_matrices(K=2048, N=16):
    """Matrices whose adaptive decision is made at every depth of the ladder relative to the
    shard size: Gaussian (per-column), a planted outlier (min group), and columns whose second half
    / quarter / eighth is 4x smaller (the decision stops at K/2, K/4, K/8 -- levels that span
    shards at t = 2, 4, 8): each of the first 1/2, 1/4, .. 1/d of every column is scaled by a
    further 1/4, so every level down to K/d has a group at a quarter of its parent's range."""
    mats = {"gauss": O.decode_bits(gaussian_bits((N, K), 0.02, 4001), "bf16"),
            "outlier": O.decode_bits(gaussian_with_outliers_bits((N, K), 0.01, 4002, 1, 1.0), "bf16")}
    for d in (2, 4, 8):
        W = O.decode_bits(gaussian_bits((N, K), 0.02, 4010 + d), "bf16").copy()
        e = 2
        while e <= d:
            W[:, :K // e] = W[:, :K // e] / 4.0
            e *= 2
        mats[f"step{d}"] = W
    return mats


def _rowshard_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2308_09723_b200.tp import rowshard_protocol, shard_bounds
        res = {}
        for name, W in _rowshard_matrices().items():
            K = W.shape[1]
            lo, hi = shard_bounds(K, world, rank, 32)
            g, colmax = rowshard_protocol(torch.from_numpy(np.ascontiguousarray(W[:, lo:hi])), K, world, rank,
                                          500, 16, _NumpyOps,
                                          lambda t: dist.all_reduce(t, op=dist.ReduceOp.MAX))
            tab_ok = np.array_equal(colmax.view(world, -1).double().numpy(),
                                    np.stack([np.abs(W[:, r * K // world:(r + 1) * K // world]).max(axis=1)
                                              for r in range(world)]))
            res[name] = (g, O.adapt_group_size(W, 500, 16), tab_ok)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_rowshard_adaptive_protocol_gloo(world):
    """Row-parallel adaptive group size: each rank holds a K-slice; the
    protocol (shard pass -> one int32 MAX all-reduce of [flags | fp32 column maxima] -> coarse levels
    from the table -> decide) reproduces the UNSHARDED decision on every rank, for decisions made
    both inside one shard and across shards."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rowshard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expected = {"gauss": 2048, "outlier": 16, "step2": 1024, "step4": 512, "step8": 256}
    for rank, r in res:
        for name, (g, g_full, tab_ok) in r.items():
            assert g_full == expected[name], (name, g_full)
            assert g == g_full, f"rank {rank} {name}: sharded g={g}, unsharded {g_full}"
            assert tab_ok, f"rank {rank} {name}: column-max table"
