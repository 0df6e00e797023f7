"""Tensor-parallel FineQuant layers (kernel A8 plumbing): one process per GPU, torch.distributed.

The paper serves OPT-175B with tensor parallelism and notes "We must issue an all reduce after
each attention and FFN block ... it is desirable to use as few GPUs as possible" (§2.1).
Megatron-style partitioning of a transformer layer:

  * column-parallel (QKV, FC1): output columns n are sharded, A is replicated, no communication.
    Groups run along K, so a column shard never splits a group; each rank's codes/scales are the
    column slice of the unsharded ones (bit-exact).
  * row-parallel (out-proj, FC2): the reduction dim K is sharded (requires group | K/t); each rank
    produces a partial C over its K slice, then an all-reduce(SUM) over NCCL (NVLink/NVSwitch).
  * adaptive group size (reading R11: one g per matrix, decided on the FULL matrix):
      - column shards hold whole columns: the level flags of all shards are OR-ed (all-reduce MAX)
        before the host decision;
      - row shards hold K-slices: `rowshard_protocol` decides g on the full-K ladder -- the levels
        whose groups lie inside one shard come from each shard's own pass (OR-ed), the coarse levels
        whose groups span shards from the MAX-all-reduced table of shard column maxima (SURVEY §8(c)
        C-T) -- and groups larger than K/t are quantized from that table's group maxima, so every
        shard's codes/scales are the K-/G-slices of the unsharded ones.

The GEMM and quantizer are the libfq kernels; this module only shards, calls and reduces.
The shard arithmetic is kept in pure functions (`shard_bounds`, `tp_forward`) so the multi-process
logic can be tested with the gloo backend on CPU by injecting a reference GEMM.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import torch
import torch.distributed as dist


def shard_bounds(n: int, world: int, rank: int, align: int = 8) -> tuple[int, int]:
    """Contiguous, equal shard [lo, hi) of a dimension of size n (n % (world*align) == 0)."""
    if n % (world * align):
        raise ValueError(f"dimension {n} does not split into {world} shards aligned to {align}")
    sz = n // world
    return rank * sz, (rank + 1) * sz


def check_row_group(K: int, world: int, group: int) -> None:
    """Row-parallel shards hold whole groups (group | K/world) or whole shards of one group
    ((K/world) | group, the group amax then comes from the shards' column maxima)."""
    ks = K // world
    if K % world or (ks % group and group % ks):
        raise ValueError(f"row-parallel shard K/t={ks} and group {group} do not nest")


def rowshard_protocol(W_shard, K: int, world: int, rank: int, alpha_milli: int, min_group: int, ops,
                      allreduce_max: Callable | None, adaptive: bool = True):
    """Adaptive group size of a row-parallel (K-sharded) matrix, decided on the full-K ladder
    (fq.h fq_adapt_flags_rowshard / fq_adapt_flags_cross).  `ops` supplies the device steps
    (fq.KERNEL_OPS on the GPU); `allreduce_max(t)` MAX-reduces an int32 tensor over the ranks of
    the matrix in place (None: a single rank).  Returns (g or None, colmax [world, N] fp32)."""
    from .fq import fq_adapt_levels
    N = W_shard.shape[0]
    nflags = max(0, fq_adapt_levels(K, min_group) - 1)
    buf, flags, colmax = ops.alloc(nflags, world, N, W_shard.device)
    ops.shard_pass(W_shard, K, world, rank, alpha_milli, min_group, flags, colmax)
    if allreduce_max is not None and world > 1:
        allreduce_max(buf)
    if not adaptive:
        return None, colmax
    if nflags:
        ops.cross(colmax, K, N, world, alpha_milli, min_group, flags)
    return ops.decide(K, min_group, flags), colmax


@dataclass
class ShardSpec:
    kind: str      # "col" or "row"
    K: int         # full reduction dim
    N: int         # full output dim
    world: int
    rank: int

    @property
    def bounds(self) -> tuple[int, int]:
        return shard_bounds(self.N if self.kind == "col" else self.K, self.world, self.rank,
                            8 if self.kind == "col" else 32)


def tp_forward(x: torch.Tensor, shards: list, gemm_fn: Callable, allreduce_fn: Callable | None,
               kinds: list[str], world: int, rank: int) -> torch.Tensor:
    """Run a chain of TP linears: column layers produce a column shard of their output; a row layer
    consumes the column shard produced before it and all-reduces its partial output.

    gemm_fn(x, shard) -> x @ W_shard^T ; allreduce_fn(t) sums t over the TP group in place."""
    h = x
    for shard, kind in zip(shards, kinds):
        if kind == "col":
            h = gemm_fn(h, shard)
        elif kind == "row":
            h = gemm_fn(h, shard)
            if allreduce_fn is not None and world > 1:
                allreduce_fn(h)
        else:
            raise ValueError(kind)
    return h


class TPLinearFQ:
    """A quantized linear shard on this rank (canonical libfq layout).  Its codes/scales are the
    slices of the unsharded matrix's quantization (bit-exact), adaptive group size included."""

    def __init__(self, W_shard: torch.Tensor, spec: ShardSpec, bits: int = 4, group: int | None = 128,
                 alpha_milli: int = 500, min_group: int = 16, process_group=None):
        from . import fq
        self.spec = spec
        W_shard = W_shard.contiguous()
        if spec.kind == "row":
            ks = spec.K // spec.world
            colmax = None
            if group is None or group > ks:
                def amax(t):
                    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=process_group)
                g, colmax = rowshard_protocol(W_shard, spec.K, spec.world, spec.rank, alpha_milli, min_group,
                                              fq.KERNEL_OPS, amax if spec.world > 1 else None,
                                              adaptive=group is None)
                group = g if group is None else group
            check_row_group(spec.K, spec.world, group)
            self.group = group
            self.qw = fq.quantize_rowshard(W_shard, spec.K, spec.world, spec.rank, bits, group, colmax)
            return
        if group is None:  # column shards: OR the flags of all shards of this matrix
            group = fq.adapt_group(W_shard, alpha_milli, min_group,
                                   process_group=process_group if spec.world > 1 else None)
        self.group = group
        self.qw = fq.quantize(W_shard, bits, group)

    def __call__(self, x: torch.Tensor, out_dtype=None) -> torch.Tensor:
        from . import fq
        return fq.gemm(x.contiguous(), self.qw, out_dtype=out_dtype)


class TPOptLayer:
    """The GEMM chain of one OPT decoder layer under TP (configs[4]):
        QKV (col) -> [attention stand-in: the first h/t columns of this rank's QKV shard]
        -> out-proj (row) -> all-reduce -> FC1 (col) -> FC2 (row) -> all-reduce.
    Attention, layer norms, residuals and the activation function are outside the FineQuant hot
    path and are not modelled; the communication pattern (two all-reduces per
    layer) and every weight byte are."""

    def __init__(self, qkv: TPLinearFQ, out: TPLinearFQ, fc1: TPLinearFQ, fc2: TPLinearFQ,
                 process_group=None, fused: bool = False):
        self.qkv, self.out, self.fc1, self.fc2 = qkv, out, fc1, fc2
        self.pg = process_group
        self.world = qkv.spec.world
        # fused=True: row-parallel GEMMs of decode size (M within the decode kernel) run the fused
        # GEMM + one-shot all-reduce over NVLink peer memory (fq.h fq_gemm_allreduce, NEXT-1) instead of
        # GEMM -> NCCL all-reduce.  Its output buffer is reused by the next call of the same layer and M.
        self.fused = fused and self.world > 1
        self._xr = {}

    def _row(self, lin: TPLinearFQ, h: torch.Tensor, dtype) -> torch.Tensor:
        from . import fq
        M = h.shape[0]
        if self.fused and M <= fq.gemv_max_m(lin.qw.bits, lin.qw.group):
            key = (id(lin), M, dtype)
            xr = self._xr.get(key)
            if xr is None:
                xr = self._xr[key] = fq.xr_group_symmetric(self.pg, M, lin.qw.desc, dtype)
            return xr.gemm(h.contiguous(), lin.qw)
        part = lin(h, out_dtype=torch.float32)  # fp32 partials, summed across ranks
        if self.world > 1:
            dist.all_reduce(part, op=dist.ReduceOp.SUM, group=self.pg)
        return part.to(dtype)

    def forward(self, x: torch.Tensor, return_all: bool = False):
        hs = self.out.qw.K  # h / t: the K shard of the out-projection
        q = self.qkv(x)
        a = q[:, :hs].contiguous()
        y = self._row(self.out, a, x.dtype)
        f = self.fc1(y)
        z = self._row(self.fc2, f, x.dtype)
        return (z, dict(qkv=q, attn=a, out=y, fc1=f, fc2=z)) if return_all else z

    @property
    def weight_bytes(self) -> int:
        return sum(l.qw.nbytes for l in (self.qkv, self.out, self.fc1, self.fc2))
