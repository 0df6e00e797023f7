"""Small invocations of every kernel class, for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): quantizer A3 + adaptive A1 (incl. row-shard TP pass), decode A4 (one / two / four
8-token tiles, nibble, group-split, int8 and per-element-scale paths, split-K), tcgen05 A6 (one- and
two-half tiles, split-K, 256-token tiles), MoE batch A7 (host and device offsets), and the round-2
kernels: int3 / int2 decode, the int8-activation path (quantizers + kind::i8 GEMM), the fused
row-parallel all-reduce.  Checks results are finite."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_09723_b200 import fq
from synth import gaussian_torch

def run(M, K, N, bits, group, opts=None, adt=torch.bfloat16):
    W = gaussian_torch((N, K), 0.02, 1)
    q = fq.quantize(W, bits, group, scale_dtype=adt)
    A = gaussian_torch((M, K), 1.0, 2).to(adt)
    C = fq.gemm(A, q, opts=opts)
    torch.cuda.synchronize()
    assert torch.isfinite(C.float()).all()
    print(f"ok M={M} K={K} N={N} b={bits} g={group} {opts and (opts.path, opts.splits, opts.tc_halves)}", flush=True)

W = gaussian_torch((256, 2048), 0.02, 3)
W[3, 5] = 1.0
g = fq.adapt_group(W, 500, 16)
print("adaptive g", g)
for M in (1, 9, 24):
    run(M, 2048, 512, 4, 128)
run(5, 2048, 512, 4, 64)                      # group-split nibble path
run(2, 1152, 264, 4, 384, fq.make_opts("decode", 3))  # double stages: ragged K, mid-group split starts
run(12, 1152, 264, 4, 128)                    # double stages, two MMA token tiles, K = 4.5 stages
run(5, 2048, 512, 8, 128)                     # int8
run(5, 2048, 520, 4, 32)                      # per-element-scale path, ragged N
run(3, 4096, 512, 4, 128, fq.make_opts("decode", 3))  # split-K
run(64, 2048, 512, 4, 128, fq.make_opts("tc", 0, 1))   # A6 one-half, split-K
run(64, 2048, 520, 4, 64, fq.make_opts("tc", 0, 2))    # A6 two-half, N tail
run(300, 1024, 384, 8, 128)                   # A6 256-token tiles, int8
run(40, 1024, 256, 4, 128, adt=torch.float16)
# MoE batch (decode + tcgen05 experts, adaptive groups)
E, K, N = 6, 1024, 512
experts = []
for e in range(E):
    We = gaussian_torch((N, K), 0.02, 10 + e)
    if e % 2 == 0:
        We[e, e] = 1.0
    experts.append(fq.quantize(We, 4, None))
off = [0, 0, 3, 20, 21, 60, 64]
A = gaussian_torch((64, K), 1.0, 4)
C = fq.gemm_grouped(A, off, experts)
torch.cuda.synchronize()
assert torch.isfinite(C.float()).all()
print("ok moe")
# row-shard TP pass (2 shards simulated)
from paper_2308_09723_b200.tp import rowshard_protocol
Wf = gaussian_torch((256, 2048), 0.02, 5)
for r in range(2):
    gr, cm = rowshard_protocol(Wf[:, r * 1024:(r + 1) * 1024].contiguous(), 2048, 2, r, 500, 16, fq.KERNEL_OPS, None)
    q = fq.quantize_rowshard(Wf[:, r * 1024:(r + 1) * 1024].contiguous(), 2048, 2, r, 4, 2048, cm)
torch.cuda.synchronize()
print("ok rowshard")
# ---- round 2 kernels ----------------------------------------------------------------------------
# int3 / int2 decode (NEXT-3): nibble path and per-element-scale path
for bits in (3, 2):
    run(5, 1024, 512, bits, 128)
    run(3, 1024, 264, bits, 64)
    run(20, 1024, 512, bits, 128)
# int8-activation x int4-weight path (NEXT-4): quantizers + the kind::i8 GEMM, every tile width,
# split-K (few tiles) and a 256-token tile
Wi = gaussian_torch((384, 2048), 0.02, 6)
Wi[1, 2] = float("nan")
st = torch.zeros(1, dtype=torch.int32, device="cuda")
qi = fq.quantize_intscale(Wi, 64, status=st)
for M in (1, 33, 200):
    Ai = gaussian_torch((M, 2048), 1.0, 7)
    Ci = fq.gemm_i8(Ai, qi)
    torch.cuda.synchronize()
    assert torch.isfinite(Ci.float()).all()
    print(f"ok i8 M={M}", flush=True)
# device-offset MoE (decode segments + tcgen05 remainder)
od = torch.tensor([0, 0, 3, 20, 21, 60, 64], dtype=torch.int64, device="cuda")
C = fq.gemm_grouped_dev(A, od, experts, 40)
torch.cuda.synchronize()
assert torch.isfinite(C.float()).all()
print("ok moe device offsets")
# fused row-parallel GEMM + one-shot all-reduce (NEXT-1), 4 ranks on one device
world, M, K, N = 4, 5, 4096, 512
Wx = gaussian_torch((N, K), 0.02, 8)
Ax = gaussian_torch((M, K), 1.0, 9)
Ks = K // world
qs = [fq.quantize(Wx[:, r * Ks:(r + 1) * Ks].contiguous(), 4, 128) for r in range(world)]
ranks = fq.xr_group_local(world, M, qs[0].desc, torch.bfloat16)
d = qs[0].desc
nb = fq.fq_gemm_workspace_bytes_ex(M, d, fq.make_opts("decode"))
wss = [torch.zeros(max(nb, 256), dtype=torch.uint8, device="cuda") for _ in range(world)]
for r, R in enumerate(ranks):
    fq.fq_gemm_allreduce(Ax[:, r * Ks:(r + 1) * Ks].contiguous(), M, d, qs[r].codes, qs[r].scales, fq.FQ_BF16,
                         R.peers, R.peers_dev, wss[r])
for R in ranks:
    fq.fq_xr_wait(R.peers, M, d)
torch.cuda.synchronize()
assert torch.isfinite(ranks[0].out.float()).all()
print("ok fused all-reduce")
# A6 with two CTAs per SM (int4 one-half tiles of <= 64 tokens that fill the GPU without a K split)
run(40, 1024, 19200, 4, 128)
run(20, 1024, 19200, 4, 64)
