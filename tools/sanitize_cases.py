"""Small invocations of every kernel class, for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): quantizer A3 + adaptive A1 (incl. row-shard TP pass), decode A4 (one / two / four
8-token tiles, nibble, group-split, int8 and per-element-scale paths, split-K), tcgen05 A6 (one- and
two-half tiles, split-K, 256-token tiles), MoE batch A7.  Checks results are finite."""
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
