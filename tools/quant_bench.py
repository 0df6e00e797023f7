"""Time fq_quantize (A3) and fq_adapt_flags (A1) on the OPT-175B FC1/FC2 matrices (bf16 W)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_09723_b200 import fq
from synth import gaussian_torch

def bench(fn, reps=10):
    for _ in range(3): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3

for name, K, N in (("FC1", 12288, 49152), ("FC2", 49152, 12288)):
    W = gaussian_torch((N, K), 0.02, 1)
    for bits in (4, 8):
        q = fq.quantize(W, bits, 128)
        d = fq.make_wdesc(K, N, bits, 128, fq.FQ_BF16)
        us = bench(lambda: fq.fq_quantize(W, d, q.codes, q.scales, None))
        nb = W.numel() * 2 + q.nbytes
        print(f"quantize {name} int{bits} g128: {us:7.1f} us  {nb/us/1e6:5.2f} TB/s", flush=True)
    us = bench(lambda: fq.adapt_group(W, 500, 16))
    print(f"adapt    {name}: {us:7.1f} us  {W.numel()*2/us/1e6:5.2f} TB/s (incl. D2H of the flags)", flush=True)
