"""Time fq_gemm decode (M = 1..16) on OPT-175B FC1/FC2 int4 g128 (and int8 with --bits 8)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_09723_b200 import fq
from synth import gaussian_torch

ap = argparse.ArgumentParser()
ap.add_argument("--bits", type=int, default=4)
ap.add_argument("--M", type=int, nargs="+", default=[1, 2, 4, 8, 9, 12, 16])
ap.add_argument("--reps", type=int, default=30)
a = ap.parse_args()

def bench(fn, reps):
    for _ in range(5): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3

for name, K, N in (("FC1", 12288, 49152), ("FC2", 49152, 12288)):
    W = gaussian_torch((N, K), 0.02, 1)
    q = fq.quantize(W, a.bits, 128); del W
    for M in a.M:
        A = gaussian_torch((M, K), 1.0, 2)
        C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        us = bench(lambda: fq.gemm(A, q, out=C), a.reps)
        print(f"{name} int{a.bits} M={M:2d}: {us:7.1f} us  {q.nbytes/us/1e6:5.2f} TB/s", flush=True)
