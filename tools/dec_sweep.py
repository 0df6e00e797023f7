"""Time fq_gemm decode (M = 1..32) on OPT-175B FC1/FC2 int4 g128 (int8 with --bits 8), per path.

    python tools/dec_sweep.py --paths decode --M 1 8 16 32 [--splits S]
Each GEMM is repeated back to back (weights 311 MB > L2, so no flush is needed)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_09723_b200 import fq
from synth import gaussian_torch

ap = argparse.ArgumentParser()
ap.add_argument("--bits", type=int, default=4)
ap.add_argument("--M", type=int, nargs="+", default=[1, 2, 4, 8, 9, 12, 16, 24, 32])
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--paths", nargs="+", default=["auto"])
ap.add_argument("--splits", type=int, nargs="+", default=[0])
ap.add_argument("--shapes", nargs="+", default=["FC1", "FC2"])
a = ap.parse_args()

def bench(fn, reps):
    for _ in range(5): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3

SH = {"FC1": (12288, 49152), "FC2": (49152, 12288), "QKV": (12288, 36864), "OUT": (12288, 12288)}
for name in a.shapes:
    K, N = SH[name]
    W = gaussian_torch((N, K), 0.02, 1)
    q = fq.quantize(W, a.bits, 128); del W
    for M in a.M:
        A = gaussian_torch((M, K), 1.0, 2)
        C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        for path in a.paths:
            for sp in a.splits:
                o = None if (path == "auto" and sp == 0) else fq.make_opts(path, sp)
                try:
                    us = bench(lambda: fq.gemm(A, q, out=C, opts=o), a.reps)
                except fq.FQError as ex:
                    print(f"{name} int{a.bits} M={M:2d} {path:12s} s={sp}: {ex}", flush=True)
                    continue
                print(f"{name} int{a.bits} M={M:2d} {path:12s} s={sp}: {us:7.1f} us  {q.nbytes/us/1e6:5.2f} TB/s",
                      flush=True)
