"""Tiny driver for ncu captures: quantize one OPT-175B matrix and launch fq_gemm a few times.

    python tools/prof_gemm.py --K 12288 --N 49152 --M 1 --bits 4 --iters 5
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2308_09723_b200 import fq  # noqa: E402
from synth import gaussian_torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--K", type=int, default=12288)
ap.add_argument("--N", type=int, default=49152)
ap.add_argument("--M", type=int, nargs="+", default=[1])
ap.add_argument("--bits", type=int, default=4)
ap.add_argument("--group", type=int, default=128)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--quantize", action="store_true", help="also launch the quantizer in the loop")
a = ap.parse_args()

W = gaussian_torch((a.N, a.K), 0.02, 1001)
qw = fq.quantize(W, a.bits, a.group)
if not a.quantize:
    del W
for M in a.M:
    A = gaussian_torch((M, a.K), 1.0, 7)
    C = fq.gemm(A, qw)
    for _ in range(a.iters):
        fq.gemm(A, qw, out=C)
        if a.quantize:
            fq.quantize(W, a.bits, a.group)
torch.cuda.synchronize()
print("done")
