"""Tiny driver for ncu captures of the MoE batch (64 experts x [16384 x 4096] int4, M_e tokens each)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_09723_b200 import fq
from synth import gaussian_torch
ap = argparse.ArgumentParser()
ap.add_argument("--me", type=int, default=64)
ap.add_argument("--experts", type=int, default=16)
ap.add_argument("--group", type=int, default=128)
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
E, K, N = a.experts, 4096, 16384
ex = []
for e in range(E):
    W = gaussian_torch((N, K), 0.02, 7000 + e)
    ex.append(fq.quantize(W, 4, a.group)); del W
off = [e * a.me for e in range(E + 1)]
A = gaussian_torch((E * a.me, K), 1.0, 3)
for _ in range(a.iters):
    fq.gemm_grouped(A, off, ex)
torch.cuda.synchronize()
print("done")
