"""Mid-M bf16 x int4 GEMM timings (A6 and the decode kernel's 17..32 range): OPT-175B FC1 / FC2 and
the OPT-13B/30B matrices at M = 24..128, plus the MoE batch at M_e = 32 / 64.  Compare libfq build
variants with FQ_LIB_PATH.  usage: python tools/mid_m.py"""
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


SH = {"175B-FC1": (12288, 49152), "175B-FC2": (49152, 12288), "13B-FFN2": (20480, 5120), "30B-QKV": (7168, 21504)}
for name, (K, N) in SH.items():
    W = gaussian_torch((N, K), 0.02, 1)
    q = fq.quantize(W, 4, 128)
    del W
    row = []
    for M in (24, 48, 64, 128):
        A = gaussian_torch((M, K), 1.0, 2)
        C = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
        row.append(f"M={M}: {bench(lambda: fq.gemm(A, q, out=C)):7.1f}")
    print(name, "  ".join(row), "us", flush=True)
    del q
E, K, N = 64, 4096, 16384
ex = [fq.quantize(gaussian_torch((N, K), 0.02, 100 + e), 4, 128) for e in range(E)]
for me in (32, 64):
    A = gaussian_torch((E * me, K), 1.0, 3)
    off = [e * me for e in range(E + 1)]
    print(f"MoE g128 M_e={me}: {bench(lambda: fq.gemm_grouped(A, off, ex), 5):8.1f} us", flush=True)
