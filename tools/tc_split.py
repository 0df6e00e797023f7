"""Prefill (A6) K-split sweep: OPT-175B FC1 / FC2 int4 g128 at M = 2048 / 4096 / 8192 with the tcgen05
path forced and 1..3 K splits (wave quantization: FC2 M=2048 has 768 tiles on 148 SMs = 5.19 rounds)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_09723_b200 import fq
from synth import gaussian_torch


def bench(fn, reps=5):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps / 1e3


for name, (K, N) in (("FC1", (12288, 49152)), ("FC2", (49152, 12288))):
    W = gaussian_torch((N, K), 0.02, 1)
    q = fq.quantize(W, 4, 128); del W
    for M in (2048, 4096, 8192):
        A = gaussian_torch((M, K), 1.0, 2)
        C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        for sp in (0, 1, 2, 3):
            o = fq.make_opts("tc", sp)
            try:
                t = bench(lambda: fq.gemm(A, q, out=C, opts=o))
            except fq.FQError as ex:
                print(f"{name} M={M} splits={sp}: {ex}", flush=True); continue
            print(f"{name} M={M} splits={sp}: {t*1e3:.3f} ms {2*M*K*N/t/1e12:.0f} TFLOP/s", flush=True)
        del A, C
