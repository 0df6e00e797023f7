"""Time the tcgen05 decode kernel's diagnostic variants (FQ_DTC_DBG bits: 1 dequant, 2 fold math,
4 stager, 8 MMA skipped) on OPT-175B FC1 int4 g128."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_09723_b200 import fq
from synth import gaussian_torch
def bench(fn, reps=30):
    for _ in range(5): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3
K, N = 12288, 49152
W = gaussian_torch((N, K), 0.02, 1); q = fq.quantize(W, 4, 128); del W
for M in (1, 16):
    A = gaussian_torch((M, K), 1.0, 2); C = fq.gemm(A, q)
    for dbg in (0, 1, 4, 8, 15, 32, 47, 63, 33, 36):
        os.environ["FQ_DTC_DBG"] = str(dbg)
        print(M, dbg, f"{bench(lambda: fq.gemm(A, q, out=C)):.1f} us", flush=True)
    os.environ["FQ_DTC_DBG"] = "0"
