"""Decode split-K sweep (FQ_GEMV_SPLITS) on OPT-175B FC1/FC2, g128.  usage: split_sweep.py [bits]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_09723_b200 import fq
from synth import gaussian_torch
BITS = int(sys.argv[1]) if len(sys.argv) > 1 else 4

def bench(fn, reps=30):
    for _ in range(5): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3

for name, K, N in (("FC1", 12288, 49152), ("FC2", 49152, 12288)):
    W = gaussian_torch((N, K), 0.02, 1); q = fq.quantize(W, BITS, 128); del W
    for M in (1, 8, 16):
        A = gaussian_torch((M, K), 1.0, 2); C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        row = []
        for sp in ["auto"] + [str(x) for x in (1, 2, 3, 4, 5, 6, 8, 10, 12, 16, 24)]:
            if sp == "auto": os.environ.pop("FQ_GEMV_SPLITS", None)
            else: os.environ["FQ_GEMV_SPLITS"] = sp
            fq._WS_BYTES.clear()  # the split count changes the workspace size
            row.append(f"{sp}:{bench(lambda: fq.gemm(A, q, out=C)):.1f}")
        os.environ.pop("FQ_GEMV_SPLITS", None)
        print(name, f"int{BITS}", M, " ".join(row), flush=True)
