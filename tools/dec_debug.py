"""Time the decode kernel's diagnostic variants (FQ_DEC_DEBUG) on FC1/FC2, M=1."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_09723_b200 import fq
from synth import gaussian_torch

def bench(fn, reps=50):
    for _ in range(5): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3

for K, N in ((12288, 49152), (49152, 12288)):
    W = gaussian_torch((N, K), 0.02, 1)
    q = fq.quantize(W, 4, 128); del W
    A = gaussian_torch((1, K), 1.0, 2)
    C = torch.empty(1, N, dtype=torch.bfloat16, device="cuda")
    for dbg in ("0", "3", "4"):
        os.environ["FQ_DEC_DEBUG"] = dbg
        for sp in (os.environ.get("SPLITS_LIST", "0").split(",")):
            if sp != "0": os.environ["FQ_GEMV_SPLITS"] = sp
            else: os.environ.pop("FQ_GEMV_SPLITS", None)
            us = bench(lambda: fq.gemm(A, q, out=C))
            print(f"K={K} N={N} dbg={dbg} splits={sp}: {us:7.1f} us  {q.nbytes/us/1e6:5.2f} TB/s", flush=True)
    os.environ["FQ_DEC_DEBUG"] = "0"
