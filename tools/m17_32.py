import os, sys
sys.path.insert(0, os.getcwd())
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
for name, (K, N) in {"FC1": (12288, 49152), "FC2": (49152, 12288), "13B-FFN1": (5120, 20480), "30B-FFN1": (7168, 28672)}.items():
    q = fq.quantize(gaussian_torch((N, K), 0.02, 1), 4, 128)
    for M in (17, 24, 32):
        A = gaussian_torch((M, K), 1.0, 2)
        r = {p: bench(lambda: fq.gemm(A, q, opts=fq.make_opts(p))) for p in ("decode", "tc")}
        print(name, M, {k: round(v, 1) for k, v in r.items()}, flush=True)
