"""Decode timing of int3 / int2 weights (NEXT-3) next to int4 at OPT-175B shapes, g = 128 and 64.
Effective bytes = codes + scales."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_09723_b200 import fq  # noqa: E402
from synth import gaussian_torch  # noqa: E402


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


out = {}
for name, (K, N) in (("FC1", (12288, 49152)), ("FC2", (49152, 12288))):
    W = gaussian_torch((N, K), 0.02, 1001)
    for g in (128, 64):
        for bits in (4, 3, 2):
            q = fq.quantize(W, bits, g)
            for M in (1, 8, 16):
                A = gaussian_torch((M, K), 1.0, 7)
                C = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
                t = timeit(lambda: fq.gemm(A, q, out=C))
                out[f"{name}_int{bits}_g{g}_M{M}"] = {"us": round(t, 1), "TB_s": round(q.nbytes / t / 1e6, 3)}
                print(name, bits, g, M, out[f"{name}_int{bits}_g{g}_M{M}"], flush=True)
            del q
    del W
    torch.cuda.empty_cache()
print(json.dumps(out))
