"""Why does bench.py's quantizer time (fq.quantize, fresh outputs per call) differ from
tools/quant_bench.py (preallocated outputs)?  Times A3 and A1 both ways on OPT-175B FC1 bf16."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2308_09723_b200 import fq
from synth import gaussian_torch


def timeit(fn, reps):
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


N, K = 49152, 12288
W = gaussian_torch((N, K), 0.02, 1001, device="cuda")
d = fq.make_wdesc(K, N, 4, 128, fq.FQ_BF16)
codes = torch.empty((N, K // 2), dtype=torch.uint8, device="cuda")
scales = torch.empty((K // 128, N), dtype=torch.bfloat16, device="cuda")
flags = torch.zeros(fq.fq_adapt_levels(K, 16), dtype=torch.int32, device="cuda")
for reps in (5, 20):
    print(f"reps={reps}")
    print(f"  A3 preallocated          {timeit(lambda: fq.fq_quantize(W, d, codes, scales, None), reps):8.1f} us")
    print(f"  A3 fq.quantize (fresh)   {timeit(lambda: fq.quantize(W, 4, 128), reps):8.1f} us")
    keep = []
    print(f"  A3 fq.quantize (kept)    {timeit(lambda: keep.append(fq.quantize(W, 4, 128)), reps):8.1f} us")
    del keep
    print(f"  A1 fq_adapt_flags        {timeit(lambda: fq.fq_adapt_flags(W, 500, 16, flags), reps):8.1f} us")
    print(f"  A1 fq.adapt_group        {timeit(lambda: fq.adapt_group(W, 500, 16), reps):8.1f} us")
