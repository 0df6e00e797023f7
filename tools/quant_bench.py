"""Time the quantizer A3 (fq_quantize) and the adaptive pass A1 (fq_adapt_flags) on OPT-175B
FC1 / FC2 weights with preallocated outputs; prints us per call and algorithmic GB/s (W read once +
codes + scales written).  Diagnostics; A/B library builds with FQ_LIB_PATH.

    python tools/quant_bench.py [--shapes FC1 FC2] [--bits 4 8 3] [--groups 128 64]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2308_09723_b200 import fq
from synth import gaussian_torch

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", nargs="+", default=["FC1", "FC2"])
ap.add_argument("--bits", type=int, nargs="+", default=[4])
ap.add_argument("--groups", type=int, nargs="+", default=[128])
ap.add_argument("--wdt", nargs="+", default=["bf16"])
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
SH = {"FC1": (49152, 12288), "FC2": (12288, 49152)}
DT = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32}


def timeit(fn, reps):
    for _ in range(2):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


for wdt in a.wdt:
    for name in a.shapes:
        N, K = SH[name]
        if wdt == "fp32":
            N //= 2  # keep W at ~1.2 GB
        W = gaussian_torch((N, K), 0.02, 1).to(DT[wdt])
        wbytes = W.numel() * W.element_size()
        flags = torch.zeros(fq.fq_adapt_levels(K, 16), dtype=torch.int32, device="cuda")
        us = timeit(lambda: fq.fq_adapt_flags(W, 500, 16, flags), a.reps)
        print(f"{name} {wdt} A1 adapt_flags           {us:8.1f} us {wbytes / us / 1e3:7.0f} GB/s", flush=True)
        for bits in a.bits:
            for g in a.groups:
                d = fq.make_wdesc(K, N, bits, g, fq.FQ_BF16)
                codes = torch.empty((N, K * bits // 8), dtype=torch.uint8, device="cuda")
                scales = torch.empty((K // g, N), dtype=torch.bfloat16, device="cuda")
                us = timeit(lambda: fq.fq_quantize(W, d, codes, scales, None), a.reps)
                tot = wbytes + codes.numel() + scales.numel() * 2
                print(f"{name} {wdt} A3 int{bits} g{g:<6d}        {us:8.1f} us {tot / us / 1e3:7.0f} GB/s", flush=True)
        del W
        torch.cuda.empty_cache()
