"""Timing of the int8-activation x int4-weight path (NEXT-4) at OPT-175B shapes next to the bf16 path.
Usage: python tools/i8_bench.py [--ms 1,16,64,2048]"""
import argparse
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
    return s.elapsed_time(e) / reps * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ms", default="1,2,4,8,16,32,64,128,256,2048,4096")
    a = ap.parse_args()
    out = {}
    for name, (K, N) in (("FC1", (12288, 49152)), ("FC2", (49152, 12288))):
        W = gaussian_torch((N, K), 0.02, 1001)
        q8 = fq.quantize_intscale(W, 128)
        q4 = fq.quantize(W, 4, 128)
        wb = q8.nbytes
        for M in [int(x) for x in a.ms.split(",")]:
            A = gaussian_torch((M, K), 1.0, 7)
            acts = fq.quantize_acts_i8(A)
            C = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
            t_g = timeit(lambda: fq.gemm_i8(None, q8, out=C, acts=acts))
            t_q = timeit(lambda: fq.quantize_acts_i8(A))
            t_f = timeit(lambda: fq.gemm(A, q4, out=C))
            fl = 2.0 * M * K * N
            out[f"{name}_M{M}"] = {"i8_gemm_us": round(t_g, 1), "act_quant_us": round(t_q, 1),
                                   "i8_TB_s": round(wb / t_g / 1e6, 3), "i8_TOPS": round(fl / t_g / 1e6, 1),
                                   "bf16_path_us": round(t_f, 1), "bf16_TFLOPs": round(fl / t_f / 1e6, 1)}
            print(name, M, out[f"{name}_M{M}"], flush=True)
            del A, acts, C
        del W, q8, q4
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
