"""Run fq_gemm_i8 on one OPT-175B shape a few times (for ncu). usage: prof_i8.py FC1|FC2 M [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_09723_b200 import fq  # noqa: E402
from synth import gaussian_torch  # noqa: E402

K, N = {"FC1": (12288, 49152), "FC2": (49152, 12288)}[sys.argv[1]]
M = int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
W = gaussian_torch((N, K), 0.02, 1001)
q = fq.quantize_intscale(W, 128)
del W
A = gaussian_torch((M, K), 1.0, 7)
acts = fq.quantize_acts_i8(A)
for _ in range(reps):
    fq.gemm_i8(None, q, acts=acts)
torch.cuda.synchronize()
