"""One launch of the FQ_DTC_PROF variant (per-warp barrier-wait cycles printed by CTA 0)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_09723_b200 import fq
from synth import gaussian_torch
K, N = 12288, 49152
W = gaussian_torch((N, K), 0.02, 1); q = fq.quantize(W, 4, 128); del W
for M in [int(x) for x in os.environ.get("PM", "1").split(",")]:
    A = gaussian_torch((M, K), 1.0, 2)
    for dbg in os.environ.get("DBGS", "0").split(","):
        os.environ["FQ_DTC_DBG"] = dbg
        C = fq.gemm(A, q); torch.cuda.synchronize()
        print(f"--- M={M} dbg={dbg} (previous lines are a warm-up launch)", flush=True)
        C = fq.gemm(A, q); torch.cuda.synchronize()
