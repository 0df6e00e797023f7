"""A6 <= 32-token variant vs the decode kernel (diagnostics): OPT-175B FC1/FC2 int4 g128 at M = 8..32,
MoE (64 x [16384 x 4096] int4 g128) at M_e = 16 / 32.  Path/tiles from the environment
(FQ_GEMM_PATH, FQ_TC_HM, FQ_TC_NO32)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_09723_b200 import fq
from synth import gaussian_torch


def bench(fn, reps=20):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps / 1e3


tag = " ".join(f"{k}={os.environ[k]}" for k in ("FQ_GEMM_PATH", "FQ_TC_HM", "FQ_TC_NO32") if k in os.environ) or "default"
for name, K, N in (("FC1", 12288, 49152), ("FC2", 49152, 12288)):
    q = fq.quantize(gaussian_torch((N, K), 0.02, 1), 4, 128)
    for M in (8, 16, 32):
        A = gaussian_torch((M, K), 1.0, 2)
        C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        t = bench(lambda: fq.gemm(A, q, out=C))
        print(f"[{tag}] {name} int4 M={M}: {t*1e6:8.1f} us {q.nbytes/t/1e12:5.2f} TB/s", flush=True)
    del q
E, K, N = 64, 4096, 16384
ex = [fq.quantize(gaussian_torch((N, K), 0.02, 7000 + e), 4, 128) for e in range(E)]
wb = sum(x.nbytes for x in ex)
for me in (16, 32):
    off = [e * me for e in range(E + 1)]
    A = gaussian_torch((E * me, K), 1.0, 3)
    t = bench(lambda: fq.gemm_grouped(A, off, ex), 5)
    print(f"[{tag}] MoE g128 M_e={me}: {t*1e6:8.0f} us {wb/t/1e12:5.2f} TB/s", flush=True)
