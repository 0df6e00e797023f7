"""MoE expert batch timing (configs[3] shape: 64 experts x [16384 x 4096] int4), g128 and adaptive
groups, M_e = 1 / 4 / 8 / 16 tokens per expert, host and device expert offsets.  A/B library builds
with FQ_LIB_PATH."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_09723_b200 import fq
from synth import gaussian_torch


def bench(fn, reps=10):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps / 1e3


E, K, N = 64, 4096, 16384
for mode in ("g128", "adaptive"):
    experts = []
    for e in range(E):
        W = gaussian_torch((N, K), 0.01 if e % 4 == 0 else 0.02, 7000 + e)
        if mode == "adaptive" and e % 4 == 0:
            W[e % N, (37 * e) % K] = 1.0
        experts.append(fq.quantize(W, 4, 128 if mode == "g128" else None)); del W
    wb = sum(q.nbytes for q in experts)
    for me in (1, 4, 8, 16):
        off = [e * me for e in range(E + 1)]
        offd = torch.tensor(off, dtype=torch.int64, device="cuda")
        A = gaussian_torch((E * me, K), 1.0, 3)
        t = bench(lambda: fq.gemm_grouped(A, off, experts))
        td = bench(lambda: fq.gemm_grouped_dev(A, offd, experts, me))
        print(f"{mode} M_e={me:2d}: host offsets {t*1e6:7.1f} us {wb/t/1e12:.2f} TB/s | device offsets {td*1e6:7.1f} us",
              flush=True)
    del experts
