"""Why does bench.py's per-launch time differ from tools/dec_sweep.py for the same GEMM?  Times FC1 M=1
through (a) the bench's low-level fq_gemm with its own zero-filled workspace and explicit stream,
(b) fq.gemm (global workspace), (c) the low-level call with the global workspace."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_09723_b200 import fq
from synth import gaussian_torch

K, N, M = 12288, 49152, 1
W = gaussian_torch((N, K), 0.02, 1001)
q = fq.quantize(W, 4, 128); del W
x = gaussian_torch((M, K), 1.0, 2001)
y = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
st = torch.cuda.current_stream()
ws_own = torch.zeros(max(fq.fq_gemm_workspace_bytes(M, q.desc), 256), dtype=torch.uint8, device="cuda")
d = q.desc
variants = {
    "bench-style (own ws, explicit stream)": lambda: fq.fq_gemm(x, M, q.desc, q.codes, q.scales, y, ws_own, st),
    "fq.gemm (global ws)": lambda: fq.gemm(x, q, out=y),
    "low-level, global ws": lambda: fq.fq_gemm(x, M, d, q.codes, q.scales, y, fq.workspace(fq.fq_gemm_workspace_bytes(M, d), x.device)),
    "bench-style, cached desc": lambda: fq.fq_gemm(x, M, d, q.codes, q.scales, y, ws_own, st),
}
for rep in range(2):
    for name, fn in variants.items():
        for _ in range(10): fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record(st)
        for _ in range(30): fn()
        b.record(st)
        tc = (time.perf_counter() - t0) / 30 * 1e6
        torch.cuda.synchronize()
        print(f"{name:40s}: {a.elapsed_time(b) / 30 * 1e3:6.1f} us/launch (host {tc:5.1f} us/call)", flush=True)
