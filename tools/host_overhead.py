"""Host-side cost of one fq_gemm call (ctypes + argument checks + TMA descriptor encoding + launches)
against its GPU time: if the enqueue rate is slower than the GPU, back-to-back runs starve the GPU."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_09723_b200 import fq
from synth import gaussian_torch

for name, K, N in (("13B-AttnOut", 5120, 5120), ("175B-FC1", 12288, 49152)):
    W = gaussian_torch((N, K), 0.02, 1)
    q = fq.quantize(W, 4, 128); del W
    A = gaussian_torch((1, K), 1.0, 2)
    C = torch.empty(1, N, dtype=torch.bfloat16, device="cuda")
    ws = torch.zeros(fq.fq_gemm_workspace_bytes(1, q.desc), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    for label, fn in (("fq.gemm", lambda: fq.gemm(A, q, out=C)),
                      ("fq.fq_gemm", lambda: fq.fq_gemm(A, 1, q.desc, q.codes, q.scales, C, ws))):
        for _ in range(20): fn()
        torch.cuda.synchronize()
        n = 200
        t0 = time.perf_counter()
        for _ in range(n): fn()
        t_cpu = (time.perf_counter() - t0) / n * 1e6
        torch.cuda.synchronize()
        t_all = (time.perf_counter() - t0) / n * 1e6
        # graph-captured
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(10): fn()
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): g.replay()
        e1.record(); torch.cuda.synchronize()
        t_graph = e0.elapsed_time(e1) / 200 * 1e3
        print(f"{name} {label}: host enqueue {t_cpu:6.1f} us/call, wall incl. GPU {t_all:6.1f} us/call, "
              f"CUDA graph {t_graph:6.1f} us/call", flush=True)
