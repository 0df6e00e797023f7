"""GPU time per call of the whole int8-activation path (fq.gemm_i8 = per-token activation quantizer +
GEMM) and of the bf16 path (fq.gemm = prep + decode), each captured 20x back to back in a CUDA graph
(no host overhead), OPT-175B FC1 / FC2, decode sizes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_09723_b200 import fq
from synth import gaussian_torch

R = 20
for name, (K, N) in (("FC1", (12288, 49152)), ("FC2", (49152, 12288))):
    W = gaussian_torch((N, K), 0.02, 1)
    qi = fq.quantize_intscale(W, 128)
    qb = fq.quantize(W, 4, 128)
    del W
    for M in (1, 8, 16):
        A = gaussian_torch((M, K), 1.0, 2)
        res = {}
        for lab, fn in (("int8-act", lambda: fq.gemm_i8(A, qi)), ("bf16", lambda: fq.gemm(A, qb))):
            fn(); torch.cuda.synchronize()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                fn()
                with torch.cuda.graph(g, stream=s):
                    for _ in range(R):
                        fn()
            torch.cuda.current_stream().wait_stream(s)
            g.replay(); torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(5):
                g.replay()
            b.record(); torch.cuda.synchronize()
            res[lab] = a.elapsed_time(b) / (5 * R) * 1e3
        print(f"{name} M={M:2d}: int8-act path {res['int8-act']:6.1f} us/call | bf16 path {res['bf16']:6.1f} us/call", flush=True)
