"""Quick check + timing of the tcgen05 decode kernel vs the mma.sync one (run under timeout)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2308_09723_b200 import fq
from synth import gaussian_torch
from oracle import fq_oracle as O

def bench(fn, reps=50):
    for _ in range(5): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3

for K, N in ((4096, 1024), (12288, 49152), (49152, 12288)):
    W = gaussian_torch((N, K), 0.02, 1)
    for bits in (4, 8):
        q = fq.quantize(W, bits, 128)
        for M in (1, 4, 16):
            A = gaussian_torch((M, K), 1.0, 2)
            res = {}
            for impl in ("1", "0"):
                os.environ["FQ_DECODE_TC"] = impl
                C = fq.gemm(A, q); torch.cuda.synchronize()
                cols = np.arange(0, N, max(1, N // 32))
                r = O.quantize(W[torch.from_numpy(cols).cuda()].float().cpu().double().numpy(), bits, 128, O.BF16)
                Cr, D = O.gemm(A.float().cpu().double().numpy(), r.q, r.s, 128)
                err = O.rel_err(C.double().cpu().numpy()[:, cols], Cr, D)
                us = bench(lambda: fq.gemm(A, q, out=C))
                res[impl] = (us, q.nbytes / us / 1e6, err)
            print(f"K={K} N={N} int{bits} M={M}: tc {res['1'][0]:7.1f}us {res['1'][1]:5.2f}TB/s err {res['1'][2]:.1e} | mma {res['0'][0]:7.1f}us {res['0'][1]:5.2f}TB/s err {res['0'][2]:.1e}", flush=True)
    del W
