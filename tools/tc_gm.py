import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2308_09723_b200 import fq
from synth import gaussian_torch
def bench(fn, reps=3):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps / 1e3
for K, N in ((49152, 12288), (12288, 49152)):
    W = gaussian_torch((N, K), 0.02, 1)
    q = fq.quantize(W, 4, 128); del W
    for M in (2048, 8192):
        A = gaussian_torch((M, K), 1.0, 2)
        C = fq.gemm(A, q)
        for gm in (1, 2, 4, 8, 16, 32):
            os.environ["FQ_TC_GM"] = str(gm)
            t = bench(lambda: fq.gemm(A, q, out=C))
            print(f"K={K} N={N} M={M} GM={gm}: {t*1e3:.3f} ms {2*M*K*N/t/1e12:.0f} TF", flush=True)
        del A, C
