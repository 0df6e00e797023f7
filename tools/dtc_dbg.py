import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2308_09723_b200 import fq
from synth import gaussian_torch
def bench(fn, reps=50):
    for _ in range(5): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3
K, N = 12288, 49152
W = gaussian_torch((N, K), 0.02, 1); q = fq.quantize(W, 4, 128); del W
os.environ["FQ_DECODE_TC"] = "1"
for M in (1,):
    A = gaussian_torch((M, K), 1.0, 2); C = fq.gemm(A, q)
    for dbg in (0, 1, 2, 4, 8, 1 | 2 | 4 | 8, 2 | 4 | 8, 1 | 2 | 8, 1 | 4 | 8):
        os.environ["FQ_DTC_DBG"] = str(dbg)
        print(M, dbg, f"{bench(lambda: fq.gemm(A, q, out=C)):.1f} us", flush=True)
    for sp in (1, 2, 3, 6, 12):
        os.environ["FQ_DTC_DBG"] = "0"; os.environ["FQ_GEMV_SPLITS"] = str(sp)
        print("splits", sp, f"{bench(lambda: fq.gemm(A, q, out=C)):.1f} us", flush=True)
