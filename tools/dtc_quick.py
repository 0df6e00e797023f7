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
for M in (1, 16):
    A = gaussian_torch((M, K), 1.0, 2); C = fq.gemm(A, q)
    for env in ({"FQ_DECODE_TC": "0"}, {"FQ_DECODE_TC": "1"}, {"FQ_DECODE_TC": "1", "FQ_DTC_NOFENCE": "1"}):
        for k in ("FQ_DECODE_TC", "FQ_DTC_NOFENCE"): os.environ.pop(k, None)
        os.environ.update(env)
        print(M, env, f"{bench(lambda: fq.gemm(A, q, out=C)):.1f} us", flush=True)
os.environ["FQ_GEMM_PATH"] = "tc"
for M in (2048,):
    A = gaussian_torch((M, K), 1.0, 2); C = fq.gemm(A, q)
    t = bench(lambda: fq.gemm(A, q, out=C), 5)
    print("prefill", M, f"{t:.1f} us {2*M*K*N/t/1e6:.1f} TFLOP/s", flush=True)
