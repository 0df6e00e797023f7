import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2308_09723_b200 import fq
from synth import gaussian_torch
def bench(fn, reps=5):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps / 1e3
E, K, N = 64, 4096, 16384
experts = []
for e in range(E):
    W = gaussian_torch((N, K), 0.01 if e % 4 == 0 else 0.02, 7000 + e)
    if e % 4 == 0: W[e % N, (37 * e) % K] = 1.0
    experts.append(fq.quantize(W, 4, None)); del W
wb = sum(q.nbytes for q in experts)
print("groups", sorted(set(q.group for q in experts)), "bytes", wb)
for me in (1, 4, 8, 16, 32, 64, 128, 256):
    off = [e * me for e in range(E + 1)]
    A = gaussian_torch((E * me, K), 1.0, 3)
    for dtc in ("0", "1"):
        os.environ["FQ_DECODE_TC"] = dtc
        t = bench(lambda: fq.gemm_grouped(A, off, experts))
        print(f"M_e={me} decode_tc={dtc}: {t*1e6:.0f} us {wb/t/1e12:.2f} TB/s {2*E*me*K*N/t/1e12:.0f} TF", flush=True)
