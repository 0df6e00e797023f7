"""Mid-M A6 timings (diagnostics): the MoE expert batch (64 x [16384 x 4096] int4 adaptive) at
M_e = 32..256 and single OPT GEMMs at M = 48..256.  Run once per FQ_TC_BK setting (read once per
process).  usage: FQ_TC_BK=64|128 python tools/tc_mid.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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


QUICK = "quick" in sys.argv  # OPT-175B FC1 at M = 64 / 128 and the MoE batch only
tag = f"BK={os.environ.get('FQ_TC_BK', 'default')} lib={os.path.basename(os.environ.get('FQ_LIB_PATH', 'libfq.so'))}"
SHAPES = (("OPT175B-FC1", 12288, 49152),) if QUICK else (("OPT13B-FFN1", 5120, 20480), ("OPT175B-FC1", 12288, 49152),
                                                          ("OPT175B-FC2", 49152, 12288))
for name, K, N in SHAPES:
    W = gaussian_torch((N, K), 0.02, 1)
    for bits in (4, 8):
        q = fq.quantize(W, bits, 128)
        for M in ((64, 128) if QUICK else (48, 64, 128, 256, 2048)):
            A = gaussian_torch((M, K), 1.0, 2)
            C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
            t = bench(lambda: fq.gemm(A, q, out=C))
            print(f"{tag} {name} int{bits} M={M}: {t*1e6:8.1f} us {q.nbytes/t/1e12:5.2f} TB/s {2*M*K*N/t/1e12:6.0f} TF",
                  flush=True)
        del q
    del W
E, K, N = 64, 4096, 16384
experts = []
for e in range(E):
    W = gaussian_torch((N, K), 0.01 if e % 4 == 0 else 0.02, 7000 + e)
    if e % 4 == 0:
        W[e % N, (37 * e) % K] = 1.0
    experts.append(fq.quantize(W, 4, None)); del W
wb = sum(q.nbytes for q in experts)
for me in ((64, 128) if QUICK else (32, 64, 128, 256)):
    off = [e * me for e in range(E + 1)]
    A = gaussian_torch((E * me, K), 1.0, 3)
    t = bench(lambda: fq.gemm_grouped(A, off, experts))
    print(f"{tag} MoE M_e={me}: {t*1e6:8.0f} us {wb/t/1e12:5.2f} TB/s {2*E*me*K*N/t/1e12:6.0f} TF", flush=True)
