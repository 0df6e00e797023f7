"""Quick correctness + timing check of the tcgen05 prefill path (run under `timeout`)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2308_09723_b200 import fq
from synth import gaussian_torch
from oracle import fq_oracle as O

os.environ["FQ_GEMM_PATH"] = "tc"

def check(M, K, N, bits, group, dt=torch.bfloat16):
    W = gaussian_torch((N, K), 0.02, 11, dtype=dt)
    A = gaussian_torch((M, K), 1.0, 12, dtype=dt)
    qw = fq.quantize(W, bits, group, scale_dtype=dt)
    C = fq.gemm(A, qw)
    torch.cuda.synchronize()
    cols = np.arange(0, N, max(1, N // 64))
    rows = np.arange(0, M, max(1, M // 48))
    Wc = W[torch.from_numpy(cols).cuda()].float().cpu().double().numpy()
    r = O.quantize(Wc, bits, group, O.BF16 if dt == torch.bfloat16 else O.FP16)
    Cr, D = O.gemm(A[torch.from_numpy(rows).cuda()].float().cpu().double().numpy(), r.q, r.s, group)
    err = O.rel_err(C.double().cpu().numpy()[np.ix_(rows, cols)], Cr, D)
    print(f"M={M} K={K} N={N} bits={bits} g={group} {dt}: rel_err={err:.2e}", flush=True)
    return err

check(256, 256, 256, 4, 64)
check(256, 1024, 384, 4, 128)
check(300, 1024, 384, 8, 128)
check(512, 2048, 1024, 4, 32, torch.float16)

def bench(M, K, N, bits=4, reps=5):
    W = gaussian_torch((N, K), 0.02, 1)
    qw = fq.quantize(W, bits, 128); del W
    A = gaussian_torch((M, K), 1.0, 2)
    C = fq.gemm(A, qw)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fq.gemm(A, qw, out=C)
    e.record(); torch.cuda.synchronize()
    t = s.elapsed_time(e) / reps / 1e3
    print(f"bench M={M} K={K} N={N} int{bits}: {t*1e3:.3f} ms  {2*M*K*N/t/1e12:.1f} TFLOP/s", flush=True)

bench(2048, 12288, 49152)
bench(2048, 49152, 12288)
bench(4096, 12288, 49152)
bench(2048, 12288, 49152, 8)
