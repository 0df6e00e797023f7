import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
from oracle import fq_oracle as O
from synth import gaussian_bits, activations_bits
from helpers import bits_to_torch, torch_to_f64
from paper_2308_09723_b200 import fq
for bits in (8, 4):
  for g in (16, 32, 64, 128):
    for M in (1, 3, 9):
        K, N = 512, 384
        Wb = gaussian_bits((N, K), 0.02, 11 + g)
        Ab = activations_bits(M, K, 21 + M)
        W = bits_to_torch(Wb, "bf16"); A = bits_to_torch(Ab, "bf16")
        qw = fq.quantize(W, bits, g)
        C = fq.gemm(A, qw, out_dtype=torch.float32); torch.cuda.synchronize()
        r = O.quantize(O.decode_bits(Wb, "bf16"), bits, g, O.BF16)
        Cr, D = O.gemm(O.decode_bits(Ab, "bf16"), r.q, r.s, g)
        e1 = O.rel_err(torch_to_f64(C), Cr, D)
        off = np.array([0, M]); Cg = fq.gemm_grouped(A, off, [qw], out_dtype=torch.float32); torch.cuda.synchronize()
        e2 = O.rel_err(torch_to_f64(Cg), Cr, D)
        print(f"bits={bits} g={g} M={M}: single {e1:.2e} grouped {e2:.2e}", flush=True)
