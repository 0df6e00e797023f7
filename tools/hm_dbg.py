"""Diagnostics: A6 two-half tiles vs the oracle on one case, per split count (env set per process)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
os.environ["FQ_GEMM_PATH"] = "tc"
from paper_2308_09723_b200 import fq
from oracle import fq_oracle as O
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from helpers import bits_to_torch, torch_to_f64
from synth import gaussian_bits, activations_bits
M, K, N, bits, group = [int(x) for x in sys.argv[1:6]]
Wb = gaussian_bits((N, K), 0.02, 1000 + M + N, "bf16"); Ab = activations_bits(M, K, 2000 + M + N, "bf16")
W = bits_to_torch(Wb, "bf16"); A = bits_to_torch(Ab, "bf16")
qw = fq.quantize(W, bits, group)
r = O.quantize(O.decode_bits(Wb, "bf16"), bits, group, O.BF16)
Cr, D = O.gemm(O.decode_bits(Ab, "bf16"), r.q, r.s, group)
for it in range(3):
    C = fq.gemm(A, qw, out_dtype=torch.float32); torch.cuda.synchronize()
    Cg = torch_to_f64(C)
    err = np.abs(Cg - Cr) / np.maximum(D, 1e-30)
    bad = err > 2e-3
    print(f"HM={os.environ.get('FQ_TC_HM','dflt')} S={os.environ.get('FQ_TC_SPLITS','dflt')} it={it} maxerr={err.max():.3g} "
          f"bad={bad.sum()}/{bad.size}", flush=True)
    if bad.any():
        toks, cols = np.nonzero(bad)
        print("  bad tokens", np.unique(toks)[:40], " bad col blocks(128)", np.unique(cols // 128))
