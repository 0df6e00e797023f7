import sys; sys.path.insert(0, ".")
import torch
from paper_2308_09723_b200 import fq
from synth import gaussian_torch
for K, N in ((12288, 49152), (49152, 12288)):
    W = gaussian_torch((N, K), 0.02, 1); q = fq.quantize_intscale(W, 128); del W
    for M in (1, 16):
        A = gaussian_torch((M, K), 1.0, 2)
        fq.gemm_i8(A, q)
torch.cuda.synchronize()
