"""Launch the quantizer (A3) and the adaptive pass (A1) on OPT-175B FC1 a few times (ncu driver)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_09723_b200 import fq
from synth import gaussian_torch
W = gaussian_torch((49152, 12288), 0.02, 1)
for _ in range(3):
    fq.quantize(W, 4, 128)
    fq.adapt_group(W, 500, 16)
torch.cuda.synchronize()
