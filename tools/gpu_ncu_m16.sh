ncu --set full --import-source on --clock-control none -k regex:decode_kernel -c 2 -o gpurun_out/dec_m16_r02 python - <<'PY' > gpurun_out/ncu_m16.log 2>&1
import sys; sys.path.insert(0, ".")
import torch
from paper_2308_09723_b200 import fq
from synth import gaussian_torch
for K, N in ((12288, 49152), (49152, 12288)):
    W = gaussian_torch((N, K), 0.02, 1); q = fq.quantize(W, 4, 128); del W
    A = gaussian_torch((16, K), 1.0, 2)
    fq.gemm(A, q)
torch.cuda.synchronize()
PY
