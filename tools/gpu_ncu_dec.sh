set -x
./tools/hmma_probe > gpurun_out/hmma_probe.txt 2>&1
python - <<'PY' > gpurun_out/ncu_dec_run.log 2>&1
import sys; sys.path.insert(0, ".")
import torch
from paper_2308_09723_b200 import fq
from synth import gaussian_torch
for K, N in ((12288, 49152), (49152, 12288)):
    W = gaussian_torch((N, K), 0.02, 1); q = fq.quantize(W, 4, 128); del W
    for M in (1, 16):
        A = gaussian_torch((M, K), 1.0, 2)
        for _ in range(3): fq.gemm(A, q)
torch.cuda.synchronize()
PY
ncu --set full --import-source on --clock-control none -k regex:decode_kernel -c 4 -o gpurun_out/dec_r02 python - <<'PY' > gpurun_out/ncu_dec.log 2>&1
import sys; sys.path.insert(0, ".")
import torch
from paper_2308_09723_b200 import fq
from synth import gaussian_torch
for K, N in ((12288, 49152), (49152, 12288)):
    W = gaussian_torch((N, K), 0.02, 1); q = fq.quantize(W, 4, 128); del W
    for M in (1, 16):
        A = gaussian_torch((M, K), 1.0, 2)
        fq.gemm(A, q)
torch.cuda.synchronize()
PY
