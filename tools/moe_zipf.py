"""MoE batch (configs[3]) with Zipf routing: host-offset vs device-offset calls."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2308_09723_b200 import fq
from synth import gaussian_torch, zipf_routing


def timeit(fn, reps=5):
    for _ in range(2): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


E, K, N = 64, 4096, 16384
experts = []
for e in range(E):
    W = gaussian_torch((N, K), 0.01 if e % 4 == 0 else 0.02, 7000 + e)
    if e % 4 == 0:
        W[e % N, (37 * e) % K] = 1.0
    experts.append(fq.quantize(W, 4, None))
    del W
for mbar in (4, 16, 64):
    off = zipf_routing(E, E * mbar, seed=3000)
    A = gaussian_torch((int(off[-1]), K), 1.0, 5)
    th = timeit(lambda: fq.gemm_grouped(A, [int(x) for x in off], experts))
    od = torch.from_numpy(off).cuda()
    mx = int(np.diff(off).max())
    td = timeit(lambda: fq.gemm_grouped_dev(A, od, experts, mx))
    print(f"zipf mean {mbar}: max {mx}: host offsets {th:8.1f} us, device offsets {td:8.1f} us", flush=True)
