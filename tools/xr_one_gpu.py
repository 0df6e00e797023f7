"""NEXT-1 on one GPU (bench.xr_one_gpu_extras): fused GEMM + one-shot all-reduce with 8 ranks on one device."""
import sys, os, torch
sys.path.insert(0, os.getcwd())
import bench
from paper_2308_09723_b200 import fq
def timeit(fn, reps=20):
    for _ in range(3): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps / 1e3
print(bench.xr_one_gpu_extras(fq, torch.device("cuda", 0), timeit))
