"""Probe: TMA streaming of a code matrix with A6-like boxes (128 rows x 32 or 64 B) through deep rings,
1 CTA per SM, no compute (diagnostics for the small-M tensor-core path)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
from probe_stream import L, bench

st = torch.cuda.current_stream().cuda_stream
for name, rows, rowbytes in (("13B-FFN2", 5120, 10240), ("175B-FC1", 49152, 6144)):
    W = torch.randint(0, 255, (rows, rowbytes), dtype=torch.uint8, device="cuda")
    nb = rows * rowbytes
    for C, S in ((32, 4), (32, 14), (64, 7), (64, 14), (128, 7)):
        best = None
        for splits in (1, 2, 4, 8, 16, 32):
            if rowbytes // C < splits: continue
            if L.probe_tma_setup(W.data_ptr(), rows, rowbytes, 128, C, 1, S, splits) != 0: continue
            us = bench(lambda: L.probe_tma_run(220 * 1024, st))
            if best is None or us < best[0]: best = (us, splits, L.probe_tma_ctas())
        us, sp, ctas = best
        print(f"{name} box=128x{C} S={S} 1cta/sm splits={sp} ctas={ctas}: {us:7.1f} us {nb/us/1e6:5.2f} TB/s", flush=True)
