"""Diagnostics (FQ_DIAG build): per-CTA timeline of one decode launch (OPT-175B FC1 / FC2 int4 g128).

    FQ_LIB_PATH=.../libfq_diag.so python tools/dec_timeline.py --M 1 [--splits S]
Prints, per shape: kernel span, CTA count, median fill latency (start -> first stage landed), main
loop and epilogue durations, idle gaps between consecutive CTAs of an SM, and how busy the SMs' CTA
slots were over the span."""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2308_09723_b200 import fq
from synth import gaussian_torch

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, nargs="+", default=[1])
ap.add_argument("--splits", type=int, default=0)
ap.add_argument("--shapes", nargs="+", default=["FC1", "FC2"])
a = ap.parse_args()
lib = ctypes.CDLL(fq.LIB_PATH)
lib.fq_diag_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
SH = {"FC1": (12288, 49152), "FC2": (49152, 12288)}


def pct(x, q):
    return float(np.percentile(x, q)) / 1e3


for name in a.shapes:
    K, N = SH[name]
    W = gaussian_torch((N, K), 0.02, 1)
    q = fq.quantize(W, 4, 128)
    del W
    for M in a.M:
        A = gaussian_torch((M, K), 1.0, 2)
        C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        o = fq.make_opts("decode", a.splits) if a.splits else None
        for _ in range(20):
            fq.gemm(A, q, out=C, opts=o)
        torch.cuda.synchronize()
        buf = np.zeros((4096, 8), dtype=np.uint64)
        assert lib.fq_diag_timeline(buf.ctypes.data, 4096, 1) == 0
        for _ in range(3):  # the last of three back-to-back launches (PDL overlap as in a real step)
            fq.gemm(A, q, out=C, opts=o)
        torch.cuda.synchronize()
        assert lib.fq_diag_timeline(buf.ctypes.data, 4096, 0) == 0
        n = int((buf[:, 1] > 0).sum())
        t = buf[:n].astype(np.int64)
        sm, t0, tf, tl, te, tg, tp0, tp1 = (t[:, j] for j in range(8))
        base = t0.min()
        nst_pre = 3
        w1 = (t0 - base) < 1000
        for lab, msk in (("wave1", w1), ("later", ~w1)):
            if msk.sum() == 0:
                continue
            print(f"  {lab}: producer start {pct((tp0 - t0)[msk], 50):.2f} us after CTA start, first {min(nst_pre, 9)} issues"
                  f" {pct((tp1 - tp0)[msk], 50):.2f} us (p90 {pct((tp1 - tp0)[msk], 90):.2f}), griddep_wait {pct((tg - tp1)[msk], 50):.2f} us")
            print(f"  {lab}: {int(msk.sum())} CTAs; start->griddep {pct((tg - t0)[msk], 50):.2f} us,"
                  f" griddep->first stage {pct((tf - tg)[msk], 50):.2f} (p90 {pct((tf - tg)[msk], 90):.2f}) us,"
                  f" loop {pct((tl - tf)[msk], 50):.1f} us, epilogue {pct((te - tl)[msk], 50):.2f} us")
        span = te.max() - base
        print(f"{name} M={M}: {n} CTAs, span {span / 1e3:.1f} us (start spread {pct(t0 - base, 100):.1f} us)")
        print(f"  fill (start->first stage) median {pct(tf - t0, 50):.2f} p90 {pct(tf - t0, 90):.2f} us;"
              f" loop median {pct(tl - tf, 50):.1f} p10 {pct(tl - tf, 10):.1f} p90 {pct(tl - tf, 90):.1f} us;"
              f" epilogue median {pct(te - tl, 50):.2f} p90 {pct(te - tl, 90):.2f} max {pct(te - tl, 100):.2f} us")
        gaps, busy = [], 0
        for s_ in np.unique(sm):
            idx = np.where(sm == s_)[0]
            ev = sorted([(t0[i], te[i]) for i in idx])
            busy += sum(e - b for b, e in ev)
            # pair CTAs of this SM by slot: a CTA that starts after another ended reuses its slot
            ends = sorted(e for _, e in ev)
            starts = sorted(b for b, _ in ev)
            late = [b for b in starts if b - base > 1000]
            for b in late:
                prev = max([e for e in ends if e <= b], default=None)
                if prev is not None:
                    gaps.append(b - prev)
        nsm = len(np.unique(sm))
        print(f"  SMs {nsm}, CTA-slot occupancy {busy / (2 * nsm * span):.3f} of 2 slots x span;"
              f" refill gaps median {pct(gaps, 50) if gaps else 0:.2f} us (n={len(gaps)})")
        # end-time distribution: how ragged is the finish
        print(f"  last CTA ends: p50 {pct(te - base, 50):.1f} p90 {pct(te - base, 90):.1f} max {pct(te - base, 100):.1f} us;"
              f" first-wave ends p10 {pct(np.sort(te - base)[: min(n, 296)], 10):.1f} max {pct(np.sort(te - base)[: min(n, 296)], 100):.1f} us")
        if os.environ.get("TL_DETAIL"):
            loop = (tl - tf) / 1e3
            gx = (N + 255) // 256
            cta = np.arange(n)
            by = (cta // gx)
            print("  loop us by split index:", " ".join(f"{s_}:{np.median(loop[by == s_]):.1f}" for s_ in np.unique(by)[:12]))
            order = np.argsort(sm)
            bands = np.array_split(order, 8)
            print("  loop us by SM-id band (8 bands):", " ".join(f"{np.median(loop[b]):.1f}" for b in bands))
            print("  loop us by SM parity:", f"{np.median(loop[sm % 2 == 0]):.1f} {np.median(loop[sm % 2 == 1]):.1f}")
            fast = loop < np.median(loop)
            print("  first-stage latency (griddep->first) fast half vs slow half:",
                  f"{np.median(((tf - tg) / 1e3)[fast]):.2f} {np.median(((tf - tg) / 1e3)[~fast]):.2f}")
            print("  sorted SM ids of the slowest 20 CTAs:", sorted(sm[np.argsort(loop)[-20:]].tolist()))
