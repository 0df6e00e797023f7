"""The paper's own GEMM micro-benchmark (Fig. "optspeedups"): speed-up of
the fused FP16 x INT GEMM over a dense FP16 x FP16 GEMM (cuBLAS via torch.matmul) on the QKV
projection, attention output, FFN1 and FFN2 matrices of OPT-13B and OPT-30B, geometric mean over the
4 GEMMs, versus the number of activation rows.  The paper's headline: "up to 2.5X" with int4, block
size 64, on A100 for small row counts.

Each timed GEMM runs after an L2 flush (a 256 MiB write), bracketed by CUDA events on the launching
stream; weights are synthetic N(0, 0.02^2) (no checkpoints), activations N(0, 1), fp16.

    python tools/paper_microbench.py [--bits 4] [--group 64] [--rows 1 2 4 ...]
"""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

MODELS = {  # hidden size d, FFN size 4d (OPT, Zhang et al. 2022)
    "OPT-13B": 5120,
    "OPT-30B": 7168,
}
ROWS = (1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048)


def shapes(d):
    # (name, K, N) with W stored [N, K] (nn.Linear layout)
    return (("QKV", d, 3 * d), ("AttnOut", d, d), ("FFN1", d, 4 * d), ("FFN2", 4 * d, d))


def run(bits=4, group=64, rows=ROWS, reps=10, models=tuple(MODELS)):
    import torch

    from paper_2308_09723_b200 import fq
    from synth import gaussian_torch

    dev = torch.device("cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def timed(fn):
        fn()
        ts = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            ts.append((a, b))
        torch.cuda.synchronize()
        v = sorted(a.elapsed_time(b) for a, b in ts)
        return v[len(v) // 2] * 1e3  # median, us

    out = {"bits": bits, "group": group, "activation": "fp16", "baseline": "torch.matmul fp16 (cuBLAS)",
           "l2": "flushed before every timed GEMM (256 MiB write)", "models": {}}
    for m in models:
        d = MODELS[m]
        res = {M: {} for M in rows}
        for name, K, N in shapes(d):
            W = gaussian_torch((N, K), 0.02, 100 + K + N).to(torch.float16)
            q = fq.quantize(W, bits, group, scale_dtype=torch.float16)
            for M in rows:
                A = gaussian_torch((M, K), 1.0, 7 + M).to(torch.float16)
                C = torch.empty((M, N), dtype=torch.float16, device=dev)
                t_fq = timed(lambda: fq.gemm(A, q, out=C))
                t_ref = timed(lambda: torch.matmul(A, W.t()))
                res[M][name] = {"fq_us": round(t_fq, 2), "fp16_us": round(t_ref, 2),
                                "speedup": round(t_ref / t_fq, 3)}
            del W, q
        geo = {M: round(math.exp(sum(math.log(v["speedup"]) for v in res[M].values()) / len(res[M])), 3)
               for M in rows}
        out["models"][m] = {"per_gemm": {str(M): res[M] for M in rows},
                            "geomean_speedup": {str(M): geo[M] for M in rows}}
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--bits", type=int, default=4)
    ap.add_argument("--group", type=int, default=64)
    ap.add_argument("--rows", type=int, nargs="+", default=list(ROWS))
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    r = run(a.bits, a.group, tuple(a.rows), a.reps)
    for m, v in r["models"].items():
        print(m, "geomean speed-up vs fp16 by rows:", v["geomean_speedup"])
        for M, g in v["per_gemm"].items():
            print("  M=%5s " % M + "  ".join(f"{n}: {x['fq_us']:.1f}/{x['fp16_us']:.1f} us ({x['speedup']:.2f}x)"
                                            for n, x in g.items()))
    print(json.dumps(r))
