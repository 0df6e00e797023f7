#!/usr/bin/env python
"""Benchmark of the FineQuant hot path on B200 (contract: one JSON line from rank 0).

Workload (BASELINE.json configs[1]): OPT-175B decode-layer GEMMs, int4 group 128, bf16
activations: FC1 W[N=49152, K=12288] and FC2 W[N=12288, K=49152].  One STEP = the config's whole
decode sweep: for each M in {1, 2, 4, 8, 16}, C = A[M,K] . dequant(Wq)^T for FC1 and FC2 (10 fused
GEMM launches, kernels A4/A5).  metric = effective weight bytes (codes + scales, the bytes the
method must move) per second, whole job.  Weights are 2 x 311 MB (> 126 MB L2), so
no L2 flush is needed between launches.

N > 1 (torchrun): every rank runs the same sweep on its own weights (independent replicas, the
paper's per-node replication model P:194, "scaling": "weak"); the decode GEMM itself has no
data-path collective.  Time = max over ranks of the CUDA-event time of the K timed steps.

--impl reference: the CPU oracle (oracle/) timed on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FC1 = (12288, 49152)   # (K, N)
FC2 = (49152, 12288)
M_SWEEP = (1, 2, 4, 8, 16)
BITS, GROUP = 4, 128
METRIC = "int4xbf16 decode GEMM effective weight TB/s (OPT-175B FC1+FC2, M=1..16 sweep, g=128)"
UNIT = "TB/s"


def eff_bytes(K, N, bits, group):
    """Algorithmic bytes per GEMM launch: packed codes + scales (bf16)."""
    return K * N * bits // 8 + (K // group) * N * 2


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained"), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


# ------------------------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.index), "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------ CPU oracle
def cpu_oracle_sample(target_s: float = 10.0):
    """Time the oracle (as it stands) on a bounded column sample of the same sweep.
    Returns (TB/s-equivalent of effective weight bytes, seconds, threads, description)."""
    from oracle import fq_oracle as O
    from synth import activations_bits, gaussian_bits
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        threads = os.cpu_count()
    cols = 256
    prep = []
    for (K, N), seed in ((FC1, 1), (FC2, 2)):
        W = O.decode_bits(gaussian_bits((cols, K), 0.02, 1000 + seed), "bf16")
        r = O.quantize(W, BITS, GROUP, O.BF16)
        As = {M: O.decode_bits(activations_bits(M, K, 2000 + M), "bf16") for M in M_SWEEP}
        prep.append((K, N, r, As))

    def one_pass():
        nbytes = 0
        for K, N, r, As in prep:
            for M in M_SWEEP:
                O.gemm(As[M], r.q, r.s, GROUP)
                nbytes += eff_bytes(K, cols, BITS, GROUP)
        return nbytes

    t0 = time.perf_counter()
    nb = one_pass()
    dt = time.perf_counter() - t0
    reps = max(1, int(target_s / max(dt, 1e-3)))
    t0 = time.perf_counter()
    nb = 0
    for _ in range(reps):
        nb += one_pass()
    dt = time.perf_counter() - t0
    desc = (f"oracle gemm (fp64 dequant + matmul) over {cols} sampled output columns of FC1 and FC2, "
            f"M in {list(M_SWEEP)}, x{reps} passes, weights pre-quantized by the oracle")
    return nb / dt / 1e12, dt, threads, desc


# ------------------------------------------------------------------------------------ main arms
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    v, dt, threads, desc = cpu_oracle_sample(target_s=max(2.0, 10.0 / max(1, args.steps)))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": "opt175b_decode_fc1_fc2_int4_g128_sweep_M1-16", "sample": desc},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": desc},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="fq", choices=["fq", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    from paper_2308_09723_b200 import fq
    from synth import gaussian_torch

    peaks = load_peaks()
    # ---- weights (quantized once, outside the timed region: the quantizer is offline)
    mats = []
    for (K, N), mid in ((FC1, 1), (FC2, 2)):
        W = gaussian_torch((N, K), 0.02, 1000 + mid + 100 * rank, device=dev)
        qw = fq.quantize(W, BITS, GROUP)
        del W
        mats.append(qw)
    torch.cuda.synchronize()
    acts = {}
    for (K, N), qw in zip((FC1, FC2), mats):
        for M in M_SWEEP:
            acts[(K, M)] = gaussian_torch((M, K), 1.0, 2000 + M, device=dev)
    outs = {(qw.K, M): torch.empty((M, qw.N), dtype=torch.bfloat16, device=dev) for qw in mats for M in M_SWEEP}
    wss = {}
    for qw in mats:
        for M in M_SWEEP:
            nb = fq.fq_gemm_workspace_bytes(M, qw.desc)
            wss[(qw.K, M)] = torch.zeros(max(nb, 256), dtype=torch.uint8, device=dev)
    launches = [(qw, M) for qw in mats for M in M_SWEEP]
    step_bytes = sum(eff_bytes(qw.K, qw.N, BITS, GROUP) for qw, M in launches)
    stream = torch.cuda.current_stream()

    def launch(qw, M):
        fq.fq_gemm(acts[(qw.K, M)], M, qw.desc, qw.codes, qw.scales, outs[(qw.K, M)], wss[(qw.K, M)], stream)

    def step():
        for qw, M in launches:
            launch(qw, M)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    # ---- timed region (device time, CUDA events on the launching stream)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in launches]
    per_launch_ms = np.zeros(len(launches))
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            step()
        t1.record(stream)
        torch.cuda.synchronize()
        total_ms = t0.elapsed_time(t1)
        # per-launch durations (same launches, bracketed individually) for the roofline
        for _ in range(max(1, args.steps // 10)):
            for i, (qw, M) in enumerate(launches):
                ev[i][0].record(stream)
                launch(qw, M)
                ev[i][1].record(stream)
            torch.cuda.synchronize()
            per_launch_ms += np.array([a.elapsed_time(b) for a, b in ev])
        per_launch_ms /= max(1, args.steps // 10)
        if world > 1:
            dist.barrier()
    clocks = clk.summary()
    t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = world * step_bytes * args.steps / (total_ms / 1e3) / 1e12

    # ---- e2e through the public API: pinned host A -> device, fused GEMM, C -> pinned host
    h_acts = {k: v.cpu().pin_memory() for k, v in acts.items()}
    h_outs = {k: torch.empty(v.shape, dtype=v.dtype).pin_memory() for k, v in outs.items()}
    d_acts = {k: torch.empty_like(v) for k, v in acts.items()}
    h2d = sum(v.numel() * 2 for v in h_acts.values())
    d2h = sum(v.numel() * 2 for v in h_outs.values())

    def e2e_step():
        for qw, M in launches:
            k = (qw.K, M)
            d_acts[k].copy_(h_acts[k], non_blocking=True)
            fq.gemm(d_acts[k], qw, out=outs[k])
            h_outs[k].copy_(outs[k], non_blocking=True)

    for _ in range(3):
        e2e_step()
    torch.cuda.synchronize()
    e_steps = max(10, args.steps // 3)
    t0.record(stream)
    for _ in range(e_steps):
        e2e_step()
    t1.record(stream)
    torch.cuda.synchronize()
    e_ms = t0.elapsed_time(t1)
    te = torch.tensor([e_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = world * step_bytes * e_steps / (float(te.item()) / 1e3) / 1e12

    # ---- roofline of the dominant kernel (the A4 decode GEMM; it is every launch of the step)
    gemv_s = per_launch_ms.sum() / 1e3
    achieved_gbs = step_bytes / gemv_s / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get("decode_bytes_per_step")
    roof = {"bound": "hbm", "achieved": round(achieved_gbs, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": round(achieved_gbs / peaks["hbm_gbs"], 4), "traffic": traffic,
            "peak_source": peaks["source"], "kernel": "fq::gemv_kernel (A4/A5)",
            "per_launch_us": {f"{'FC1' if qw.K == FC1[0] else 'FC2'}_M{M}": round(x * 1e3, 2)
                              for (qw, M), x in zip(launches, per_launch_ms)}}

    extras = {}
    if rank == 0 and not args.no_extras:
        extras = measure_extras(fq, dev, peaks)

    line = {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "opt175b_decode_fc1_fc2_int4_g128_sweep_M1-16",
                       "shapes": {"FC1": {"K": FC1[0], "N": FC1[1]}, "FC2": {"K": FC2[0], "N": FC2[1]}},
                       "M": list(M_SWEEP), "bits": BITS, "group": GROUP,
                       "l2": "inputs larger than L2 (2 x 311 MB packed weights), no flush",
                       "parallelism": f"replicas x{world}"},
            "clocks": clocks, "e2e": {"value": round(e2e_value, 4), "unit": UNIT,
                                      "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": len(launches) * args.steps, "roofline": roof}
    if extras:
        line["extras"] = extras
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, dt, threads, desc = cpu_oracle_sample(10.0)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": desc,
                                "seconds": round(dt, 2)}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def measure_extras(fq, dev, peaks):
    """Secondary paths reported next to the headline: int8 decode, the large-M GEMM, the quantizer."""
    import torch
    from synth import gaussian_torch
    out = {}

    def timeit(fn, reps=20):
        for _ in range(3):
            fn()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / reps / 1e3

    K, N = FC1
    W = gaussian_torch((N, K), 0.02, 1001, device=dev)
    # quantizer (A3), bf16 W -> int4 g128: bytes = read 2B/w + write codes+scales
    t = timeit(lambda: fq.quantize(W, 4, 128), 5)
    qb = K * N * 2 + eff_bytes(K, N, 4, 128)
    out["quantize_int4_g128_FC1"] = {"us": round(t * 1e6, 1), "GB_s": round(qb / t / 1e9, 1),
                                     "frac_hbm": round(qb / t / 1e9 / peaks["hbm_gbs"], 3)}
    t = timeit(lambda: fq.adapt_group(W, 500, 16), 3)
    out["adapt_flags_FC1"] = {"us": round(t * 1e6, 1), "GB_s": round(K * N * 2 / t / 1e9, 1)}
    q8 = fq.quantize(W, 8, 128)
    for M in (1, 16):
        A = gaussian_torch((M, K), 1.0, 7, device=dev)
        t = timeit(lambda: fq.gemm(A, q8))
        b = eff_bytes(K, N, 8, 128)
        out[f"decode_int8_FC1_M{M}"] = {"us": round(t * 1e6, 1), "TB_s": round(b / t / 1e12, 3)}
    q4 = fq.quantize(W, 4, 128)
    del W
    for M in (2048,):
        A = gaussian_torch((M, K), 1.0, 8, device=dev)
        t = timeit(lambda: fq.gemm(A, q4), 3)
        fl = 2.0 * M * K * N
        out[f"prefill_int4_FC1_M{M}"] = {"ms": round(t * 1e3, 3), "TFLOP_s": round(fl / t / 1e12, 1),
                                         "frac_bf16_peak": round(fl / t / 1e12 / peaks["bf16_tflops"], 3)}
        Wb = gaussian_torch((N, K), 0.02, 1001, device=dev)
        tb = timeit(lambda: torch.matmul(A, Wb.t()), 3)
        out[f"torch_matmul_bf16_FC1_M{M}"] = {"ms": round(tb * 1e3, 3), "TFLOP_s": round(fl / tb / 1e12, 1)}
        del Wb
    return out


if __name__ == "__main__":
    sys.exit(main())
