#!/usr/bin/env python
"""Benchmark of the FineQuant hot path on B200 (contract: one JSON line from rank 0).

Workload (BASELINE.json configs[1]): OPT-175B decode-layer GEMMs, int4 group 128, bf16
activations: FC1 W[N=49152, K=12288] and FC2 W[N=12288, K=49152].  One STEP = the config's whole
decode sweep: for each M in {1, 2, 4, 8, 16}: Y = X[M,K] . dequant(Wq_FC1)^T, Z = Y . dequant(Wq_FC2)^T
(10 fused GEMM launches, kernels A4/A5).  metric = effective weight bytes (codes + scales, the bytes the
method must move) per second, whole job.  Weights are 2 x 311 MB (> 126 MB L2), so
no L2 flush is needed between launches.

N > 1 (torchrun, configs[4]): the same two matrices are tensor-parallel over the N ranks - FC1
column-parallel (N sharded), FC2 row-parallel (K sharded) with an NCCL all-reduce of its fp32
partial output, the exchange the paper names.  Total work is fixed ("scaling": "strong");
value = the whole job's effective weight bytes per second.  Time = max over ranks of the
CUDA-event time of the K timed steps.

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

# fq_gemm on the decode path launches fq::prep_acts_kernel (activation pre-conversion, M x K
# elements) + fq::decode_kernel (A4/A5, split-K fixup fused)
LAUNCHES_PER_GEMM = 2

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
def nproc() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_oracle_sample(target_s: float = 10.0, bits: int = 4, group: int = 128):
    """Time the oracle (as it stands) on a bounded column sample of the same sweep, its BLAS
    threaded over every host core (nproc).
    Returns (TB/s-equivalent of effective weight bytes, seconds, threads, description)."""
    from oracle import fq_oracle as O
    from synth import activations_bits, gaussian_bits
    threads = nproc()
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(threads)
    except Exception:
        pass
    BITS, GROUP = bits, group
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
    v, dt, threads, desc = cpu_oracle_sample(target_s=max(2.0, 10.0 / max(1, args.steps)), bits=args.bits,
                                             group=args.group)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"opt175b_decode_fc1_fc2_int{BITS}_g{GROUP}_sweep_M1-16", "sample": desc},
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
    ap.add_argument("--no-tp-layer", action="store_true")
    ap.add_argument("--xr-layer", action="store_true",
                    help="N>1: also time the TP layer with the fused GEMM + one-shot all-reduce (NEXT-1)")
    # SURVEY §5 knobs: headline GEMM precision / group; adaptive parameters of the MoE extras
    ap.add_argument("--bits", type=int, default=4, choices=[4, 8])
    ap.add_argument("--group", type=int, default=128)
    ap.add_argument("--alpha", type=int, default=500, help="adaptive alpha in thousandths (MoE extras)")
    ap.add_argument("--min-group", type=int, default=16, help="adaptive minimum group (MoE extras)")
    ap.add_argument("--seed", type=int, default=1000, help="base seed of the synthetic weights")
    args = ap.parse_args()
    global BITS, GROUP, METRIC
    BITS, GROUP = args.bits, args.group
    METRIC = (f"int{BITS}xbf16 decode GEMM effective weight TB/s (OPT-175B FC1+FC2, M=1..16 sweep, g={GROUP})")
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # FQ_BENCH_ONE_GPU=1 (diagnostics only): every rank on cuda:0 with the gloo backend, so the
    # N > 1 code path (shards, row-parallel all-reduce, max-over-ranks timing) can be exercised on a
    # one-GPU box; its numbers are not bench values.
    one_gpu = os.environ.get("FQ_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    from paper_2308_09723_b200 import fq
    from paper_2308_09723_b200.tp import shard_bounds, check_row_group
    from synth import gaussian_torch

    peaks = load_peaks()
    t = world
    # ---- weights: every rank derives its shard from the same global matrices (seeded), then
    # quantizes it (offline, outside the timed region).  FC1 column-parallel (N sharded),
    # FC2 row-parallel (K sharded, group | K/t) -> partial outputs all-reduced over NCCL.
    c0, c1 = shard_bounds(FC1[1], t, rank)
    r0, r1 = shard_bounds(FC2[0], t, rank, 32)
    check_row_group(FC2[0], t, GROUP)
    W1 = gaussian_torch((FC1[1], FC1[0]), 0.02, args.seed + 1, device=dev)
    q1 = fq.quantize(W1[c0:c1].contiguous(), BITS, GROUP)
    del W1
    W2 = gaussian_torch((FC2[1], FC2[0]), 0.02, args.seed + 2, device=dev)
    q2 = fq.quantize(W2[:, r0:r1].contiguous(), BITS, GROUP)
    del W2
    torch.cuda.synchronize()
    xs = {M: gaussian_torch((M, FC1[0]), 1.0, 2000 + M, device=dev) for M in M_SWEEP}
    ys = {M: torch.empty((M, q1.N), dtype=torch.bfloat16, device=dev) for M in M_SWEEP}
    zs = {M: torch.empty((M, q2.N), dtype=torch.float32 if t > 1 else torch.bfloat16, device=dev)
          for M in M_SWEEP}
    ws = {}
    for q in (q1, q2):
        for M in M_SWEEP:
            ws[(q.K, M)] = torch.zeros(max(fq.fq_gemm_workspace_bytes(M, q.desc), 256), dtype=torch.uint8,
                                       device=dev)
    # algorithmic bytes: full FC1 + full FC2 per M (sum over ranks' shards)
    step_bytes_total = len(M_SWEEP) * (eff_bytes(*FC1, BITS, GROUP) + eff_bytes(*FC2, BITS, GROUP))
    step_bytes_rank = len(M_SWEEP) * (q1.nbytes + q2.nbytes)
    stream = torch.cuda.current_stream()

    def gemm1(M, st=None):
        fq.fq_gemm(xs[M], M, q1.desc, q1.codes, q1.scales, ys[M], ws[(q1.K, M)], st or stream)

    def gemm2(M, st=None):
        fq.fq_gemm(ys[M], M, q2.desc, q2.codes, q2.scales, zs[M], ws[(q2.K, M)], st or stream)

    def reduce(M):
        if t > 1:
            dist.all_reduce(zs[M], op=dist.ReduceOp.SUM)

    def step(st=None):
        for M in M_SWEEP:
            gemm1(M, st)
            gemm2(M, st)
            reduce(M)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    # ---- timed region: CUDA events on the launching stream, barrier + sync on both sides
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        total_ms = e0.elapsed_time(e1)
        if world > 1:
            dist.barrier()
        # per-launch durations: each launch of the step repeated R times back to back between one
        # pair of CUDA events on the launching stream (steady state, PDL overlap included)
        # Three rounds; each launch's figure is the median of its three round averages, so one
        # transient (a power-cap clock dip, a neighbour's interference) cannot skew the roofline.
        names = [f"FC1_M{M}" for M in M_SWEEP] + [f"FC2_M{M}" for M in M_SWEEP]
        rounds = {n: [] for n in names}
        comms = []
        reps = 20
        for _ in range(3):
            evs = []
            for M in M_SWEEP:
                for n, fn in ((f"FC1_M{M}", gemm1), (f"FC2_M{M}", gemm2), (f"AR_M{M}", reduce)):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    for _ in range(reps):
                        fn(M)
                    b.record(stream)
                    evs.append((n, a, b))
            torch.cuda.synchronize()
            c = 0.0
            for n, a, b in evs:
                if n.startswith("AR"):
                    c += a.elapsed_time(b) / reps
                else:
                    rounds[n].append(a.elapsed_time(b) / reps)
            comms.append(c)
        per = {n: sorted(v)[1] for n, v in rounds.items()}
        comm = sorted(comms)[1]
        if world > 1:
            dist.barrier()
    clocks = clk.summary()
    tt = torch.tensor([total_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    total_ms = float(tt.item())
    ms_per_step = total_ms / args.steps
    value = step_bytes_total * args.steps / (total_ms / 1e3) / 1e12

    # ---- the same step captured once in a CUDA graph and replayed (the API is graph-safe: no host
    # sync, self-resetting workspace counters, PDL edges kept): host enqueue cost leaves the step
    graph_ms = None
    if world == 1:
        try:
            g = torch.cuda.CUDAGraph()
            cs = torch.cuda.Stream(device=dev)
            cs.wait_stream(stream)
            with torch.cuda.stream(cs):
                step(cs)  # warm the TMA-descriptor cache on the capture stream
                with torch.cuda.graph(g, stream=cs):
                    step(cs)
            stream.wait_stream(cs)
            for _ in range(3):
                g.replay()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(args.steps):
                g.replay()
            b.record(stream)
            torch.cuda.synchronize()
            graph_ms = a.elapsed_time(b) / args.steps
        except Exception as e:  # report, keep the eager numbers
            graph_ms = f"capture failed: {str(e)[:120]}"

    # ---- e2e through the public API: pinned host x -> device, FC1 -> FC2 (-> all-reduce),
    # result -> pinned host, every step.
    h_x = {M: xs[M].cpu().pin_memory() for M in M_SWEEP}
    h_z = {M: torch.empty(zs[M].shape, dtype=zs[M].dtype).pin_memory() for M in M_SWEEP}
    d_x = {M: torch.empty_like(xs[M]) for M in M_SWEEP}
    h2d = sum(v.numel() * v.element_size() for v in h_x.values())
    d2h = sum(v.numel() * v.element_size() for v in h_z.values())

    # Host <-> device traffic on its own stream (a serving loop overlaps its input upload and
    # result download with compute): every input of the step is uploaded up front, each GEMM
    # pair waits only for its own input, each result is downloaded as soon as it is ready.
    copy_stream = torch.cuda.Stream(device=dev)
    up_ev = {M: torch.cuda.Event() for M in M_SWEEP}
    done_ev = {M: torch.cuda.Event() for M in M_SWEEP}

    def e2e_step():
        copy_stream.wait_stream(stream)  # previous step's results are consumed in order
        with torch.cuda.stream(copy_stream):
            for M in M_SWEEP:
                d_x[M].copy_(h_x[M], non_blocking=True)
                up_ev[M].record(copy_stream)
        for M in M_SWEEP:
            stream.wait_event(up_ev[M])
            y = fq.gemm(d_x[M], q1, out=ys[M])
            fq.gemm(y, q2, out=zs[M])
            reduce(M)
            done_ev[M].record(stream)
            with torch.cuda.stream(copy_stream):
                copy_stream.wait_event(done_ev[M])
                h_z[M].copy_(zs[M], non_blocking=True)
        stream.wait_stream(copy_stream)  # the step ends when its results are on the host

    for _ in range(3):
        e2e_step()
    torch.cuda.synchronize()
    e_steps = max(10, args.steps // 3)
    if world > 1:
        dist.barrier()
    e0.record(stream)
    for _ in range(e_steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    te = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = step_bytes_total * e_steps / (float(te.item()) / 1e3) / 1e12

    # ---- roofline of the dominant kernel (A4 decode GEMM = every GEMM launch of the step)
    gemv_s = sum(per.values()) / 1e3
    achieved_gbs = step_bytes_rank / gemv_s / 1e9
    # DRAM traffic per launch of the dominant kernel from the committed ncu --set full capture
    # (FC1, M=1): compare with the algorithmic bytes of the same launch (311,427,072).
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f)
        d1 = tj.get("decode_fc1_m1")
        if d1:
            traffic = d1["dram_bytes_read"] + d1["dram_bytes_write"]
            traffic_src = "bytes per launch, FC1 M=1, " + tj.get("source", "")
    roof = {"bound": "hbm", "achieved": round(achieved_gbs, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": round(achieved_gbs / peaks["hbm_gbs"], 4), "traffic": traffic, "traffic_source": traffic_src,
            "peak_source": peaks["source"], "kernel": "fq::decode_kernel (A4/A5) + its fq::prep_acts_kernel (bracketed together)",
            "algorithmic_bytes_per_step_per_rank": step_bytes_rank,
            "per_launch_us": {n: round(v * 1e3, 2) for n, v in per.items()},
            "allreduce_us_per_step": round(comm * 1e3, 2)}

    # ---- configs[4]: the full OPT-175B layer under TP (every N, all ranks): QKV col, out row + AR,
    # FC1 col, FC2 row + AR; 4 distinct layers rotated; layer time and all-reduce share per M.
    del xs, ys, zs, d_x, h_x
    q1 = q2 = None
    torch.cuda.empty_cache()
    tp_layer = None
    if not args.no_tp_layer:
        tp_layer = measure_tp_layer(fq, dev, world, rank, args)

    extras = {}
    if rank == 0 and world == 1 and not args.no_extras:
        extras = measure_extras(fq, dev, peaks, args)
        try:
            extras.update(hbm_read_probe(dev))
        except Exception as e:  # nvcc / probe unavailable: the line still prints
            extras["hbm_read_probe_error"] = str(e)[:200]

    line = {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"opt175b_decode_fc1_fc2_int{BITS}_g{GROUP}_sweep_M1-16",
                       "shapes": {"FC1": {"K": FC1[0], "N": FC1[1]}, "FC2": {"K": FC2[0], "N": FC2[1]}},
                       "M": list(M_SWEEP), "bits": BITS, "group": GROUP,
                       "l2": "inputs larger than L2 (2 x 311 MB packed weights at N=1), no flush",
                       "parallelism": f"tp{world} (FC1 column-parallel, FC2 row-parallel + NCCL all-reduce)"},
            "clocks": clocks, "e2e": {"value": round(e2e_value, 4), "unit": UNIT,
                                      "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": LAUNCHES_PER_GEMM * 2 * len(M_SWEEP) * args.steps, "roofline": roof}
    if graph_ms is not None:
        line["cuda_graph_step"] = ({"ms_per_step": round(graph_ms, 4),
                                    "TB_s": round(step_bytes_total / (graph_ms / 1e3) / 1e12, 4)}
                                   if isinstance(graph_ms, float) else {"error": graph_ms})
    if tp_layer:
        line["tp_layer"] = tp_layer
    if extras:
        line["extras"] = extras
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, dt, threads, desc = cpu_oracle_sample(10.0, BITS, GROUP)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": desc,
                                "seconds": round(dt, 2)}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def measure_tp_layer(fq, dev, world, rank, args, n_layers=4, Ms=(1, 16, 2048), reps=10):
    """configs[4]: one OPT-175B decoder layer's GEMM chain under tensor parallelism (tp.TPOptLayer):
    QKV [3h, h] column-parallel -> out-proj [h, h] row-parallel + all-reduce -> FC1 [4h, h]
    column-parallel -> FC2 [h, 4h] row-parallel + all-reduce, int4 g128, h = 12288.  Four
    distinct layers rotated (> L2 at every t).  layer_us = CUDA-event time per layer (max over
    ranks); comm_us = the layer's two all-reduces timed alone on the same stream; comm_frac =
    comm_us / layer_us; TB_s = the whole layer's effective weight bytes (all shards) / layer time."""
    import torch
    import torch.distributed as dist
    from paper_2308_09723_b200.tp import ShardSpec, TPLinearFQ, TPOptLayer, shard_bounds
    from synth import gaussian_torch
    h = 12288
    shapes = dict(qkv=(3 * h, h, "col"), out=(h, h, "row"), fc1=(4 * h, h, "col"), fc2=(h, 4 * h, "row"))
    pg = dist.group.WORLD if world > 1 else None
    layers = []
    full_bytes = 0
    for li in range(n_layers):
        lin = {}
        for j, (name, (n, k, kind)) in enumerate(shapes.items()):
            W = gaussian_torch((n, k), 0.02, args.seed + 100 * li + j, device=dev)
            if kind == "col":
                lo, hi = shard_bounds(n, world, rank)
                Ws = W[lo:hi].contiguous()
            else:
                lo, hi = shard_bounds(k, world, rank, 32)
                Ws = W[:, lo:hi].contiguous()
            del W
            lin[name] = TPLinearFQ(Ws, ShardSpec(kind, k, n, world, rank), 4, 128, process_group=pg)
            del Ws
            full_bytes += eff_bytes(k, n, 4, 128) if li == 0 else 0
        layers.append(TPOptLayer(lin["qkv"], lin["out"], lin["fc1"], lin["fc2"], process_group=pg))
    # the same layers with the row-parallel decode GEMMs fused with a one-shot all-reduce over NVLink
    # peer memory (NEXT-1), on one-rank-per-GPU NCCL groups only
    # Opt-in (--xr-layer): the fused path is verified on one GPU (all ranks on one device,
    # tests/test_gpu_xr.py) but has never run on a multi-GPU box, and a failure there (a trapped wait
    # kernel) would cost the whole scaling line.
    fused_ok = world > 1 and args.xr_layer and os.environ.get("FQ_BENCH_ONE_GPU") != "1"
    flayers = [TPOptLayer(L.qkv, L.out, L.fc1, L.fc2, process_group=pg, fused=True) for L in layers] if fused_ok else []
    torch.cuda.empty_cache()
    stream = torch.cuda.current_stream()
    out = {"layers": n_layers, "h": h, "bits": 4, "group": 128, "tp": world,
           "weight_bytes_per_layer_all_ranks": full_bytes,
           "weight_bytes_per_layer_per_rank": sum(l.weight_bytes for l in layers) // n_layers}
    for M in Ms:
        x = gaussian_torch((M, h), 1.0, 2000 + M, device=dev)
        parts = [torch.empty((M, h), dtype=torch.float32, device=dev) for _ in range(2)]

        def chain():
            for L in layers:
                L.forward(x)

        def comms():
            for _ in layers:
                for t_ in parts:
                    dist.all_reduce(t_, op=dist.ReduceOp.SUM, group=pg)

        for _ in range(2):
            chain()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            chain()
        b.record(stream)
        torch.cuda.synchronize()
        lay = a.elapsed_time(b) / (reps * n_layers) * 1e3
        com = 0.0
        if world > 1:
            comms()
            torch.cuda.synchronize()
            dist.barrier()
            a.record(stream)
            for _ in range(reps):
                comms()
            b.record(stream)
            torch.cuda.synchronize()
            com = a.elapsed_time(b) / (reps * n_layers) * 1e3
        tt = torch.tensor([lay, com], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        lay, com = float(tt[0]), float(tt[1])
        ent = {"layer_us": round(lay, 1), "comm_us": round(com, 1), "comm_frac": round(com / lay, 3),
               "TB_s": round(full_bytes / (lay * 1e-6) / 1e12, 3)}
        if flayers and M <= 16:
            try:
                for _ in range(2):
                    for L in flayers:
                        L.forward(x)
                torch.cuda.synchronize()
                dist.barrier()
                a.record(stream)
                for _ in range(reps):
                    for L in flayers:
                        L.forward(x)
                b.record(stream)
                torch.cuda.synchronize()
                fl_us = torch.tensor([a.elapsed_time(b) / (reps * n_layers) * 1e3], device=dev, dtype=torch.float64)
                dist.all_reduce(fl_us, op=dist.ReduceOp.MAX)
                ent["fused_allreduce_layer_us"] = round(float(fl_us), 1)
                ent["fused_allreduce_TB_s"] = round(full_bytes / (float(fl_us) * 1e-6) / 1e12, 3)
            except Exception as e:  # symmetric memory unavailable on this box: report, keep the NCCL numbers
                ent["fused_allreduce_error"] = str(e)[:200]
        if M >= 256:
            fl = 2.0 * M * full_bytes / (0.5 + 2 / 128)  # 2 M FLOP per weight (full layer)
            ent["TFLOP_s"] = round(fl / (lay * 1e-6) / 1e12, 1)
        out[f"M={M}"] = ent
        del x, parts
    del layers
    torch.cuda.empty_cache()
    return out


def measure_extras(fq, dev, peaks, args):
    """Secondary paths reported next to the headline (rank 0, N=1): int8 decode, the tcgen05
    prefill GEMM (configs[2]) against torch.matmul bf16, the quantizer and adaptive pass, and the
    MoE expert batch (configs[3])."""
    import torch
    from synth import gaussian_torch, gaussian_with_outliers_bits
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

    for name, (K, N) in (("FC1", FC1), ("FC2", FC2)):
        W = gaussian_torch((N, K), 0.02, 1001, device=dev)
        if name == "FC1":
            # quantizer (A3): read 2 B/weight + write codes/scales; adaptive flags (A1): read 2 B/w
            tq = timeit(lambda: fq.quantize(W, 4, 128), 5)
            qb = K * N * 2 + eff_bytes(K, N, 4, 128)
            out["quantize_int4_g128_FC1"] = {"us": round(tq * 1e6, 1), "GB_s": round(qb / tq / 1e9, 1),
                                             "frac_hbm": round(qb / tq / 1e9 / peaks["hbm_gbs"], 3)}
            ta = timeit(lambda: fq.adapt_group(W, 500, 16), 3)
            out["adapt_flags_FC1"] = {"us": round(ta * 1e6, 1), "GB_s": round(K * N * 2 / ta / 1e9, 1),
                                      "frac_hbm": round(K * N * 2 / ta / 1e9 / peaks["hbm_gbs"], 3)}
        q8 = fq.quantize(W, 8, 128)
        for M in (1, 16):
            A = gaussian_torch((M, K), 1.0, 7, device=dev)
            tt = timeit(lambda: fq.gemm(A, q8))
            b = eff_bytes(K, N, 8, 128)
            out[f"decode_int8_{name}_M{M}"] = {"us": round(tt * 1e6, 1), "TB_s": round(b / tt / 1e12, 3),
                                               "frac_hbm": round(b / tt / 1e9 / peaks["hbm_gbs"], 3)}
        del W, q8
        torch.cuda.empty_cache()

    def prefill_extras():
        for name, (K, N) in (("FC1", FC1), ("FC2", FC2)):
            W = gaussian_torch((N, K), 0.02, 1001, device=dev)
            q8 = fq.quantize(W, 8, 128)
            q4 = fq.quantize(W, 4, 128)
            for M in (2048, 4096, 8192):
                A = gaussian_torch((M, K), 1.0, 8, device=dev)
                fl = 2.0 * M * K * N
                for bits, q in ((4, q4), (8, q8)):
                    tt = timeit(lambda: fq.gemm(A, q), 3)
                    out[f"prefill_int{bits}_{name}_M{M}"] = {
                        "ms": round(tt * 1e3, 3), "TFLOP_s": round(fl / tt / 1e12, 1),
                        "frac_bf16_peak": round(fl / tt / 1e12 / peaks["bf16_tflops"], 3),
                        # the sustained (power-capped, back-to-back) bf16 figure, when measured
                        "frac_bf16_sustained": (round(fl / tt / 1e12 / peaks["bf16_tflops_sustained"], 3)
                                                if peaks.get("bf16_tflops_sustained") else None)}
                if M == 2048:
                    tb = timeit(lambda: torch.matmul(A, W.t()), 3)
                    out[f"torch_matmul_bf16_{name}_M{M}"] = {"ms": round(tb * 1e3, 3),
                                                             "TFLOP_s": round(fl / tb / 1e12, 1)}
                del A
            del W, q4, q8
            torch.cuda.empty_cache()

    # The bandwidth-bound decode and MoE timings run before the compute-bound prefill ones: the
    # prefill GEMMs drive the GPU into its power cap, which would otherwise bleed into the next
    # timings (measured: FC2 int8 decode 113 us after the quantizer, 150 us after prefill).
    # MoE expert batch (configs[3]): 64 experts [16384, 4096], int4 adaptive (alpha 0.5, min 16),
    # outliers planted in experts e % 4 == 0 -> g_e in {16, 4096}; uniform M_e sweep.
    E, K, N = 64, 4096, 16384
    experts = []
    for e in range(E):
        W = gaussian_torch((N, K), 0.01 if e % 4 == 0 else 0.02, 7000 + e, device=dev)
        if e % 4 == 0:
            W[e % N, (37 * e) % K] = 1.0
        experts.append(fq.quantize(W, 4, None, alpha_milli=args.alpha, min_group=args.min_group))
        del W
    torch.cuda.empty_cache()
    gh = {}
    for q in experts:
        gh[q.group] = gh.get(q.group, 0) + 1
    wbytes = sum(q.nbytes for q in experts)
    moe = {"group_histogram": {str(k): v for k, v in sorted(gh.items())}, "weight_bytes": wbytes}
    for me in (1, 4, 16, 64, 256):
        off = [e * me for e in range(E + 1)]
        A = gaussian_torch((E * me, K), 1.0, 3000 + me, device=dev)
        tt = timeit(lambda: fq.gemm_grouped(A, off, experts), 5)
        fl = 2.0 * E * me * K * N
        moe[f"M_e={me}"] = {"us": round(tt * 1e6, 1), "TB_s": round(wbytes / tt / 1e12, 3),
                            "frac_hbm": round(wbytes / tt / 1e9 / peaks["hbm_gbs"], 3),
                            "TFLOP_s": round(fl / tt / 1e12, 1)}
        del A
    # Zipf(1) skewed routing with the same totals (seed 3000): host offsets and the
    # device-offset call (fq_gemm_grouped_dev, token bound = the largest expert) next to each other
    from synth import zipf_routing
    for mbar in (16, 64):
        off = zipf_routing(E, E * mbar, seed=3000)
        cnt = np.diff(off)
        A = gaussian_torch((int(off[-1]), K), 1.0, 3100 + mbar, device=dev)
        tt = timeit(lambda: fq.gemm_grouped(A, [int(x) for x in off], experts), 5)
        off_dev = torch.from_numpy(off).to(dev)
        mx = int(cnt.max())
        td = timeit(lambda: fq.gemm_grouped_dev(A, off_dev, experts, mx), 5)
        fl = 2.0 * int(off[-1]) * K * N
        moe[f"zipf_mean_M_e={mbar}"] = {"M_e_min": int(cnt.min()), "M_e_median": float(np.median(cnt)),
                                       "M_e_max": mx, "empty_experts": int((cnt == 0).sum()),
                                       "us": round(tt * 1e6, 1), "TB_s": round(wbytes / tt / 1e12, 3),
                                       "TFLOP_s": round(fl / tt / 1e12, 1),
                                       "device_offsets_us": round(td * 1e6, 1)}
        del A
    out["moe_64x16384x4096_int4_adaptive"] = moe
    del experts
    torch.cuda.empty_cache()

    # ---- the paper's own kernel benchmark: speed-up over a dense
    # FP16 x FP16 GEMM (cuBLAS via torch.matmul) on OPT-13B / OPT-30B QKV, attention-out, FFN1,
    # FFN2, geometric mean over the 4 GEMMs; int4, block size 64 as in the paper (and 128), fp16
    # activations, L2 flushed before every timed GEMM.  The paper reports "up to 2.5X" on A100.
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import paper_microbench as PM
    pm = {}
    for g in (64, 128):
        r = PM.run(bits=4, group=g, rows=(1, 8, 16, 64, 256, 2048), reps=5)
        pm[f"int4_g{g}"] = {m: v["geomean_speedup"] for m, v in r["models"].items()}
    pm["baseline"] = "torch.matmul fp16 (cuBLAS), L2 flushed per GEMM; geomean of QKV/AttnOut/FFN1/FFN2 speed-ups by rows"
    pm["paper_a100"] = "up to 2.5x (int4, block 64, small row counts; figure data not in the text, P:189/P:308)"
    out["paper_microbench_opt13b_opt30b"] = pm
    out.update(next_rows_extras(fq, dev, peaks, timeit))
    out.update(xr_one_gpu_extras(fq, dev, timeit))
    prefill_extras()
    out.update(dequant_cublas_extras(fq, dev, peaks, timeit))
    return out


def hbm_read_probe(dev):
    """Read-only HBM probe in the same run: 16-byte LDG sweep over one OPT-175B
    FC matrix's worth of codes (302 MB) and over 2 GiB (tools/probe_stream.cu, built on demand)."""
    import ctypes
    import subprocess
    import torch
    so = os.path.join(ROOT, "tools", "libprobe_stream.so")
    if not os.path.exists(so):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                               "-fPIC", "-o", so, os.path.join(ROOT, "tools", "probe_stream.cu")])
    L = ctypes.CDLL(so)
    L.probe_ldg.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                            ctypes.c_void_p]
    st = torch.cuda.current_stream().cuda_stream
    sink = torch.zeros(4, dtype=torch.int32, device=dev)
    big = torch.randint(0, 255, (2 * 1024 ** 3,), dtype=torch.uint8, device=dev)
    res = {}
    for name, nbytes in (("302MB", 12288 * 49152 // 2), ("2GiB", 2 * 1024 ** 3)):
        best = []
        for cps in (2, 4):
            def fn():
                L.probe_ldg(ctypes.c_void_p(big.data_ptr()), nbytes, 148 * cps, 512, ctypes.c_void_p(sink.data_ptr()),
                            ctypes.c_void_p(st))
            for _ in range(3):
                fn()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                fn()
            b.record()
            torch.cuda.synchronize()
            best.append(nbytes / (a.elapsed_time(b) / 20 / 1e3) / 1e9)
        res[name] = round(max(best), 1)
    del big
    torch.cuda.empty_cache()
    return {"hbm_read_probe_GB_s": res}


def next_rows_extras(fq, dev, peaks, timeit):
    """SURVEY NEXT-3 / NEXT-4 at OPT-175B shapes: int3 / int2 decode (the canonical bit stream) and
    the int8-activation x int4-weight path with integer group scales (tcgen05 kind::i8), next to
    the bf16 path of the same matrices."""
    import torch
    from synth import gaussian_torch
    out = {}
    for name, (K, N) in (("FC1", FC1), ("FC2", FC2)):
        W = gaussian_torch((N, K), 0.02, 1001, device=dev)
        for bits in (3, 2):
            q = fq.quantize(W, bits, 128)
            for M in (1, 16):
                A = gaussian_torch((M, K), 1.0, 7, device=dev)
                tt = timeit(lambda: fq.gemm(A, q))
                out[f"decode_int{bits}_{name}_M{M}"] = {"us": round(tt * 1e6, 1), "TB_s": round(q.nbytes / tt / 1e12, 3)}
            del q
        qi = fq.quantize_intscale(W, 128)
        for M in (1, 16, 64, 256, 2048):
            A = gaussian_torch((M, K), 1.0, 8, device=dev)
            acts = fq.quantize_acts_i8(A)
            C = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
            tg = timeit(lambda: fq.gemm_i8(None, qi, out=C, acts=acts))
            tq = timeit(lambda: fq.quantize_acts_i8(A))
            fl = 2.0 * M * K * N
            ent = {"gemm_us": round(tg * 1e6, 1), "act_quant_us": round(tq * 1e6, 1),
                   "TB_s": round(qi.nbytes / tg / 1e12, 3), "TOPS": round(fl / tg / 1e12, 1)}
            if M >= 256:  # int8 dense peak = 2 x the measured bf16 peak (B200_PROFILING.md nominal ratio)
                ent["frac_int8_peak"] = round(fl / tg / 1e12 / (2 * peaks["bf16_tflops"]), 3)
            out[f"int8act_int4w_{name}_M{M}"] = ent
            del A, acts, C
        del W, qi
        torch.cuda.empty_cache()
    return out


def xr_one_gpu_extras(fq, dev, timeit):
    """NEXT-1 on one GPU: the fused row-parallel GEMM + one-shot all-reduce with every rank of an
    8-way group on this device (its pushes are local writes, so no NVLink latency is in these
    numbers): per-rank time of the OPT-175B FC2 shard GEMM [12288 x 6144] plain vs with the fused
    epilogue, and the group's completion waits."""
    import torch
    from synth import gaussian_torch
    K, N, world = 49152, 12288, 8
    Ks = K // world
    W = gaussian_torch((N, K), 0.02, 1001, device=dev)
    qs = [fq.quantize(W[:, r * Ks:(r + 1) * Ks].contiguous(), 4, 128) for r in range(world)]
    del W
    out = {"world": world, "shard": [N, Ks], "note": "all ranks on one GPU; pushes are local writes"}
    for M in (1, 16):
        A = gaussian_torch((M, K), 1.0, 9, device=dev)
        As = [A[:, r * Ks:(r + 1) * Ks].contiguous() for r in range(world)]
        d = qs[0].desc
        ranks = fq.xr_group_local(world, M, d, torch.bfloat16, device=dev)
        nb = fq.fq_gemm_workspace_bytes_ex(M, d, fq.make_opts("decode"))
        wss = [torch.zeros(max(nb, 256), dtype=torch.uint8, device=dev) for _ in range(world)]
        C = torch.empty((M, N), dtype=torch.float32, device=dev)

        def plain():
            for r in range(world):
                fq.gemm(As[r], qs[r], out=C, opts=fq.make_opts("decode"))

        def fused():
            for r, R in enumerate(ranks):
                fq.fq_gemm_allreduce(As[r], M, d, qs[r].codes, qs[r].scales, fq.FQ_BF16, R.peers, R.peers_dev, wss[r])
            for R in ranks:
                fq.fq_xr_wait(R.peers, M, d)

        tp_, tf = timeit(plain, 10), timeit(fused, 10)
        out[f"M={M}"] = {"plain_gemm_us_per_rank": round(tp_ * 1e6 / world, 2),
                         "fused_gemm_allreduce_us_per_rank": round(tf * 1e6 / world, 2)}
        del A, As, ranks, wss
    torch.cuda.empty_cache()
    return {"xr_fused_allreduce_one_gpu": out}


def dequant_cublas_extras(fq, dev, peaks, timeit):
    """The naive alternative to the fused kernel at prefill: dequantize the int4
    codes to a bf16 matrix (torch ops) and call cuBLAS (torch.matmul); times of both steps."""
    import torch
    from synth import gaussian_torch
    out = {}
    for name, (K, N) in (("FC1", FC1), ("FC2", FC2)):
        W = gaussian_torch((N, K), 0.02, 1001, device=dev)
        q = fq.quantize(W, 4, 128)
        del W
        A = gaussian_torch((2048, K), 1.0, 8, device=dev)

        def dequant():
            c = q.codes
            lo = (c & 0xF).to(torch.int16)
            hi = (c >> 4).to(torch.int16)
            qq = torch.stack((lo - ((lo & 8) << 1), hi - ((hi & 8) << 1)), dim=2).view(N, K)
            return (qq.to(torch.bfloat16).view(N, K // 128, 128) * q.scales.t().unsqueeze(2)).view(N, K)

        Wd = dequant()
        td = timeit(dequant, 3)
        tm = timeit(lambda: torch.matmul(A, Wd.t()), 3)
        tf = timeit(lambda: fq.gemm(A, q), 3)
        fl = 2.0 * 2048 * K * N
        out[f"prefill_dequant_cublas_{name}_M2048"] = {
            "dequant_ms": round(td * 1e3, 3), "matmul_ms": round(tm * 1e3, 3),
            "total_ms": round((td + tm) * 1e3, 3), "fused_ms": round(tf * 1e3, 3),
            "fused_TFLOP_s": round(fl / tf / 1e12, 1), "dequant_cublas_TFLOP_s": round(fl / (td + tm) / 1e12, 1)}
        del A, Wd, q
        torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    sys.exit(main())
