#!/usr/bin/env python
"""Benchmark of the B200-native t-product (BASELINE.json metric: t-product TFLOP/s and % of
roofline, rel. Frobenius error vs oracle).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c3]

A "step" is one full pass of the hot path (Algorithm 1: scales, forward DFTs, per-frequency
GEMMs, inverse DFT) over one t-product of the workload.  Default workload: config 3 (A 1024 x
1024 x 31, B 1024 x 512 x 31, fp32) -- the largest single-GPU configuration of BASELINE.json.
With N > 1 (torchrun, one rank per GPU) every rank owns a 512-wide lateral-slice shard of a
global B of width 512*N and the same A (broadcast once from rank 0 with NCCL, untimed); per-GPU
work is fixed ("scaling": "weak") and there is no collective in the timed region.

Metric flops (BASELINE.json / SURVEY.md 8(d)):  F = 8*n1*n2*n4*h + 2.5*n3*log2(n3)*(n1n2+n2n4+n1n4)
with h = ceil((n3+1)/2).  value = F * ranks / (max over ranks of the mean device time per step).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "c2": dict(n1=256, n2=256, n3=32, n4=256, seedA=10, seedB=11),
    "c3": dict(n1=1024, n2=1024, n3=31, n4=512, seedA=20, seedB=21),
    "c4": dict(n1=64, n2=64, n3=4096, n4=64, seedA=30, seedB=31),
    "c5": dict(n1=4096, n2=4096, n3=64, n4=8192, seedA=40, seedB=41),
}
METRIC = "t-product TFLOP/s and % of roofline (1/2/4/8 B200), rel. Frobenius err vs oracle"


def h_slices(n3):
    return n3 // 2 + 1


def metric_flops(n1, n2, n3, n4):
    """BASELINE.json flop count: 8*n1*n2*n4*h GEMM flops + 2.5*n3*log2(n3) per transformed tube."""
    tf = 2.5 * n3 * math.log2(n3) if n3 > 1 else 0.0
    return 8.0 * n1 * n2 * n4 * h_slices(n3) + tf * (n1 * n2 + n2 * n4 + n1 * n4)


def gemm_flops(n1, n2, n3, n4):
    return 8.0 * n1 * n2 * n4 * h_slices(n3)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 5 + i and r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def cpu_baseline(wl, budget_cols=96):
    """The fp64 oracle (literal Eq. (9), block-row form) on the host cores, on a bounded sample of
    the workload: C(:, J, :) for |J| = budget_cols lateral slices.  Value in the metric's unit:
    metric flops of an n1 x n2 x n3 * n2 x |J| x n3 product / oracle wall time."""
    import numpy as np
    import oracle as O
    from synth import normal
    n1, n2, n3, n4 = wl["n1"], wl["n2"], wl["n3"], wl["n4"]
    ncols = min(budget_cols, n4)
    A = normal((n1, n2, n3), wl["seedA"]).astype(np.float64)
    B = normal((n2, ncols, n3), wl["seedB"] + 7).astype(np.float64)
    t0 = time.perf_counter()
    O.tprod_columns(A, B, np.arange(ncols))
    dt = time.perf_counter() - t0
    cores = os.cpu_count()
    try:
        import threadpoolctl
        info = threadpoolctl.threadpool_info()
        cores = max((d.get("num_threads", 0) for d in info), default=cores) or cores
    except Exception:
        pass
    return {"value": metric_flops(n1, n2, n3, ncols) / dt / 1e12, "unit": "TFLOP/s", "cores": cores,
            "kind": "oracle", "seconds": dt,
            "sample": f"C(:, 0:{ncols}, :) of {n1}x{n2}x{n3} * {n2}x{ncols}x{n3} (literal Eq. (9) "
                      f"block rows, fp64 numpy/BLAS) in {dt:.2f} s"}


def run_reference(args, wl, rank, world):
    """--impl reference: the oracle as it stands, timed on the host cores (rank 0 only)."""
    if rank != 0:
        return
    import numpy as np
    import oracle as O
    from synth import normal
    n1, n2, n3, n4 = wl["n1"], wl["n2"], wl["n3"], wl["n4"]
    ncols = min(32, n4)
    A = normal((n1, n2, n3), wl["seedA"]).astype(np.float64)
    B = normal((n2, ncols, n3), wl["seedB"]).astype(np.float64)
    for _ in range(args.warmup):
        O.tprod_columns(A, B, np.arange(ncols))
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.tprod_columns(A, B, np.arange(ncols))
        ts.append(time.perf_counter() - t0)
    dt = sum(ts) / len(ts)
    val = metric_flops(n1, n2, n3, ncols) / dt / 1e12
    cores = os.cpu_count()
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "TFLOP/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic N(0,1), seeded (synth.normal)",
            "config": {"workload": args.workload, "n1": n1, "n2": n2, "n3": n3, "n4": n4,
                       "sample_n4": ncols},
            "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
                             "sample": f"each step: C(:, 0:{ncols}, :) of {n1}x{n2}x{n3} * "
                                       f"{n2}x{ncols}x{n3}, literal Eq. (9) block rows, fp64"},
            "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--engine", type=int, default=0, help="0 tcgen05 (default), 1 SIMT reference")
    ap.add_argument("--bn", type=int, default=0, help="force the GEMM N tile (0 = library heuristic)")
    ap.add_argument("--cn", type=int, default=0, help="force GEMM cluster width 1/2 (0 = heuristic)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    wl = dict(WORKLOADS[args.workload])

    if args.impl == "reference":
        run_reference(args, wl, rank, world)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1806_07247_b200 as tp
    from paper_1806_07247_b200 import build as tpbuild
    from synth import normal

    tpbuild.build()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    n1, n2, n3, n4 = wl["n1"], wl["n2"], wl["n3"], wl["n4"]
    handle = tp.Handle(local)
    handle.set_option(tp._lib.TPROD_OPT_ENGINE, args.engine)
    if args.bn:
        handle.set_option(tp._lib.TPROD_OPT_GEMM_BN, args.bn)
    if args.cn:
        handle.set_option(tp._lib.TPROD_OPT_GEMM_CLUSTER, args.cn)

    # ---- inputs: A on rank 0 then one NCCL broadcast (setup, untimed); B = this rank's shard
    A_host = torch.from_numpy(normal((n1, n2, n3), wl["seedA"])) if rank == 0 else None
    B_host = torch.from_numpy(normal((n2, n4, n3), wl["seedB"] + 1000 * rank))
    B = B_host.to(dev)
    if world > 1:
        from paper_1806_07247_b200 import dist as tpdist
        handle.set_world(rank, world, tpdist.exchange_uid(tp.nccl_unique_id))
        A = tp.matlab_empty(n1, n2, n3, torch.float32, dev)
        if rank == 0:
            A.copy_(A_host)
        tpdist.replicate(A, root=0, handle=handle)       # one ncclBroadcast, setup only
        torch.cuda.synchronize()
        if rank != 0:
            A_host = A.cpu()
    else:
        A = A_host.to(dev)
    C = tp.matlab_empty(n1, n4, n3, torch.float32, dev)
    stream = torch.cuda.current_stream(dev)

    # L2 flush between timed steps, outside the events: write a buffer of 2x L2 (evicts every
    # line of the previous step), then read a second one so the write-backs of those dirty lines
    # also complete before the next step starts (cold, clean L2).
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(max(2 * l2, 256 << 20) // 4, dtype=torch.float32, device=dev)
    flush_rd = torch.ones_like(flush)
    flush_sink = torch.empty((), dtype=torch.float32, device=dev)

    def l2_flush():
        flush.zero_()
        torch.sum(flush_rd, dim=(0,), out=flush_sink)

    def step():
        tp.tprod_f32(A, B, out=C, handle=handle, stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, per-step events, L2 flushed between steps
    handle.set_option(tp._lib.TPROD_OPT_TIMING, 1)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    stage_ms = []
    launches = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            l2_flush()
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
            launches += handle.last_launch_count()
            stage_ms.append(handle.last_stage_ms())   # waits for this step's last event
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    my_ms = sum(step_ms) / len(step_ms)
    gemm_ms = statistics.mean(s[2] for s in stage_ms)
    t = torch.tensor([my_ms, gemm_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, gemm_ms_max = float(t[0]), float(t[1])
    handle.set_option(tp._lib.TPROD_OPT_TIMING, 0)

    F = metric_flops(n1, n2, n3, n4)
    value = F * world / (ms * 1e-3) / 1e12

    # ---- e2e: the same metric through the C-ABI host entry point (pinned buffers, H2D+D2H inside)
    Ap = A_host.pin_memory() if A_host is not None else A.cpu().pin_memory()
    Ap = tp.to_matlab(Ap) if not tp.is_matlab_layout(Ap) else Ap
    Bp = B_host.pin_memory()
    Cp = tp.matlab_empty(n1, n4, n3, torch.float32, "cpu").pin_memory()
    Cp = tp.to_matlab(Cp) if not tp.is_matlab_layout(Cp) else Cp
    for _ in range(2):
        tp.tprod_f32_host(Ap, Bp, out=Cp, handle=handle, stream=stream)
    e2e_steps = max(3, min(args.steps, 10))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        tp.tprod_f32_host(Ap, Bp, out=Cp, handle=handle, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1) / e2e_steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_val = F * world / (float(e2e_ms) * 1e-3) / 1e12

    # ---- parity spot check of the timed output (sampled lateral slices vs the oracle)
    parity = None
    if rank == 0 and args.workload in ("c2", "c3"):
        import oracle as O
        J = np.array([0, 1, n4 // 2, n4 - 1])
        ref = O.tprod_columns(A_host.numpy(), B_host.numpy(), J)
        parity = O.rel_err(C[:, torch.from_numpy(J).to(dev), :].cpu().numpy(), ref)

    if rank == 0:
        peaks, src = load_peaks()
        peak_alg = peaks["bf16_tflops"] / 3.0
        gflops = gemm_flops(n1, n2, n3, n4)
        achieved = gflops / (gemm_ms_max * 1e-3) / 1e12
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic N(0,1), seeded (synth.normal, PCG64)",
            "config": {"workload": args.workload, "n1": n1, "n2": n2, "n3": n3, "n4_per_gpu": n4,
                       "h": h_slices(n3), "global_n4": n4 * world,
                       "parallelism": f"lateral-slice shards x{world}, A broadcast once (NCCL)",
                       "l2": "flushed between timed steps (write 2x L2 then read 2x L2, outside the step events)",
                       "engine": "tcgen05" if args.engine == 0 else "simt-reference"},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_alg,
                         "unit": "TFLOP/s", "frac": achieved / peak_alg, "traffic": None,
                         "kernel": "K2 per-frequency complex GEMM",
                         "note": (f"peak = {src} bf16 burst {peaks['bf16_tflops']} / 3: an fp32-accurate "
                                  "product costs 3 fp16 tensor-core products (hi*hi+hi*lo+lo*hi)"),
                         "gemm_ms": gemm_ms_max,
                         "stage_ms": [round(statistics.mean(s[i] for s in stage_ms), 5) for i in range(4)]},
            "e2e": {"value": e2e_val, "unit": "TFLOP/s",
                    "h2d_bytes_per_step": 4 * (n1 * n2 * n3 + n2 * n4 * n3),
                    "d2h_bytes_per_step": 4 * n1 * n4 * n3},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "parity_rel_err_sampled": parity,
        }
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(wl)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    handle.close()


if __name__ == "__main__":
    main()
