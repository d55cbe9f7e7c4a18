#!/usr/bin/env python
"""Benchmark of the B200-native t-product (BASELINE.json metric: "t-product TFLOP/s and % of
roofline (1/2/4/8 B200), rel. Frobenius err vs oracle").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c5]

A "step" is one full pass of the hot path (Algorithm 1: operand scales,
forward DFTs of A and B, the h per-frequency complex GEMMs, the fused conjugate fill + inverse
DFT) over one t-product of the workload.

Default workload: config 5 of BASELINE.json -- A 4096 x 4096 x 64, B 4096 x 8192 x 64, fp32 --
the configuration the metric's "1/2/4/8 B200" is quoted on, and at N = 1 the largest configuration
that fits one GPU.  The global problem is fixed ("scaling": "strong"): with N ranks (torchrun, one
per GPU) rank r owns the contiguous lateral-slice block r of B and C (synth.lateral_shard) and the
same A, broadcast once from rank 0 with the library's NCCL broadcast (setup, untimed).  Lateral
slices are independent (Eq. (9)), so the timed region has no collective.
At N = 1 the line also carries configs 3 (the north star's >= 60 %-of-roofline target config), 4
and 2 as the extra keys "c3", "c4", "c2", measured with the same protocol.

Metric flops (BASELINE.json / SURVEY.md 8(d)):  F = 8*n1*n2*n4*h + 2.5*n3*log2(n3)*(n1n2+n2n4+n1n4)
with h = ceil((n3+1)/2).  value = F / (max over ranks of the mean device time per step).
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
    """Flops the K2 stage performs: the DC slice (and the Nyquist slice for even n3) of real inputs
    is real (Eq. (8)), so it is one real product (2 n1 n2 n4) instead of a complex one
    (8 n1 n2 n4); the metric's formula counts every slice as complex (R11)."""
    r = 1 + (1 if n3 % 2 == 0 and n3 >= 2 else 0)
    return 8.0 * n1 * n2 * n4 * (h_slices(n3) - r) + 2.0 * n1 * n2 * n4 * r


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    # /opt/skills/guides/B200_PROFILING.md fallback
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def load_traffic(workload):
    """DRAM bytes per launch of the GEMM kernel from the committed `ncu --set full` capture of this
    workload (profiles/*_<workload>_gemm_ncu.json), or None."""
    import glob
    best = None
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", f"*_{workload}_gemm_ncu.json"))):
        try:
            with open(p) as f:
                d = json.load(f)
            best = float(d["dram_read_bytes"]) + float(d["dram_write_bytes"])
        except Exception:
            pass
    return best


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
            self._stop.wait(0.05)

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


# ----------------------------------------------------------------------------- CPU oracle legs
def _cores():
    cores = os.cpu_count()
    try:
        import threadpoolctl
        info = threadpoolctl.threadpool_info()
        cores = max((d.get("num_threads", 0) for d in info), default=cores) or cores
    except Exception:
        pass
    return cores


def oracle_sample(wl, A64, B, ncols, nslices):
    """One bounded sample of the workload through the oracle as it stands (literal Eq. (9),
    block-row form, fp64 numpy/BLAS): C(:, J, T) for |J| = ncols lateral slices (the first ncols
    columns of B) and |T| = nslices frontal slices.  Returns (seconds, metric flops credited =
    F * |J||T| / (n4 n3), description)."""
    import numpy as np
    import oracle as O
    n1, n2, n3, n4 = wl["n1"], wl["n2"], wl["n3"], wl["n4"]
    B = B[:, :ncols, :]
    T = np.arange(nslices)
    t0 = time.perf_counter()
    O.tprod_blockrow(A64, B, T, np.arange(ncols))
    dt = time.perf_counter() - t0
    F = metric_flops(n1, n2, n3, n4) * (ncols * nslices) / (n4 * n3)
    desc = (f"C(:, 0:{ncols}, 0:{nslices}) of the {n1}x{n2}x{n3} * {n2}x{n4}x{n3} workload "
            f"(literal Eq. (9) block rows, fp64 numpy/BLAS), credited {ncols * nslices}/{n4 * n3} "
            f"of the metric flops")
    return dt, F, desc


def sample_size(wl, A64, B, budget_s):
    """(|J|, |T|) for a CPU sample of roughly budget_s seconds: |J| = 16 lateral slices, and as
    many frontal slices as fit the budget after timing one block row of the oracle."""
    n3, n4 = wl["n3"], wl["n4"]
    ncols = min(n4, 16)
    dt1, _, _ = oracle_sample(wl, A64, B, ncols, 1)
    return ncols, int(max(1, min(n3, budget_s / max(dt1, 1e-6))))


def cpu_baseline(wl, A_f32, B_cols, budget_s=15.0):
    import numpy as np
    A64 = np.asarray(A_f32, dtype=np.float64)
    ncols, nslices = sample_size(wl, A64, B_cols, budget_s)
    dt, F, desc = oracle_sample(wl, A64, B_cols, ncols, nslices)
    return {"value": F / dt / 1e12, "unit": "TFLOP/s", "cores": _cores(), "kind": "oracle",
            "seconds": dt, "sample": desc + f" in {dt:.2f} s"}


def run_reference(args, wl, rank, world):
    """--impl reference: the oracle as it stands, timed on the host cores (rank 0 only), one
    bounded sample of the same workload per step."""
    if rank != 0:
        return
    import numpy as np
    from synth import normal
    A64 = normal((wl["n1"], wl["n2"], wl["n3"]), wl["seedA"]).astype(np.float64)
    # the sample's lateral slices of B (a timing sample: drawn directly, not from B's full stream)
    B = normal((wl["n2"], min(16, wl["n4"]), wl["n3"]), wl["seedB"])
    ncols, nslices = sample_size(wl, A64, B, 3.0)
    for _ in range(args.warmup):
        oracle_sample(wl, A64, B, ncols, nslices)
    ts, F, desc = [], 0.0, ""
    for _ in range(args.steps):
        dt, F, desc = oracle_sample(wl, A64, B, ncols, nslices)
        ts.append(dt)
    dt = sum(ts) / len(ts)
    val = F / dt / 1e12
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "TFLOP/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic N(0,1), seeded (synth.normal, PCG64)",
            "config": {"workload": args.workload, "n1": wl["n1"], "n2": wl["n2"], "n3": wl["n3"],
                       "n4": wl["n4"], "sample_cols": ncols, "sample_slices": nslices},
            "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": _cores(), "kind": "oracle",
                             "sample": "each step: " + desc},
            "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def _allmax(dist, world, vals, dev):
    """Max over ranks of a list of floats (the job's time is the slowest rank's).  NCCL reduces a
    device tensor; gloo (the multi-rank test on one GPU) a host tensor."""
    import torch
    if world == 1:
        return [float(v) for v in vals]
    on_dev = dist.get_backend() == "nccl"
    t = torch.tensor([float(v) for v in vals], dtype=torch.float64, device=dev if on_dev else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.cpu()]


def stage_bytes(n1, n2, n3, n4):
    """Algorithmic bytes of the memory-bound stages: K0 reads A and B once (4 B per
    element); K1 reads a tube (4 n3 B) and writes its Hermitian half as 4 fp16 planes (8 h B); K3
    reads a C-bar tube (re, im fp32: 8 h B) and writes the real tube (4 n3 B)."""
    h = h_slices(n3)
    return {"K0": 4.0 * n3 * (n1 * n2 + n2 * n4),
            "K1": (4.0 * n3 + 8.0 * h) * (n1 * n2 + n2 * n4),
            "K3": (8.0 * h + 4.0 * n3) * (n1 * n4)}


def time_workload(tp, torch, dist, handle, wl, args, rank, world, local, dev, stream, label):
    """Set up one workload (global n4 sharded over the ranks), time K steps on the device and
    end to end; returns a dict of measurements (timings are the max over ranks)."""
    import numpy as np
    from synth import lateral_shard, normal, normal_lateral
    n1, n2, n3, n4g = wl["n1"], wl["n2"], wl["n3"], wl["n4"]
    j0, j1 = lateral_shard(n4g, world, rank)
    n4 = j1 - j0

    # ---- inputs: A on rank 0 then one broadcast (setup, untimed); B = this rank's shard
    A_host = torch.from_numpy(normal((n1, n2, n3), wl["seedA"])) if rank == 0 else None
    if world == 1:
        B_np = normal((n2, n4g, n3), wl["seedB"])
    else:
        B_np = normal_lateral((n2, n4g, n3), wl["seedB"], j0, j1)
    B_host = torch.from_numpy(B_np)
    B = B_host.to(dev)
    A = tp.matlab_empty(n1, n2, n3, torch.float32, dev)
    t_bcast = None
    if rank == 0:
        A.copy_(A_host)
    if world > 1:
        from paper_1806_07247_b200 import dist as tpdist
        torch.cuda.synchronize()
        dist.barrier()
        if dist.get_backend() == "nccl":                   # one ncclBroadcast through the C ABI
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            tpdist.replicate(A, root=0, handle=handle)
            e1.record(stream)
            torch.cuda.synchronize()
            t_bcast = e0.elapsed_time(e1)
        else:                                              # gloo (tests): the host copy
            Ah = A.cpu() if rank == 0 else tp.matlab_empty(n1, n2, n3, torch.float32, "cpu")
            tpdist.replicate(Ah, root=0, handle=None)
            A.copy_(Ah)
            torch.cuda.synchronize()
        if rank != 0:
            A_host = A.cpu()
    C = tp.matlab_empty(n1, n4, n3, torch.float32, dev)

    # L2 flush between timed steps, outside the events: write a buffer of 2x L2 (evicts every line
    # of the previous step), then read a second one so the write-backs of those dirty lines also
    # complete before the next step starts (cold, clean L2).
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

    # ---- timed region: K steps, per-step events on the launching stream, L2 flushed in between
    handle.set_option(tp._lib.TPROD_OPT_TIMING, 1)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    stage_ms, launches = [], 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
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
    st_mean = [statistics.mean(s[i] for s in stage_ms) for i in range(4)]
    serial = None
    if st_mean[3] == 0.0:
        # K3 ran overlapped with the GEMM (TPROD_OPT_OVERLAP): the step has one K2 + K3 stage.  The
        # GEMM's own time (its roofline) comes from a few extra steps in the serial order (same
        # kernels, K3 launched after the GEMM completes), outside the timed region.
        handle.set_option(tp._lib.TPROD_OPT_OVERLAP, 0)
        sst = []
        for _ in range(max(3, args.steps // 4)):
            l2_flush()
            step()
            sst.append(handle.last_stage_ms())
        handle.set_option(tp._lib.TPROD_OPT_OVERLAP, 1)
        serial = [statistics.mean(s[i] for s in sst) for i in range(4)]
    handle.set_option(tp._lib.TPROD_OPT_TIMING, 0)
    ms, *st_max = _allmax(dist, world, [statistics.mean(step_ms)] + st_mean, dev)
    gemm_ms = st_max[2]
    if serial is not None:
        serial = _allmax(dist, world, serial, dev)
        gemm_ms = serial[2]
    F = metric_flops(n1, n2, n3, n4g)
    out = {"label": label, "n1": n1, "n2": n2, "n3": n3, "n4": n4g, "n4_local": n4,
           "ms": ms, "ms_min": min(step_ms), "value": F / (ms * 1e-3) / 1e12,
           "gemm_ms": gemm_ms, "gemm_flops_local": gemm_flops(n1, n2, n3, n4),
           "metric_flops_local": metric_flops(n1, n2, n3, n4),
           "stage_ms": [round(x, 5) for x in st_max], "stage_bytes_local": stage_bytes(n1, n2, n3, n4),
           "compulsory_bytes_local": 4.0 * n3 * (n1 * n2 + n2 * n4 + n1 * n4),
           "launches": launches, "clocks": clk.summary(), "bcast_ms": t_bcast,
           "serial_stage_ms": None if serial is None else [round(x, 5) for x in serial]}

    # ---- NEXT-1 prepared left operand: A's scales + forward DFT once (untimed), then K steps of the
    # B-side path (tprod_f32_prepared), same protocol; reported separately, never as `value`
    handle.prepare_a(A, stream=stream)
    Cp_dev = tp.tprod_prepared(B, handle=handle, stream=stream)
    torch.cuda.synchronize()
    evp = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        l2_flush()
        evp[i][0].record(stream)
        tp.tprod_prepared(B, out=Cp_dev, handle=handle, stream=stream)
        evp[i][1].record(stream)
    torch.cuda.synchronize()
    (tpm,) = _allmax(dist, world, [statistics.mean(a.elapsed_time(b) for a, b in evp)], dev)
    same = bool(torch.equal(Cp_dev, C))
    handle.release_a()
    del Cp_dev
    out["prepared_a"] = {"ms_per_step": tpm, "value": F / (tpm * 1e-3) / 1e12, "unit": "TFLOP/s",
                         "bitwise_equal_to_full_path": same,
                         "note": "A prepared once per A (tprod_prepare_a_f32, untimed); each step runs K0/K1 of B, "
                                 "the GEMM and the inverse; value credits the full metric flops"}

    # ---- e2e: the same metric through the C-ABI host entry point (pinned buffers, H2D + D2H inside)
    Ap, Bp = A_host.pin_memory(), B_host.pin_memory()
    Cp = tp.matlab_empty(n1, n4, n3, torch.float32, "cpu").pin_memory()
    Ap, Bp, Cp = (x if tp.is_matlab_layout(x) else tp.to_matlab(x) for x in (Ap, Bp, Cp))
    tp.tprod_f32_host(Ap, Bp, out=Cp, handle=handle, stream=stream)
    e2e_steps = max(2, min(args.steps, 10 if F < 1e13 else 3))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        tp.tprod_f32_host(Ap, Bp, out=Cp, handle=handle, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    (e2e_ms,) = _allmax(dist, world, [e0.elapsed_time(e1) / e2e_steps], dev)
    out["e2e"] = {"value": F / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
                  "h2d_bytes_per_step": 4 * (n1 * n2 * n3 + n2 * n4g * n3),
                  "d2h_bytes_per_step": 4 * n1 * n4g * n3, "steps": e2e_steps}
    del Ap, Bp, Cp

    # ---- parity spot check of the timed output on every rank: sampled lateral (and, for long
    # tubes, frontal) slices of the rank's shard vs the fp64 oracle; the line reports the max
    import oracle as O
    Jl = np.unique(np.array([0, 1, n4 // 2, n4 - 1]))
    big = n1 * n2 * n3 > (1 << 27) or n3 > 64          # the oracle gathers A once per slice
    Tl = np.array([0, 1, n3 // 2, n3 - 1]) if big else np.arange(n3)
    Cj = C[:, torch.from_numpy(Jl).to(dev), :][:, :, torch.from_numpy(Tl).to(dev)].cpu().numpy()
    ref = O.tprod_blockrow(A_host.numpy(), B_np[:, Jl, :], Tl, np.arange(len(Jl)))
    (err,) = _allmax(dist, world, [O.rel_err(Cj, ref)], dev)
    out["parity_rel_err_sampled"] = err
    out["parity_sample"] = (f"C(:, {Jl.tolist()}, {Tl.tolist() if big else 'all'}) of every rank's shard "
                            f"(global columns {j0}+...), max over ranks")
    out["shard"] = [j0, j1]
    if rank == 0:
        out["A_host"] = A_host
        out["B_cols"] = np.asfortranarray(B_np[:, :16, :])
    del A, B, C, flush, flush_rd
    torch.cuda.empty_cache()
    return out


def roofline(meas, peaks, src, workload, sustained):
    """The dominant kernel's roofline (K2 GEMM, tensor-bound) plus SURVEY 8(d)'s whole-call
    fraction T_roof / T (T_roof = max(F / P_tc, B / BW) for this rank's share) and each
    memory-bound stage's achieved algorithmic GB/s against the measured HBM peak."""
    P = peaks["bf16_tflops_sustained" if sustained else "bf16_tflops"] / 3.0
    BW = peaks["hbm_gbs"]
    achieved = meas["gemm_flops_local"] / (meas["gemm_ms"] * 1e-3) / 1e12
    tr = load_traffic(workload)
    t_roof_ms = max(meas["metric_flops_local"] / (P * 1e12), meas["compulsory_bytes_local"] / (BW * 1e9)) * 1e3
    sb = meas["stage_bytes_local"]
    k0, k1, k2, k3 = meas["stage_ms"]

    def gbs(b, t):
        return b / (t * 1e-3) / 1e9 if t > 0 else None
    if k1 == 0.0:
        # the A chain (K0 + K1 of A) ran concurrently with the B chain: one combined stage (tprod.h)
        b01 = sb["K0"] + sb["K1"]
        stages = {"K0 + K1 scales and forward DFTs (A, B chains concurrent)": {
            "ms": k0, "bytes": b01, "GB/s": gbs(b01, k0), "frac": gbs(b01, k0) / BW}}
    else:
        stages = {
            "K0 scales": {"ms": k0, "bytes": sb["K0"], "GB/s": gbs(sb["K0"], k0), "frac": gbs(sb["K0"], k0) / BW},
            "K1 forward DFT (A, B)": {"ms": k1, "bytes": sb["K1"], "GB/s": gbs(sb["K1"], k1),
                                      "frac": gbs(sb["K1"], k1) / BW}}
    ser = meas.get("serial_stage_ms")
    if k3 == 0.0 and ser:
        # K3 overlapped with the GEMM's last tile round (TPROD_OPT_OVERLAP): one combined stage; the
        # GEMM / K3 split below is from extra steps in the serial order (bench.time_workload)
        g, i3 = ser[2], ser[3]
        stages.update({
            "K2 + K3 GEMM and inverse DFT (overlapped)": {"ms": k2},
            "K2 GEMM (serial-order steps)": {"ms": g, "TFLOP/s": achieved, "frac": achieved / P},
            "K3 fill + inverse DFT (serial-order steps)": {"ms": i3, "bytes": sb["K3"], "GB/s": gbs(sb["K3"], i3),
                                                           "frac": gbs(sb["K3"], i3) / BW},
        })
    else:
        stages.update({
            "K2 GEMM": {"ms": k2, "TFLOP/s": achieved, "frac": achieved / P},
            "K3 fill + inverse DFT": {"ms": k3, "bytes": sb["K3"], "GB/s": gbs(sb["K3"], k3),
                                      "frac": gbs(sb["K3"], k3) / BW},
        })
    return {"bound": "tensor", "achieved": achieved, "peak": P, "unit": "TFLOP/s",
            "frac": achieved / P, "traffic": tr,
            "kernel": "K2 per-frequency complex GEMM (gemm_tc2_kernel / gemm_tc_kernel)",
            "call_frac": t_roof_ms / meas["ms"], "call_t_roof_ms": t_roof_ms,
            "note": (f"achieved = the GEMM's algorithmic flops (8*n1*n2*n4 per complex slice, 2*n1*n2*n4 "
                     f"per real DC/Nyquist slice) / mean K2 time (CUDA events on the "
                     f"launching stream, every timed step); peak = {src} bf16 "
                     f"{'sustained' if sustained else 'burst'} / 3: an fp32-accurate product costs 3 "
                     f"fp16 tensor-core products (hi*hi + hi*lo + lo*hi).  call_frac = T_roof / ms_per_step "
                     f"with T_roof = max(metric flops / peak, compulsory bytes (A, B read, C written) / "
                     f"{src} HBM {BW:.0f} GB/s) (SURVEY 8(d))"),
            "gemm_ms": meas["gemm_ms"], "stage_ms": meas["stage_ms"], "stages": stages}


def side_line(m, peaks, src, workload, steps):
    """A secondary workload measured with the same protocol, reported as an extra key."""
    return {"value": m["value"], "unit": "TFLOP/s", "ms_per_step": m["ms"],
            "config": {k: m[k] for k in ("n1", "n2", "n3", "n4")},
            "roofline": roofline(m, peaks, src, workload, m["ms"] * steps > 500.0),
            "e2e": m["e2e"], "gpu_launches": m["launches"], "clocks": m["clocks"],
            "prepared_a": m["prepared_a"], "parity_rel_err_sampled": m.get("parity_rel_err_sampled")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c5", choices=sorted(WORKLOADS))
    ap.add_argument("--extra", default="c3,c4,c2",
                    help="secondary workloads measured at N = 1 with the same protocol (extra keys)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c3", action="store_true", help="no secondary workloads (same as --extra '')")
    ap.add_argument("--engine", type=int, default=0, help="0 tcgen05 (default), 1 SIMT reference")
    ap.add_argument("--bn", type=int, default=0, help="force the GEMM N tile (0 = library heuristic)")
    ap.add_argument("--cn", type=int, default=0, help="force GEMM cluster width 1/2 (0 = heuristic)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="torch.distributed backend for N > 1 (gloo: the multi-rank test on one GPU)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    wl = dict(WORKLOADS[args.workload])

    if args.impl == "reference":
        run_reference(args, wl, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_1806_07247_b200 as tp
    from paper_1806_07247_b200 import build as tpbuild

    if rank == 0 or world == 1:
        tpbuild.build()
    ngpu = torch.cuda.device_count()
    gpu = local % max(ngpu, 1)           # one rank per GPU; the gloo test runs 2 ranks on one GPU
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
        dist.barrier()                   # rank 0 has built the library before anyone loads it
    handle = tp.Handle(gpu)
    handle.set_option(tp._lib.TPROD_OPT_ENGINE, args.engine)
    if args.bn:
        handle.set_option(tp._lib.TPROD_OPT_GEMM_BN, args.bn)
    if args.cn:
        handle.set_option(tp._lib.TPROD_OPT_GEMM_CLUSTER, args.cn)
    if world > 1 and args.dist_backend == "nccl":
        from paper_1806_07247_b200 import dist as tpdist
        handle.set_world(rank, world, tpdist.exchange_uid(tp.nccl_unique_id))
    stream = torch.cuda.current_stream(dev)

    meas = time_workload(tp, torch, dist, handle, wl, args, rank, world, local, dev, stream, args.workload)
    extras = {}
    if world == 1 and not args.no_c3:
        for name in [x for x in args.extra.split(",") if x and x != args.workload]:
            extras[name] = time_workload(tp, torch, dist, handle, dict(WORKLOADS[name]), args, rank, world, local,
                                         dev, stream, name)

    if rank == 0:
        peaks, src = load_peaks()
        sustained = meas["ms"] * args.steps > 500.0       # long timed region: sustained clocks
        n1, n2, n3, n4 = wl["n1"], wl["n2"], wl["n3"], wl["n4"]
        line = {
            "metric": METRIC, "value": meas["value"], "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": meas["ms"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic N(0,1), seeded (synth.normal, PCG64)",
            "config": {"workload": args.workload, "n1": n1, "n2": n2, "n3": n3, "n4": n4,
                       "h": h_slices(n3), "n4_per_gpu": meas["n4_local"],
                       "parallelism": f"lateral-slice shards x{world} (no collective in the step), "
                                      f"A broadcast once ({args.dist_backend})",
                       "l2": "flushed between timed steps (write 2x L2 then read 2x L2, outside the step events)",
                       "engine": "tcgen05" if args.engine == 0 else "simt-reference"},
            "roofline": roofline(meas, peaks, src, args.workload, sustained),
            "e2e": meas["e2e"],
            "gpu_launches": meas["launches"],
            "clocks": meas["clocks"],
            "parity_rel_err_sampled": meas.get("parity_rel_err_sampled"),
            "parity_sample": meas.get("parity_sample"),
            "ms_per_step_min": meas["ms_min"],
            "prepared_a": meas["prepared_a"],
        }
        if meas["bcast_ms"] is not None:
            line["setup_bcast_ms"] = meas["bcast_ms"]
        for name, m in extras.items():
            line[name] = side_line(m, peaks, src, name, args.steps)
        if not args.no_cpu_baseline and world == 1:      # rank 0 at N = 1 only
            line["cpu_baseline"] = cpu_baseline(wl, meas["A_host"].numpy(), meas["B_cols"])
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    handle.close()


if __name__ == "__main__":
    main()
