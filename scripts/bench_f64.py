#!/usr/bin/env python
"""fp64 path timing (the paper's arithmetic is Matlab double): one t-product of a workload shape in
fp64, CUDA events, L2 flushed between steps; TFLOP/s of the metric's flop count and the fraction of
the B200's FP64 peak (37 TFLOP/s nominal, fp64 FMA units; B200_PROFILING.md gives no measured fp64
number).  python scripts/bench_f64.py [c3|c2|c5] [steps]"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import bench
    import oracle as O
    import paper_1806_07247_b200 as tp
    from synth import normal
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    wl = bench.WORKLOADS[name]
    n1, n2, n3, n4 = wl["n1"], wl["n2"], wl["n3"], wl["n4"]
    A_np = normal((n1, n2, n3), wl["seedA"], np.float64)
    B_np = normal((n2, n4, n3), wl["seedB"], np.float64)
    A = torch.from_numpy(A_np).cuda()
    B = torch.from_numpy(B_np).cuda()
    A, B = tp.to_matlab(A), tp.to_matlab(B)
    C = tp.matlab_empty(n1, n4, n3, torch.float64)
    h = tp.Handle()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        tp.tprod(A, B, out=C, handle=h)
    ts = []
    for _ in range(steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        tp.tprod(A, B, out=C, handle=h)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.mean(ts)
    F = bench.metric_flops(n1, n2, n3, n4)
    cols = np.array([0, n4 // 2, n4 - 1])
    Cs = C[:, torch.from_numpy(cols).cuda(), :].cpu().numpy()
    err = O.rel_err(Cs, O.tprod_columns(A_np, B_np, cols))
    print(json.dumps({"workload": name, "dtype": "f64", "ms": ms, "TFLOP/s": F / ms / 1e9,
                      "frac_of_fp64_peak_37": F / ms / 1e9 / 37.0, "rel_err_sampled": err}))


if __name__ == "__main__":
    main()
