#!/usr/bin/env python
"""Same-box A/B of library options on the per-stage times (CUDA events, TPROD_OPT_TIMING) of a
workload: python scripts/stage_ab.py --workload c5 --opt 5=0 --opt 5=2 [--steps 10]
(--opt OPTION=VALUE pairs; each is one arm).  L2 flushed between steps like bench.py."""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c5")
    ap.add_argument("--opt", action="append", default=[])
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    import torch
    import bench
    import paper_1806_07247_b200 as tp
    from synth import normal
    wl = bench.WORKLOADS[a.workload]
    n1, n2, n3, n4 = wl["n1"], wl["n2"], wl["n3"], wl["n4"]
    A = torch.from_numpy(normal((n1, n2, n3), wl["seedA"])).cuda()
    B = torch.from_numpy(normal((n2, n4, n3), wl["seedB"])).cuda()
    C = tp.matlab_empty(n1, n4, n3)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ref = None
    for arm in a.opt or ["5=0"]:
        h = tp.Handle()
        for kv in arm.split(","):
            k, v = kv.split("=")
            h.set_option(int(k), int(v))
        for _ in range(3):
            tp.tprod(A, B, out=C, handle=h)
        h.set_option(tp._lib.TPROD_OPT_TIMING, 1)
        st, tot = [], []
        for _ in range(a.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            tp.tprod(A, B, out=C, handle=h)
            e1.record()
            st.append(h.last_stage_ms())
            torch.cuda.synchronize()
            tot.append(e0.elapsed_time(e1))
        out = C.cpu()
        diff = None if ref is None else float((out - ref).norm() / ref.norm())
        if ref is None:
            ref = out
        print(json.dumps({"workload": a.workload, "arm": arm, "ms": round(statistics.mean(tot), 5),
                          "stage_ms": [round(statistics.mean(s[i] for s in st), 5) for i in range(4)],
                          "rel_diff_vs_first_arm": diff}), flush=True)
        h.close()


if __name__ == "__main__":
    main()
