#!/usr/bin/env python
"""t-SVT timing (NEXT-2) on large slices: CUDA events around tp.tsvt, L2 flushed between steps,
plus the oracle check.  python scripts/bench_tsvt.py [out.json]"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import oracle as O
    import paper_1806_07247_b200 as tp
    from synth import normal
    rows = []
    for (n1, n2, n3, tau, steps) in ((64, 64, 64, 20.0, 10), (256, 256, 3, 20.0, 5), (512, 512, 8, 60.0, 3),
                                     (1024, 1024, 31, 200.0, 2)):
        Y = normal((n1, n2, n3), 181 if n1 == 1024 else 171 + n3)
        dY = tp.to_matlab(torch.from_numpy(Y).cuda())
        h = tp.Handle()
        X = tp.tsvt(dY, tau, handle=h)
        torch.cuda.synchronize()
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        ts = []
        for _ in range(steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            tp.tsvt(dY, tau, out=X, handle=h)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        err = O.rel_err(X.cpu().numpy(), O.tsvt(Y.astype(np.float64), tau))
        row = {"op": "tsvt", "n1": n1, "n2": n2, "n3": n3, "tau": tau, "ms": statistics.mean(ts),
               "rel_err_vs_oracle": err, "path": "per-slice CTA" if max(n1, n2) <= 64 else "blocked Jacobi"}
        print(json.dumps(row), flush=True)
        rows.append(row)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
