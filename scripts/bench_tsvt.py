#!/usr/bin/env python
"""NEXT-row timings on large slices -- t-SVT (NEXT-2), t-SVD scalars and factors (NEXT-3), tinv
(NEXT-4): CUDA events around each call, L2 flushed between steps, plus the oracle checks.
python scripts/bench_tsvt.py [out.json]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _time(fn, steps):
    import statistics
    import torch
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.mean(ts)


def main():
    import numpy as np
    import torch
    import oracle as O
    import paper_1806_07247_b200 as tp
    from synth import normal
    rows = []

    def emit(row):
        print(json.dumps(row), flush=True)
        rows.append(row)

    for (n1, n2, n3, tau, steps) in ((64, 64, 64, 20.0, 10), (256, 256, 3, 20.0, 5), (512, 512, 8, 60.0, 3),
                                     (1024, 1024, 31, 200.0, 2)):
        Y = normal((n1, n2, n3), 181 if n1 == 1024 else 171 + n3)
        dY = tp.to_matlab(torch.from_numpy(Y).cuda())
        h = tp.Handle()
        X = tp.tsvt(dY, tau, handle=h)
        torch.cuda.synchronize()
        ms = _time(lambda: tp.tsvt(dY, tau, out=X, handle=h), steps)
        err = O.rel_err(X.cpu().numpy(), O.tsvt(Y.astype(np.float64), tau))
        emit({"op": "tsvt", "n1": n1, "n2": n2, "n3": n3, "tau": tau, "ms": ms, "rel_err_vs_oracle": err,
              "path": "per-slice CTA" if max(n1, n2) <= 64 else "blocked Jacobi", "status": h.status()})
    # t-SVD scalars and factors (full rank and tubal rank 10: the completion of the left vectors)
    for (n1, n2, n3, rank, steps) in ((256, 256, 3, 0, 3), (512, 512, 8, 0, 2), (512, 512, 8, 10, 2)):
        if rank:
            A = O.tprod_bcirc(normal((n1, rank, n3), 191, np.float64), normal((rank, n2, n3), 192, np.float64))
            A = A.astype(np.float32)
        else:
            A = normal((n1, n2, n3), 193 + n3)
        dA = tp.to_matlab(torch.from_numpy(A).cuda())
        h = tp.Handle()
        out = tp.tsvd_values(dA, handle=h)
        ms_v = _time(lambda: tp.tsvd_values(dA, handle=h), steps)
        U, S, V = tp.tsvd(dA, handle=h)
        ms_f = _time(lambda: tp.tsvd(dA, handle=h), steps)
        _, S_ref, _ = O.tsvd(A.astype(np.float64))
        r = min(n1, n2)
        s_ref = np.array([S_ref[i, i, 0] for i in range(r)])
        Uh = U.cpu().numpy()
        orth = O.rel_err(O.tprod_bcirc(O.tran(Uh), Uh), O.teye(r, n3))
        emit({"op": "tsvd", "n1": n1, "n2": n2, "n3": n3, "tubal_rank": rank or r, "ms_values": ms_v,
              "ms_factors": ms_f, "rel_err_S_vs_oracle": O.rel_err(S.cpu().numpy(), S_ref),
              "rel_err_values_vs_oracle": O.rel_err(out.cpu().numpy()[:r].astype(np.float64), s_ref),
              "rel_err_UtU_vs_I": orth, "status": h.status()})
    # tinv beyond the shared-memory kernel
    for (n, n3, steps) in ((96, 8, 5), (256, 8, 3), (1024, 3, 2)):
        A = normal((n, n, n3), 197, np.float64) * (0.2 / np.sqrt(n3))
        A[:, :, 0] += 2.0 * np.eye(n)
        A = A.astype(np.float32)
        dA = tp.to_matlab(torch.from_numpy(A).cuda())
        h = tp.Handle()
        X = tp.tinv(dA, handle=h)
        ms = _time(lambda: tp.tinv(dA, out=X, handle=h), steps)
        Xh = X.cpu().numpy()
        emit({"op": "tinv", "n": n, "n3": n3, "ms": ms, "path": "smem fp32" if n <= 96 else "global fp64",
              "rel_err_AX_vs_I": O.rel_err(O.tprod_bcirc(A.astype(np.float64), Xh.astype(np.float64)),
                                           O.teye(n, n3))})
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
