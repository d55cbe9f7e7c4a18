#!/usr/bin/env python
"""Small t-products that reach every kernel family of libtprod.so, for compute-sanitizer
(memcheck / synccheck / racecheck / initcheck):

    compute-sanitizer --tool racecheck python scripts/sanitize_cases.py [--quick]

Each case is also checked against the fp64 oracle, so a run that corrupts memory silently still
fails.  Exit code 0 = all cases ran and matched."""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# (n1, n2, n3, n4, dtype, what it reaches)
CASES = [
    (20, 30, 10, 15, np.float64, "config 1 fp64: fwd_f64 / gemm_simt_f64 / inv f64"),
    (20, 30, 10, 15, np.float32, "config 1 dims fp32: dense register kernels, single-CTA tcgen05 GEMM"),
    (256, 256, 32, 256, np.float32, "config 2: pair dense kernels n3 = 32, GEMM"),
    (512, 96, 64, 256, np.float32, "tube FFT K1/K3 n3 = 64, cta_group::2 pair GEMM"),
    (300, 64, 31, 130, np.float32, "odd n3 dense, ragged tiles"),
    (64, 40, 45, 20, np.float32, "TMA dense forward (33..64, not a power of two)"),
    (36, 20, 128, 12, np.float32, "tube FFT n3 = 128"),
    (33, 17, 100, 9, np.float32, "mixed-radix FFT n3 = 100"),
    (16, 12, 4096, 8, np.float32, "four-step long tubes n3 = 4096"),
    (12, 10, 67, 6, np.float32, "generic O(n3^2) n3 = 67"),
]


def main():
    import torch
    import oracle as O
    import paper_1806_07247_b200 as T
    from paper_1806_07247_b200 import build
    from synth import normal
    build.build()
    quick = "--quick" in sys.argv
    h = T.Handle()
    h.set_option(T._lib.TPROD_OPT_GRAPHS, 0)     # direct launches: every kernel is seen by the tool
    bad = 0
    for (n1, n2, n3, n4, dt, what) in (CASES[:4] if quick else CASES):
        A = normal((n1, n2, n3), 1 + n3, dt)
        B = normal((n2, n4, n3), 2 + n3, dt)
        C = T.tprod(torch.from_numpy(np.asfortranarray(A)).cuda(), torch.from_numpy(np.asfortranarray(B)).cuda(),
                    handle=h)
        torch.cuda.synchronize()
        C = C.cpu().numpy()
        cols = np.arange(min(n4, 4))
        ref = O.tprod_columns(A.astype(np.float64), B.astype(np.float64), cols)
        err = O.rel_err(C[:, cols], ref)
        tol = 1e-12 if dt == np.float64 else 1e-5
        ok = err <= tol
        bad += not ok
        print(f"{'ok ' if ok else 'BAD'} {n1}x{n2}x{n3}x{n4} {np.dtype(dt).name} rel_err {err:.2e}  ({what})", flush=True)
    if not quick:
        Y = normal((24, 20, 9), 5)
        X = T.tsvt(torch.from_numpy(np.asfortranarray(Y)).cuda(), 3.0, handle=h)
        torch.cuda.synchronize()
        e = O.rel_err(X.cpu().numpy(), O.tsvt(Y.astype(np.float64), 3.0))
        print(f"{'ok ' if e <= 1e-5 else 'BAD'} tsvt 24x20x9 rel_err {e:.2e}", flush=True)
        bad += e > 1e-5
        Z = normal((16, 16, 7), 6) + 8 * O.teye(16, 7).astype(np.float32)
        Xi = T.tinv(torch.from_numpy(np.asfortranarray(Z)).cuda(), handle=h)
        torch.cuda.synchronize()
        e = O.rel_err(Xi.cpu().numpy(), O.tinv(Z.astype(np.float64)))
        print(f"{'ok ' if e <= 1e-5 else 'BAD'} tinv 16x16x7 rel_err {e:.2e}", flush=True)
        bad += e > 1e-5
    h.close()
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
