"""Diagnostics: run the t-product a few times with TPROD_GEMM_DEBUG=1 so the GEMM kernel reports
per-role barrier-wait cycles (see csrc/gemm_tc.cu).  Usage:
    TPROD_GEMM_DEBUG=1 python scripts/gemm_diag.py [n1 n2 n3 n4] [--bn B] [--cn C]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1806_07247_b200 as tp  # noqa: E402
from synth import normal  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("dims", nargs="*", type=int, default=[1024, 1024, 31, 512])
ap.add_argument("--bn", type=int, default=0)
ap.add_argument("--cn", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
n1, n2, n3, n4 = a.dims
h = tp.Handle(0)
if a.bn:
    h.set_option(tp._lib.TPROD_OPT_GEMM_BN, a.bn)
if a.cn:
    h.set_option(tp._lib.TPROD_OPT_GEMM_CLUSTER, a.cn)
h.set_option(tp._lib.TPROD_OPT_TIMING, 1)
A = torch.from_numpy(normal((n1, n2, n3), 1)).cuda()
B = torch.from_numpy(normal((n2, n4, n3), 2)).cuda()
for _ in range(a.reps):
    C = tp.tprod_f32(A, B, handle=h)
    torch.cuda.synchronize()
    print("stage ms", h.last_stage_ms(), flush=True)
