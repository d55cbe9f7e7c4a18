"""One t-product step on a workload shape with device-side random inputs, for ncu captures.

    python scripts/profile_step.py c5        # ncu --set full -k regex:... python scripts/profile_step.py c5
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1806_07247_b200 as tp  # noqa: E402
from bench import WORKLOADS  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
n1, n2, n3, n4 = wl["n1"], wl["n2"], wl["n3"], wl["n4"]
g = torch.Generator(device="cuda").manual_seed(0)
A = tp.to_matlab(torch.randn(n1, n2, n3, device="cuda", generator=g))
B = tp.to_matlab(torch.randn(n2, n4, n3, device="cuda", generator=g))
h = tp.Handle()
C = tp.tprod(A, B, handle=h)
torch.cuda.synchronize()
tp.tprod(A, B, out=C, handle=h)
torch.cuda.synchronize()
print("done", n1, n2, n3, n4)
