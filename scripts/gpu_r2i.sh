timeout 1200 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k "stage or non_smooth or tsvd or tsvt or tinv or operand_scales" > gpurun_out/pytest_blue.log 2>&1; tail -3 gpurun_out/pytest_blue.log; grep -E "^FAILED|^E  .*assert" gpurun_out/pytest_blue.log | head -20
python - <<'PY'
import time, torch, numpy as np, sys
sys.path.insert(0, '.')
import paper_1806_07247_b200 as tp
from synth import normal
for n3 in (97, 1021, 4099, 8209):
    A = tp.to_matlab(torch.from_numpy(normal((64, 64, n3), 1)).cuda()); B = tp.to_matlab(torch.from_numpy(normal((64, 16, n3), 2)).cuda())
    h = tp.Handle(); C = tp.tprod(A, B, handle=h); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): tp.tprod(A, B, out=C, handle=h)
    e1.record(); torch.cuda.synchronize()
    print("n3", n3, "ms", e0.elapsed_time(e1) / 5, flush=True)
PY
