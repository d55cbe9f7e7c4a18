import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1806_07247_b200 as T
n3 = int(sys.argv[1]) if len(sys.argv) > 1 else 8
X = np.zeros((128, 1, n3), np.float32)
X[0, 0, :] = np.arange(1, n3 + 1)
X[1, 0, 0] = 1.0
d = torch.from_numpy(X).permute(2, 1, 0).contiguous().permute(2, 1, 0).cuda()
spec = T.dft_f32(d, role=1)
torch.cuda.synchronize()
print("gpu", spec[0, 0].cpu().numpy())
print("ref", np.fft.rfft(X[0, 0].astype(np.float64)))
print("gpu1", spec[1, 0].cpu().numpy())
