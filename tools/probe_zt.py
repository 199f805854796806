"""Zero-tree / full OMP device calls for ncu captures (dev tool)."""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1511_05174_b200 import device as D, workloads as W
ci, P, what = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
w = W.CONFIGS[ci]; d = W.dictionaries(ci)
ys = W.signals(ci, 0, P).astype(np.float32); yd = torch.from_numpy(ys).cuda()
lo, hi = D.device_dictionary(d.low_t), D.device_dictionary(d.high_t)
for _ in range(2):
    if 'zt' in what:
        D.zero_tree_raw(lo, hi, w.fine_shape, w.factors, yd, P, w.k, w.k, W.REL_TOL, False, 'auto')
    if 'full' in what:
        eps = torch.from_numpy(W.REL_TOL * np.linalg.norm(ys.astype(np.float64), axis=1)).cuda()
        D.omp_batch_raw(hi, yd, P, w.k, eps, None, 'auto')
torch.cuda.synchronize(); print('ok')
