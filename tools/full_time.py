"""Median device time of the cfg-1 full-OMP kernels over 7 calls (dev tool)."""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1511_05174_b200 import device as D, workloads as W, _native as N
ci = int(sys.argv[1]) if len(sys.argv) > 1 else 1
w = W.CONFIGS[ci]; d = W.dictionaries(ci); P = 100000
ys = W.signals(ci, 0, P).astype(np.float32)
yd = torch.from_numpy(ys).cuda()
eps = torch.from_numpy(W.REL_TOL * np.linalg.norm(ys.astype(np.float64), axis=1)).cuda()
hi = D.device_dictionary(d.high_t)
acc = {}
for rep in range(8):
    N.profile_enable(True)
    D.omp_batch_raw(hi, yd, P, w.k, eps, None, 'auto')
    torch.cuda.synchronize()
    prof = N.profile_read(); N.profile_enable(False)
    if rep:
        for k, v in prof.items():
            acc.setdefault(k, []).append(v[0])
print({k: round(float(np.median(v)), 3) for k, v in acc.items()}, N.last_run_info())
