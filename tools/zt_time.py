"""Median device time of the cfg-1 zero-tree kernels over 7 calls (dev tool)."""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1511_05174_b200 import device as D, workloads as W, _native as N
ci = int(sys.argv[1]) if len(sys.argv) > 1 else 1
w = W.CONFIGS[ci]; d = W.dictionaries(ci); P = 100000
yd = torch.from_numpy(W.signals(ci, 0, P).astype(np.float32)).cuda()
lo, hi = D.device_dictionary(d.low_t), D.device_dictionary(d.high_t)
acc = {}
for rep in range(8):
    N.profile_enable(True)
    D.zero_tree_raw(lo, hi, w.fine_shape, w.factors, yd, P, w.k, w.k, W.REL_TOL, False, 'auto')
    torch.cuda.synchronize()
    prof = N.profile_read(); N.profile_enable(False)
    if rep:
        for k, v in prof.items():
            acc.setdefault(k, []).append(v[0])
print({k: round(float(np.median(v)), 3) for k, v in acc.items()})
