"""Time zero-tree with different engines (dev tool)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1511_05174_b200 import device as D, workloads as W, _native as N
ci, P = int(sys.argv[1]), int(sys.argv[2])
w = W.CONFIGS[ci]; d = W.dictionaries(ci)
ys = W.signals(ci, 0, P).astype(np.float32); yd = torch.from_numpy(ys).cuda()
lo, hi = D.device_dictionary(d.low_t), D.device_dictionary(d.high_t)
for eng in sys.argv[3].split(','):
    for rep in range(3):
        N.profile_enable(True)
        torch.cuda.synchronize(); t0 = time.time()
        D.zero_tree_raw(lo, hi, w.fine_shape, w.factors, yd, P, w.k, w.k, W.REL_TOL, False, eng)
        torch.cuda.synchronize(); t1 = time.time()
        prof = N.profile_read()
    print(eng, f'{(t1-t0)*1e3:.2f} ms', {k: round(v[0], 3) for k, v in prof.items()}, flush=True)
