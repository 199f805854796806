"""Per-kernel device times of one zero-tree and one full-OMP call on any BASELINE config (dev tool).
usage: probe_kernels.py ci P"""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1511_05174_b200 import device as D, workloads as W, _native as N
ci, P = int(sys.argv[1]), int(sys.argv[2])
w = W.CONFIGS[ci]; d = W.dictionaries(ci)
ys = W.signals(ci, 0, P).astype(np.float32); yd = torch.from_numpy(ys).cuda()
phi = bool(w.measurements)
lo = D.device_dictionary(d.e_low_t if phi else d.low_t)
hi = D.device_dictionary(d.e_high_t if phi else d.high_t)
k1 = min(w.k, w.n_signal, w.t_low) if phi else w.k
eps = torch.from_numpy(W.REL_TOL * np.linalg.norm(ys.astype(np.float64), axis=1)).cuda()
for what in ('zt', 'full'):
    for rep in range(2):
        N.profile_enable(True)
        if what == 'zt':
            D.zero_tree_raw(lo, hi, None if phi else w.fine_shape, None if phi else w.factors, yd, P, k1, w.k, W.REL_TOL, phi, 'auto')
        else:
            D.omp_batch_raw(hi, yd, P, w.k, eps, None, 'auto')
        torch.cuda.synchronize()
        prof = N.profile_read(); N.profile_enable(False)
    print(f'cfg{ci} {what} P={P}', {k: (round(v[0], 2), v[1]) for k, v in prof.items()}, N.last_run_info(), flush=True)
