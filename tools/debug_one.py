import sys, numpy as np
sys.path.insert(0, '.')
from paper_1511_05174_b200 import device as D, workloads as W, _native as N
ci, sig = int(sys.argv[1]), int(sys.argv[2])
w = W.CONFIGS[ci]; d = W.dictionaries(ci); ys = W.signals(ci, sig, sig + 1)
hi = D.device_dictionary(d.high_t); eps = W.REL_TOL * np.linalg.norm(ys, axis=1)
o = D.omp_batch_raw(hi, ys.astype(np.float32), 1, w.k, eps, None, 'tensor')
print('sel', o['sel'][0], N.last_run_info())
y = ys[0]; print('|y|', np.linalg.norm(y))
s0 = o['sel'][0][0]; A = d.high_t[[s0]].T; x = np.linalg.lstsq(A, y, rcond=None)[0]; r = y - A @ x
c = d.high_t @ r; oo = np.argsort(-np.abs(c))[:4]; print('iter1 exact', oo, c[oo], '|r|', np.linalg.norm(r))
