"""Step-1 problem of a BASELINE config under each engine (dev tool): OMP of the
step-1 input on D_low (or E_low for the Phi config)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
sys.path.insert(0, 'oracle')
from paper_1511_05174_b200 import device as D, workloads as W
import oracle as O
ci, P = int(sys.argv[1]), int(sys.argv[2])
w = W.CONFIGS[ci]; d = W.dictionaries(ci)
ys = W.signals(ci, 0, P).astype(np.float32).astype(np.float64)
phi = bool(w.measurements)
y1 = ys if phi else O.downsample_rows(ys, w.fine_shape, w.factors)
lo = D.device_dictionary(d.e_low_t if phi else d.low_t)
k1 = min(w.k, w.n_signal, w.t_low) if phi else w.k
eps = W.REL_TOL * np.linalg.norm(y1, axis=1)
yd = torch.from_numpy(y1).cuda(); ed = torch.from_numpy(eps).cuda()
for eng in sys.argv[3].split(','):
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.time()
        D.omp_batch_raw(lo, yd, P, k1, ed, None, eng)
        torch.cuda.synchronize(); t1 = time.time()
    print(f'cfg{ci} step1 P={P} {eng}: {(t1-t0)*1e3:.2f} ms', flush=True)
