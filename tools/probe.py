"""Quick device timing probe of the engines on one BASELINE config (dev tool)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1511_05174_b200 import device as D, workloads as W, _native as N

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 1
P = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
engines = sys.argv[3].split(',') if len(sys.argv) > 3 else ['gram']
what = sys.argv[4] if len(sys.argv) > 4 else 'zt,full'
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
w = W.CONFIGS[ci]; d = W.dictionaries(ci)
t0 = time.time(); ys = W.signals(ci, 0, P).astype(np.float32); print('gen', time.time()-t0, flush=True)
yd = torch.from_numpy(ys).cuda()
lo = D.device_dictionary(d.low_t if not w.measurements else d.e_low_t)
hi = D.device_dictionary(d.high_t if not w.measurements else d.e_high_t)
eps = torch.from_numpy(W.REL_TOL * np.linalg.norm(ys.astype(np.float64), axis=1)).cuda()
phi = bool(w.measurements)
k1 = min(w.k, w.n_signal, w.t_low) if phi else w.k
def outs(k):
    return dict(sel=torch.empty((P, k), dtype=torch.int64, device='cuda'), alpha=torch.empty((P, k), dtype=torch.float64, device='cuda'),
                counts=torch.empty(P, dtype=torch.int64, device='cuda'), rnorm=torch.empty(P, dtype=torch.float64, device='cuda'),
                scans=torch.empty(P, dtype=torch.int64, device='cuda'), flag=torch.empty(P, dtype=torch.uint8, device='cuda'))
for eng in engines:
    ol, oh, of = outs(k1), outs(w.k), outs(w.k)
    for rep in range(reps if 'zt' in what else 0):
        torch.cuda.synchronize(); t0 = time.time()
        _, _, ms = D.zero_tree_raw(lo, hi, None if phi else w.fine_shape, None if phi else w.factors, yd, P, k1, w.k, W.REL_TOL, phi, eng, ol, oh)
        torch.cuda.synchronize(); t1 = time.time()
        print(f'cfg{ci} P={P} {eng} zero-tree: {t1-t0:.4f}s  steps ms {ms}  -> {P/(t1-t0):.0f} sig/s', flush=True)
    for rep in range(reps if 'full' in what else 0):
        torch.cuda.synchronize(); t0 = time.time()
        D.omp_batch_raw(hi, yd, P, w.k, eps, None, eng, of)
        torch.cuda.synchronize(); t1 = time.time()
        print(f'cfg{ci} P={P} {eng} full: {t1-t0:.4f}s -> {P/(t1-t0):.0f} sig/s  run_info={N.last_run_info()}', flush=True)
