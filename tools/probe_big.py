"""Per-kernel device times of zero-tree / full OMP on a BASELINE config with
device-generated signals (dev tool).  usage: probe_big.py ci P [zt,full] [reps]"""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1511_05174_b200 import device as D, workloads as W, _native as N
ci, P = int(sys.argv[1]), int(sys.argv[2])
what = sys.argv[3].split(',') if len(sys.argv) > 3 else ['zt', 'full']
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
w = W.CONFIGS[ci]; d = W.dictionaries(ci)
t0 = time.time(); yd = W.signals_device(ci, 0, P); torch.cuda.synchronize()
print('gen', round(time.time() - t0, 2), 's', flush=True)
phi = bool(w.measurements)
lo = D.device_dictionary(d.e_low_t if phi else d.low_t)
hi = D.device_dictionary(d.e_high_t if phi else d.high_t)
k1 = min(w.k, w.n_signal, w.t_low) if phi else w.k
eps = (W.REL_TOL * torch.linalg.vector_norm(yd.double(), dim=1)).contiguous()
def outs(k):
    return dict(sel=torch.empty((P, k), dtype=torch.int64, device='cuda'), alpha=torch.empty((P, k), dtype=torch.float64, device='cuda'),
                counts=torch.empty(P, dtype=torch.int64, device='cuda'), rnorm=torch.empty(P, dtype=torch.float64, device='cuda'),
                scans=torch.empty(P, dtype=torch.int64, device='cuda'), flag=torch.empty(P, dtype=torch.uint8, device='cuda'))
ol, oh, of = outs(k1), outs(w.k), outs(w.k)
for wh in what:
    for rep in range(reps):
        N.profile_enable(True)
        torch.cuda.synchronize(); t0 = time.time()
        if wh == 'zt':
            D.zero_tree_raw(lo, hi, None if phi else w.fine_shape, None if phi else w.factors, yd, P, k1, w.k, W.REL_TOL, phi, 'auto', ol, oh)
        else:
            D.omp_batch_raw(hi, yd, P, w.k, eps, None, 'auto', of)
        torch.cuda.synchronize(); el = time.time() - t0
        prof = N.profile_read(); N.profile_enable(False)
        print(f'cfg{ci} {wh} P={P} {el:.3f}s -> {P/el:.0f} sig/s', {k: (round(v[0], 2), v[1]) for k, v in prof.items()}, N.last_run_info(), flush=True)
