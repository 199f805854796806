"""Full-OMP e2e (pinned host buffers) vs device-resident, cfg 1 (dev tool)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1511_05174_b200 import device as D, workloads as W
P = 100000; w = W.CONFIGS[1]; d = W.dictionaries(1)
ys = W.signals(1, 0, P).astype(np.float32)
eps = W.REL_TOL * np.linalg.norm(ys.astype(np.float64), axis=1)
hi = D.device_dictionary(d.high_t)
yh = torch.from_numpy(ys).pin_memory().numpy()
def mk(shape, dt): return torch.empty(shape, dtype=dt, pin_memory=True).numpy()
o = dict(sel=mk((P, w.k), torch.int64), alpha=mk((P, w.k), torch.float64), counts=mk((P,), torch.int64),
         rnorm=mk((P,), torch.float64), scans=mk((P,), torch.int64), flag=mk((P,), torch.uint8))
yd = torch.from_numpy(ys).cuda(); ed = torch.from_numpy(eps).cuda()
def t(fn, reps=4):
    fn(); torch.cuda.synchronize(); best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    return best * 1e3
dev = t(lambda: D.omp_batch_raw(hi, yd, P, w.k, ed, None, "auto"))
host = t(lambda: D.omp_batch_raw(hi, yh, P, w.k, eps, None, "auto", o))
print(f"full: device {dev:.2f} ms  host-pipelined {host:.2f} ms")
