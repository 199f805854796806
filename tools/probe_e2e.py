"""e2e pipeline probe: device-only vs host-buffer zero-tree, and raw copy time (dev tool)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1511_05174_b200 import device as D, workloads as W
ci, P = 1, 100000
w = W.CONFIGS[ci]; d = W.dictionaries(ci)
ys = W.signals(ci, 0, P).astype(np.float32)
lo, hi = D.device_dictionary(d.low_t), D.device_dictionary(d.high_t)
def outs(k, dev, pin):
    mk = lambda shape, dt: torch.empty(shape, dtype=dt, device=dev, pin_memory=pin)
    return dict(sel=mk((P, k), torch.int64), alpha=mk((P, k), torch.float64), counts=mk((P,), torch.int64),
                rnorm=mk((P,), torch.float64), scans=mk((P,), torch.int64), flag=mk((P,), torch.uint8))
yd = torch.from_numpy(ys).cuda(); dl, dh = outs(w.k, 'cuda', False), outs(w.k, 'cuda', False)
yh = torch.from_numpy(ys).pin_memory(); hl, hh = outs(w.k, 'cpu', True), outs(w.k, 'cpu', True)
npv = lambda o: {k: v.numpy() for k, v in o.items()}
hln, hhn = npv(hl), npv(hh)
def t(fn, reps=5):
    fn(); torch.cuda.synchronize(); best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    return best * 1e3
dev = t(lambda: D.zero_tree_raw(lo, hi, w.fine_shape, w.factors, yd, P, w.k, w.k, W.REL_TOL, False, 'auto', dl, dh))
host = t(lambda: D.zero_tree_raw(lo, hi, w.fine_shape, w.factors, yh.numpy(), P, w.k, w.k, W.REL_TOL, False, 'auto', hln, hhn))
def copies():
    yd.copy_(yh, non_blocking=True)
    for o, h in ((dl, hl), (dh, hh)):
        for k in o: h[k].copy_(o[k], non_blocking=True)
cp = t(copies)
def h2d(): yd.copy_(yh, non_blocking=True)
print(f"device {dev:.3f} ms  host-pipelined {host:.3f} ms  copies(all serial) {cp:.3f} ms  h2d {t(h2d):.3f} ms")
