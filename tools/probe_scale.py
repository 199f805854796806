"""Device-only zero-tree time vs batch size, per-kernel (dev tool)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1511_05174_b200 import device as D, workloads as W, _native as N
ci = 1
w = W.CONFIGS[ci]; d = W.dictionaries(ci)
ys_all = W.signals(ci, 0, 100000).astype(np.float32)
lo, hi = D.device_dictionary(d.low_t), D.device_dictionary(d.high_t)
for P in (int(x) for x in sys.argv[1:]):
    yd = torch.from_numpy(ys_all[:P]).cuda()
    mk = lambda k: dict(sel=torch.empty((P, k), dtype=torch.int64, device='cuda'), alpha=torch.empty((P, k), dtype=torch.float64, device='cuda'),
                        counts=torch.empty(P, dtype=torch.int64, device='cuda'), rnorm=torch.empty(P, dtype=torch.float64, device='cuda'),
                        scans=torch.empty(P, dtype=torch.int64, device='cuda'), flag=torch.empty(P, dtype=torch.uint8, device='cuda'))
    ol, oh = mk(w.k), mk(w.k)
    f = lambda: D.zero_tree_raw(lo, hi, w.fine_shape, w.factors, yd, P, w.k, w.k, W.REL_TOL, False, 'auto', ol, oh)
    f(); torch.cuda.synchronize()
    N.profile_enable(True)
    t0 = time.perf_counter(); f(); torch.cuda.synchronize(); dt = (time.perf_counter() - t0) * 1e3
    prof = N.profile_read(); N.profile_enable(False)
    print(P, f'{dt:.3f} ms', {k: round(v[0], 3) for k, v in prof.items()})
