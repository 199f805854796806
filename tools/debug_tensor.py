"""Compare tensor vs exact engine on a config subset and print mismatches (dev tool)."""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_1511_05174_b200 import device as D, workloads as W, _native as N
ci = int(sys.argv[1]) if len(sys.argv) > 1 else 0
P = int(sys.argv[2]) if len(sys.argv) > 2 else 512
w = W.CONFIGS[ci]; d = W.dictionaries(ci)
ys = W.signals(ci, 0, P)
hi_t = d.e_high_t if w.measurements else d.high_t
hi = D.device_dictionary(hi_t)
eps = W.REL_TOL * np.linalg.norm(ys, axis=1)
a = D.omp_batch_raw(hi, ys.astype(np.float32), P, w.k, eps, None, 'tensor'); ia = N.last_run_info()
b = D.omp_batch_raw(hi, ys.astype(np.float32), P, w.k, eps, None, 'exact')
print('tensor run info', ia)
bad = [p for p in range(P) if not np.array_equal(a['sel'][p], b['sel'][p])]
print('mismatched signals', len(bad), bad[:10])
for p in bad[:3]:
    print(p, 'tensor', a['sel'][p], a['counts'][p], a['scans'][p], np.round(a['alpha'][p], 5))
    print(p, 'exact ', b['sel'][p], b['counts'][p], b['scans'][p], np.round(b['alpha'][p], 5))
    # exact correlations at pick 1 given exact pick 0 solution
    y = ys[p]; s0 = b['sel'][p][0]
    dd = hi_t[s0]; x0 = dd @ y / (dd @ dd); r = y - x0 * dd
    c = np.abs(hi_t @ r); o = np.argsort(-c)[:5]
    print('   iter1 top', o, c[o])
    # single-signal rerun
    one = D.omp_batch_raw(hi, ys[p:p+1].astype(np.float32), 1, w.k, eps[p:p+1], None, 'tensor')
    print('   single', one['sel'][0], N.last_run_info())

# ---- candidate lists on real residuals (iteration 1..5 of the exact run)
import torch
for p in bad[:2]:
    y = ys[p]
    sel = b['sel'][p]
    for it in range(1, 6):
        A = hi_t[sel[:it]].T
        x = np.linalg.lstsq(A, y, rcond=None)[0]
        r = (y - A @ x).astype(np.float32)[None, :]
        rd = torch.from_numpy(r).cuda()
        idx = torch.empty((1, 8), dtype=torch.int32, device='cuda'); val = torch.empty((1, 8), dtype=torch.float32, device='cuda'); drop = torch.empty((1,), dtype=torch.float32, device='cuda')
        N.check(N.load().cdb_debug_corr_topk(hi.handle, N.ptr(rd), 1, N.ptr(idx), N.ptr(val), N.ptr(drop), 0, None))
        c = np.abs(hi_t @ r[0].astype(np.float64)); o = np.argsort(-c)[:10]
        print(p, it, 'kernel', idx.cpu().numpy()[0], np.round(val.cpu().numpy()[0], 4), 'drop', round(float(drop.cpu()), 4))
        print(p, it, 'numpy ', o, np.round(c[o], 4), 'taken', sel[:it])
