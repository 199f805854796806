"""A/B of the cfg-4 step-2 Gram kernels (dev tool): zero-tree on P device
signals with CDB_GRAM_REG=0 (streamed H) and with the on-chip kernel at each
register-row count; prints per-kernel times and output agreement.
usage: ab_gram.py [ci] [P]"""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1511_05174_b200 import device as D, workloads as W, _native as N
ci = int(sys.argv[1]) if len(sys.argv) > 1 else 4
P = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
w = W.CONFIGS[ci]; d = W.dictionaries(ci)
yd = W.signals_device(ci, 0, P); torch.cuda.synchronize()
phi = bool(w.measurements)
lo = D.device_dictionary(d.e_low_t if phi else d.low_t)
hi = D.device_dictionary(d.e_high_t if phi else d.high_t)
k1 = min(w.k, w.n_signal, w.t_low) if phi else w.k
def outs(k):
    return dict(sel=torch.empty((P, k), dtype=torch.int64, device='cuda'), alpha=torch.empty((P, k), dtype=torch.float64, device='cuda'),
                counts=torch.empty(P, dtype=torch.int64, device='cuda'), rnorm=torch.empty(P, dtype=torch.float64, device='cuda'),
                scans=torch.empty(P, dtype=torch.int64, device='cuda'), flag=torch.empty(P, dtype=torch.uint8, device='cuda'))
res = {}
for label, env in (("stream", {"CDB_GRAM_TMA": "0"}), ("tma", {})):
    for k in ("CDB_GRAM_REG", "CDB_GRAM_R", "CDB_GRAM_TMA"):
        os.environ.pop(k, None)
    os.environ.update(env)
    ol, oh = outs(k1), outs(w.k)
    for rep in range(2):
        N.profile_enable(True)
        torch.cuda.synchronize(); t0 = time.time()
        D.zero_tree_raw(lo, hi, None if phi else w.fine_shape, None if phi else w.factors, yd, P, k1, w.k, W.REL_TOL, phi, 'auto', ol, oh)
        torch.cuda.synchronize(); el = time.time() - t0
        prof = N.profile_read(); N.profile_enable(False)
    g = {k: round(v[0], 2) for k, v in prof.items() if 'step2' in k or 'alpha0' in k}
    print(f"{label}: {el*1e3:.1f} ms total, {g}", flush=True)
    res[label] = {k: v.cpu().numpy() for k, v in oh.items()}
base = res["stream"]
for label, r in res.items():
    if label == "stream":
        continue
    same_sel = (r["sel"] == base["sel"]).all(axis=1).mean()
    nz = base["alpha"] != 0
    rel = np.abs(r["alpha"] - base["alpha"])[nz] / np.abs(base["alpha"][nz])
    print(f"{label}: bitwise equal sel/alpha/rnorm: {(r['sel']==base['sel']).all()} {(r['alpha']==base['alpha']).all()} {(r['rnorm']==base['rnorm']).all()}")
    print(f"{label}: rows with identical sel {same_sel:.5f}, counts equal {(r['counts']==base['counts']).mean():.5f}, "
          f"scans equal {(r['scans']==base['scans']).mean():.5f}, coef max rel diff (same-sel rows) "
          f"{np.max(np.abs(r['alpha']-base['alpha'])[(r['sel']==base['sel']).all(axis=1)]) if same_sel>0 else -1:.3e}, "
          f"rnorm max rel {np.max(np.abs(r['rnorm']-base['rnorm'])/np.maximum(base['rnorm'],1e-300)):.3e}", flush=True)
