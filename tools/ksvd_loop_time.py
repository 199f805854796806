"""Where a device K-SVD iteration spends its time (dev tool)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import ksvd_oracle as KO
from paper_1511_05174_b200 import learn as L, device as D
y, _, _ = KO.problem(64, 256, 20000, 8, 7, (3, 4))
L.ksvd(y[:, :2000], L.TrainConfig(256, 8, iterations=1))
d = L.init_atoms(y, L.TrainConfig(256, 8), np.random.default_rng(0))
def t(label, fn, reps=5):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); print(f"{label}: {(time.perf_counter()-t0)/reps*1e3:.2f} ms", flush=True)
t("DeviceDictionary(d.T)", lambda: D.DeviceDictionary(np.ascontiguousarray(d.T)))
yrows = torch.from_numpy(np.ascontiguousarray(y.T)).cuda()
eps = torch.from_numpy(1e-6 * np.linalg.norm(y, axis=0)).cuda()
dd = D.DeviceDictionary(np.ascontiguousarray(d.T))
t("code stage (omp_batch_raw)", lambda: D.omp_batch_raw(dd, yrows, 20000, 8, eps, None, "auto"))
t("init_atoms", lambda: L.init_atoms(y, L.TrainConfig(256, 8), np.random.default_rng(0)), 1)
t("cleanup_duplicates", lambda: L.cleanup_duplicates(y, d.copy(), np.ones(20000)), 3)
t0 = time.perf_counter(); L.ksvd(y, L.TrainConfig(256, 8, iterations=3)); print(f"ksvd 3 it: {(time.perf_counter()-t0)*1e3:.1f} ms")
# instrument one iteration of the loop body
import paper_1511_05174_b200._native as N
m, n, t, k = 20000, 64, 256, 8
outs = dict(sel=torch.empty((m, k), dtype=torch.int64, device='cuda'), alpha=torch.empty((m, k), dtype=torch.float64, device='cuda'),
            counts=torch.empty(m, dtype=torch.int64, device='cuda'), rnorm=torch.empty(m, dtype=torch.float64, device='cuda'),
            scans=torch.empty(m, dtype=torch.int64, device='cuda'), flag=torch.empty(m, dtype=torch.uint8, device='cuda'))
T = {}
def mark(lbl, t0):
    torch.cuda.synchronize(); T[lbl] = T.get(lbl, 0) + (time.perf_counter() - t0) * 1e3; return time.perf_counter()
for rep in range(3):
    t0 = time.perf_counter()
    o = L._code_device(d, yrows, eps, k, None, outs); t0 = mark("code", t0)
    sel, coef = o["sel"], o["alpha"]
    drows = torch.from_numpy(np.ascontiguousarray(d.T)).to('cuda'); t0 = mark("drows h2d", t0)
    valid = (sel >= 0) & (coef != 0.0); selc = sel.clamp(min=0); e = yrows.clone()
    for l in range(k):
        e -= torch.where(valid[:, l, None], coef[:, l, None] * drows[selc[:, l]], 0.0)
    t0 = mark("E", t0)
    pre = float(torch.linalg.norm(e)); t0 = mark("norm", t0)
    pp, ll = torch.nonzero(valid, as_tuple=True); atoms = sel[pp, ll]; order = torch.argsort(atoms * m + pp)
    pp, ll, atoms = pp[order], ll[order], atoms[order]; vals = coef[pp, ll].contiguous()
    counts = torch.bincount(atoms, minlength=t); ptr = torch.zeros(t + 1, dtype=torch.int64, device='cuda'); ptr[1:] = torch.cumsum(counts, 0)
    sig = pp.contiguous(); mx = int(counts.max()); t0 = mark("csr", t0)
    rep_ = np.zeros(1, dtype=np.int64)
    N.check(N.load().cdb_ksvd_update(n, m, t, N.ptr(yrows), N.ptr(e), N.ptr(drows), N.ptr(ptr), N.ptr(sig), N.ptr(vals), int(vals.numel()), mx, 1, N.ptr(rep_), None)); t0 = mark("update", t0)
    coef[pp, ll] = vals; post = float(torch.linalg.norm(e)); dd_ = drows.cpu().numpy(); rn = torch.linalg.norm(e, dim=1).cpu().numpy(); t0 = mark("tail", t0)
print({k2: round(v / 3, 2) for k2, v in T.items()})
