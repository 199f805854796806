"""A/B of env switches on one configs[CI] full-OMP call (dev tool): per-kernel
device times for each setting and bitwise agreement with the first.
usage: ab_env_full.py P "ENV=a,ENV2=b" "ENV=c" ..."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1511_05174_b200 import device as D, workloads as W, _native as N
P = int(sys.argv[1]); ci = int(os.environ.get('CI', 4))
w = W.CONFIGS[ci]; d = W.dictionaries(ci)
yd = W.signals_device(ci, 0, P); torch.cuda.synchronize()
hi = D.device_dictionary(d.high_t)
eps = (W.REL_TOL * torch.linalg.vector_norm(yd.double(), dim=1)).contiguous()
def outs(k):
    return dict(sel=torch.empty((P, k), dtype=torch.int64, device='cuda'), alpha=torch.empty((P, k), dtype=torch.float64, device='cuda'),
                counts=torch.empty(P, dtype=torch.int64, device='cuda'), rnorm=torch.empty(P, dtype=torch.float64, device='cuda'),
                scans=torch.empty(P, dtype=torch.int64, device='cuda'), flag=torch.empty(P, dtype=torch.uint8, device='cuda'))
base = None
for spec in sys.argv[2:]:
    env = dict(kv.split('=') for kv in spec.split(',') if kv)
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    of = outs(w.k)
    for rep in range(2):
        N.profile_enable(True); torch.cuda.synchronize(); t0 = time.time()
        D.omp_batch_raw(hi, yd, P, w.k, eps, None, 'auto', of)
        torch.cuda.synchronize(); el = time.time() - t0
        prof = N.profile_read(); N.profile_enable(False)
    r = {k: v.cpu().numpy() for k, v in of.items()}
    eq = None if base is None else all((r[k] == base[k]).all() for k in ('sel', 'alpha', 'rnorm', 'counts'))
    if base is None: base = r
    import hashlib
    hsh = hashlib.sha1(b''.join(r[k].tobytes() for k in ('sel', 'alpha', 'rnorm', 'counts'))).hexdigest()[:12]
    print(hsh, f"{spec or 'default'}: {el*1e3:.1f} ms ({P/el:.0f} sig/s), bitwise={eq}, " + ", ".join(f"{k} {v[0]:.2f}" for k, v in prof.items() if v[0] > 0.5), N.last_run_info(), flush=True)
    for k, v in saved.items():
        if v is None: os.environ.pop(k, None)
        else: os.environ[k] = v
