"""Full-OMP per-kernel times on a random N x T dictionary (dev tool; env switches are read once per
process: one setting per run).  usage: ab_shape_full.py N T K P"""
import sys, time, hashlib
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1511_05174_b200 import device as D, _native as NN
n, t, k, P = map(int, sys.argv[1:5])
g = torch.Generator(device='cuda').manual_seed(1)
d = torch.randn((t, n), generator=g, device='cuda', dtype=torch.float64)
d /= d.norm(dim=1, keepdim=True)
x = torch.zeros((P, t), device='cuda', dtype=torch.float32)
idx = torch.randint(0, t, (P, k), generator=g, device='cuda')
x.scatter_(1, idx, torch.randn((P, k), generator=g, device='cuda'))
yd = (x @ d.float() + 0.01 * torch.randn((P, n), generator=g, device='cuda')).contiguous()
del x
eps = (1e-3 * torch.linalg.vector_norm(yd.double(), dim=1)).contiguous()
dd = D.DeviceDictionary(d.cpu().numpy())
of = dict(sel=torch.empty((P, k), dtype=torch.int64, device='cuda'), alpha=torch.empty((P, k), dtype=torch.float64, device='cuda'),
          counts=torch.empty(P, dtype=torch.int64, device='cuda'), rnorm=torch.empty(P, dtype=torch.float64, device='cuda'),
          scans=torch.empty(P, dtype=torch.int64, device='cuda'), flag=torch.empty(P, dtype=torch.uint8, device='cuda'))
for rep in range(2):
    NN.profile_enable(True); torch.cuda.synchronize(); t0 = time.time()
    D.omp_batch_raw(dd, yd, P, k, eps, None, 'tensor', of)
    torch.cuda.synchronize(); el = time.time() - t0
    prof = NN.profile_read(); NN.profile_enable(False)
h = hashlib.sha1(b''.join(of[q].cpu().numpy().tobytes() for q in ('sel', 'alpha', 'rnorm', 'counts'))).hexdigest()[:12]
print(h, f"N={n} T={t} K={k} P={P}: {el*1e3:.1f} ms, " + ", ".join(f"{q} {v[0]:.2f}" for q, v in prof.items() if v[0] > 0.5), flush=True)
