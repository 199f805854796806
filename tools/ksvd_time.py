"""Device vs CPU (oracle restatement of the reference) K-SVD update stage (dev tool)."""
import sys, time
import numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import ksvd_oracle as KO
from paper_1511_05174_b200.learn import update_stage
from paper_1511_05174_b200 import _native as N
for n, t, m, k in ((64, 256, 20000, 8), (256, 1024, 20000, 16)):
    y, d, x = KO.problem(n, t, m, k, 7, (3, 4))
    d1, x1 = d.copy(), x.copy(); update_stage(y, d1, x1, 2)  # warm
    d1, x1 = d.copy(), x.copy()
    t0 = time.perf_counter(); update_stage(y, d1, x1, 2); t1 = time.perf_counter()
    N.profile_enable(True); d3, x3 = d.copy(), x.copy(); update_stage(y, d3, x3, 2); prof = N.profile_read(); N.profile_enable(False)
    d2, x2 = d.copy(), x.copy()
    t2 = time.perf_counter(); KO.update_stage(y, d2, x2, 2); t3 = time.perf_counter()
    print(f"N={n} T={t} M={m} K={k}: device call {1e3*(t1-t0):.1f} ms (kernel {prof.get('ksvd_update', (0,))[0]:.1f} ms), CPU reference {1e3*(t3-t2):.1f} ms", flush=True)
