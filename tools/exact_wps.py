"""exact_omp device time on the operator-recovery problem (dev tool)."""
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_1511_05174_b200 import sensing as S, _native as N
from paper_1511_05174_b200.pipelines import recover_operator
rng = np.random.default_rng(3)
h = w = 512; c = 3
img = np.cumsum(rng.standard_normal((h, w, c)), axis=0) / 8
a = rng.integers(1, c + 1, size=h * w)
op = S.make_channel_mosaic(h * w, c, a)
coded = op.apply(img.ravel()).reshape(h, w)
d = rng.standard_normal((192, 384)); d /= np.linalg.norm(d, axis=0)
recover_operator(coded, op, (8, 8, 3), (2, 2, 1), dictionary=d, sparsity=6)
ts = []
for _ in range(3):
    N.profile_enable(True)
    recover_operator(coded, op, (8, 8, 3), (2, 2, 1), dictionary=d, sparsity=6)
    ts.append(N.profile_read()["exact_omp"][0]); N.profile_enable(False)
print(sorted(ts)[1])
