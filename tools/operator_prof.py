"""cProfile of recover_operator on the demosaic problem (dev tool)."""
import cProfile, pstats, sys
import numpy as np
sys.path.insert(0, '.')
from paper_1511_05174_b200 import sensing as S
from paper_1511_05174_b200.pipelines import recover_operator
rng = np.random.default_rng(3)
H = W = 512; C = 3
img = np.cumsum(rng.standard_normal((H, W, C)), axis=0) / 8
a = rng.integers(1, C + 1, size=H * W)
op = S.make_channel_mosaic(H * W, C, a)
coded = op.apply(img.ravel()).reshape(H, W)
d = rng.standard_normal((192, 384)); d /= np.linalg.norm(d, axis=0)
recover_operator(coded, op, (8, 8, 3), (2, 2, 1), dictionary=d, sparsity=6)
pr = cProfile.Profile(); pr.enable()
recover_operator(coded, op, (8, 8, 3), (2, 2, 1), dictionary=d, sparsity=6)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(14)
