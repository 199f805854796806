import cProfile, pstats, sys
import numpy as np
sys.path.insert(0, '.')
import paper_1511_05174_b200 as P
rng = np.random.default_rng(0)
d = rng.standard_normal((64, 256)); d /= np.linalg.norm(d, axis=0)
ys = rng.standard_normal((64, 500)); cfg = P.PursuitConfig(8)
P.omp(d, ys[:, 0], cfg)
pr = cProfile.Profile(); pr.enable()
for i in range(300): P.omp(d, ys[:, i], cfg)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
