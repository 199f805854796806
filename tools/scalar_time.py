"""Per-call latency of the scalar drop-in omp / zero_tree_omp (dev tool)."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_1511_05174_b200 as P
rng = np.random.default_rng(0)
d = rng.standard_normal((64, 256)); d /= np.linalg.norm(d, axis=0)
ys = rng.standard_normal((64, 500))
cfg = P.PursuitConfig(8)
P.omp(d, ys[:, 0], cfg)
t0 = time.perf_counter()
for i in range(500): P.omp(d, ys[:, i], cfg)
t1 = time.perf_counter()
print(f"scalar omp: {(t1 - t0) / 500 * 1e6:.0f} us per call")
sets = [frozenset(range(1, 257, 2))] * 500
P.omp(d, ys[:, 0], P.PursuitConfig(8, allowed_support=sets[0]))
t0 = time.perf_counter()
for i in range(500): P.omp(d, ys[:, i], P.PursuitConfig(8, allowed_support=sets[i]))
print(f"scalar omp with allowed_support: {(time.perf_counter() - t0) / 500 * 1e6:.0f} us per call")
