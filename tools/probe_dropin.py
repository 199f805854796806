"""Drop-in API timing: crossscale.zero_tree_many_arrays on numpy N x P columns (dev tool)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1511_05174_b200 import workloads as W
from paper_1511_05174_b200.crossscale import CrossScaleModel, zero_tree_many_arrays
from paper_1511_05174_b200.tensor import Dictionary
from paper_1511_05174_b200.scaling import ScaleSpec
ci = 1; w = W.CONFIGS[ci]; d = W.dictionaries(ci)
model = CrossScaleModel(Dictionary(d.low_t.T), Dictionary(d.high_t.T), ScaleSpec(w.fine_shape, w.factors), w.k, w.k)
cols = np.ascontiguousarray(W.signals(ci, 0, w.signals).astype(np.float32).T)
for rep in range(4):
    t0 = time.perf_counter(); low, high, tm = zero_tree_many_arrays(model, cols); dt = time.perf_counter() - t0
    print(f'drop-in zero_tree_many_arrays: {dt * 1e3:.2f} ms ({w.signals / dt / 1e6:.2f} M sig/s), device steps {tm}')
