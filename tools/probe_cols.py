"""Drop-in column-batch timing on configs[4] (dev tool): zero_tree_many_arrays
on an N x P fp64 pageable batch through the cols ABI vs the old host-transpose
rows path; host staging bandwidth; CDB_PIPE_TRACE=1 prints the chunk timeline.
usage: python tools/probe_cols.py [signals] [reps]"""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1511_05174_b200 import workloads as W, pursuit as PU, device as D
from paper_1511_05174_b200 import crossscale as C
from paper_1511_05174_b200.tensor import Dictionary
from paper_1511_05174_b200.scaling import ScaleSpec
m = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ci = 4; w = W.CONFIGS[ci]; d = W.dictionaries(ci)
PU.REL_RESIDUAL_TOL = W.REL_TOL
yd = W.signals_device(ci, 0, m)
cols = yd.T.contiguous().double().cpu().numpy()
del yd
model = C.CrossScaleModel(Dictionary(np.ascontiguousarray(d.low_t.T)),
                          Dictionary(np.ascontiguousarray(d.high_t.T)),
                          ScaleSpec(w.fine_shape, w.factors), w.k, w.k)
t0 = time.perf_counter(); x = np.array(cols); print(f'numpy copy {cols.nbytes / (time.perf_counter() - t0) / 1e9:.1f} GB/s', flush=True); del x
print('cpus', os.cpu_count(), flush=True)
for rep in range(reps):
    t0 = time.perf_counter(); low, high, tm = C.zero_tree_many_arrays(model, cols); dt = time.perf_counter() - t0
    print(f'cols path: {dt:.3f} s {m / dt / 1e3:.1f} k sig/s device {tm}', flush=True)
if os.environ.get('ROWS'):
    for rep in range(2):
        t0 = time.perf_counter(); r = D.rows_for_device(cols); t1 = time.perf_counter()
        lo2, hi2, tm2 = C._solve(model, r, None); dt = time.perf_counter() - t0
        print(f'rows path: {dt:.3f} s ({t1 - t0:.3f} transpose) {m / dt / 1e3:.1f} k sig/s device {tm2}', flush=True)
    print('equal sel', np.array_equal(low.sel, lo2.sel), np.array_equal(high.sel, hi2.sel))
