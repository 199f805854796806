"""Operator-recovery throughput (row f3) on a demosaic-sized problem (dev tool)."""
import sys, time
import numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
from paper_1511_05174_b200 import sensing as S
from paper_1511_05174_b200.pipelines import recover_operator
import operator_oracle as OO
rng = np.random.default_rng(3)
H = W = 512; C = 3
img = np.cumsum(rng.standard_normal((H, W, C)), axis=0) / 8
a = rng.integers(1, C + 1, size=H * W)
op = S.make_channel_mosaic(H * W, C, a)
coded = op.apply(img.ravel()).reshape(H, W)
patch, stride = (8, 8, 3), (2, 2, 1)
n = 192
d = rng.standard_normal((n, 384)); d /= np.linalg.norm(d, axis=0)
recover_operator(coded[:64, :64], op if False else S.make_channel_mosaic(64 * 64, C, a.reshape(H, W)[:64, :64].ravel()), patch, stride, dictionary=d, sparsity=6)
t0 = time.perf_counter()
est, met, _ = recover_operator(coded, op, patch, stride, dictionary=d, sparsity=6)
t1 = time.perf_counter()
P = met.patch_count
print(f"device: {P} patches in {(t1 - t0) * 1e3:.1f} ms -> {P / (t1 - t0):.0f} patches/s (coding {met.coding_time_s * 1e3:.1f} ms)")
# CPU oracle on a crop (bounded sample)
hs = 96
g = dict(kind="channel-mosaic", assignment=a.reshape(H, W)[:hs, :hs].ravel(), channels=C,
         sig_shape=np.array((hs, hs, C)), patch=np.array(patch), stride=np.array(stride),
         meas=coded[:hs, :hs], method="omp-single", atoms=d, k=6)
t2 = time.perf_counter(); r = OO.recover(g); t3 = time.perf_counter()
pc = ((hs - 8) // 2 + 1) ** 2
print(f"cpu oracle (1 thread): {pc} patches in {(t3 - t2) * 1e3:.0f} ms -> {pc / (t3 - t2):.0f} patches/s")
est, met, codes = recover_operator(coded, op, patch, stride, dictionary=d, sparsity=6)
c = codes["code"]
print("flags", int(np.asarray(c["flag"]).sum()), "mean count", float(np.asarray(c["counts"]).mean()), "scans", int(np.asarray(c["scans"]).sum()))
import torch
from paper_1511_05174_b200 import _native as N
N.profile_enable(True)
recover_operator(coded, op, patch, stride, dictionary=d, sparsity=6)
print(N.profile_read())
