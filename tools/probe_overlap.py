import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1511_05174_b200 import device as D, workloads as W
print('asyncEngineCount', torch.cuda.get_device_properties(0).__dict__ if False else '', flush=True)
ci, P = 1, 100000
w = W.CONFIGS[ci]; d = W.dictionaries(ci)
ys = W.signals(ci, 0, P).astype(np.float32)
lo, hi = D.device_dictionary(d.low_t), D.device_dictionary(d.high_t)
yd = torch.from_numpy(ys).cuda()
yh = torch.from_numpy(ys).pin_memory(); ydst = torch.empty_like(yd)
big_h = torch.empty(200 << 20, dtype=torch.uint8).pin_memory(); big_d = torch.empty(200 << 20, dtype=torch.uint8, device='cuda')
s2 = torch.cuda.Stream()
def zt(): D.zero_tree_raw(lo, hi, w.fine_shape, w.factors, yd, P, w.k, w.k, W.REL_TOL, False, 'auto')
def cp():
    with torch.cuda.stream(s2): big_d.copy_(big_h, non_blocking=True)
def tm(fn):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); return (time.perf_counter() - t0) * 1e3
a = tm(zt); b = tm(cp)
def both(): cp(); zt()
c = tm(both)
print(f'zt {a:.2f} ms  copy200MB {b:.2f} ms  both {c:.2f} ms')
from cuda.bindings import runtime as rt
err, prop = rt.cudaGetDeviceProperties(0)
print('asyncEngineCount', prop.asyncEngineCount, 'concurrentKernels', prop.concurrentKernels)
