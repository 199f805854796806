"""Per-step kernel composition from an ncu launch list of bench.py (dev tool).

Segments the serialised launch list into the bench's zero-tree calls (from
downsample_kernel<float> to the gram_omp step and its delegate pass) and
full-OMP calls (ls_init_kernel<float> .. ls_final_kernel<float> + delegates),
and prints the mean device time per call of each kernel and its share of the
step, to compare with bench.py's CUDA-event `kernels_ms_per_step`.
usage: launch_steps.py launches.csv [first_n_calls]  (default 5: the bench's
warm-up + timed calls; later calls are the e2e leg's smaller pipeline chunks)"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
kn, mv, mu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
seq = []
for r in rows[hdr + 1:]:
    if len(r) > mv:
        name = r[kn].split("(")[0].replace("void ", "").replace("cdb::<unnamed>::", "").replace("unnamed>::", "")
        seq.append((name, float(r[mv].replace(",", "")) * scale.get(r[mu], 1e-6)))


def segments(start, end):
    out, i = [], 0
    while i < len(seq):
        if seq[i][0] == start:
            j = i + 1
            while j < len(seq) and not seq[j][0].startswith(end):
                j += 1
            j += 1
            while j < len(seq) and seq[j][0].split("<")[0] in ("collect_delegates_kernel", "exact_omp_kernel"):
                j += 1
            out.append(seq[i:j])
            i = j
        else:
            i += 1
    return out


for label, start, end in (("zero-tree call (configs[1], 100k signals)", "downsample_kernel<float>", "gram_omp_kernel"),
                          ("full-OMP call (configs[1], 100k signals)", "ls_init_kernel<float>", "ls_final_kernel"),
                          ("zero-tree step (configs[4], 1M signals)", "downsample_direct_kernel<float, 2>", "gram_reg2_kernel")):
    segs = segments(start, end)[: int(sys.argv[2]) if len(sys.argv) > 2 else 5]
    if not segs:
        continue
    per = defaultdict(float)
    cnt = defaultdict(int)
    for s in segs:
        for name, ms in s:
            per[name] += ms / len(segs)
            cnt[name] += 1
    tot = sum(per.values())
    print(f"== {label}: {len(segs)} calls in the list, {tot:.3f} ms per call (serialised, cold caches)")
    for name, ms in sorted(per.items(), key=lambda kv: -kv[1]):
        print(f"   {ms:8.3f} ms {100 * ms / tot:5.1f}%  x{cnt[name] / len(segs):5.1f}  {name[:70]}")
