"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list (dev tool)."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hdr_i]; ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value'); ui = hdr.index('Metric Unit')
agg = collections.defaultdict(lambda: [0, 0.0]); seq = []
for r in rows[hdr_i + 1:]:
    if len(r) <= vi: continue
    name = r[ki].split('(')[0].replace('void ', '').replace('(anonymous namespace)::', '').replace('unnamed>::', '')[:48]
    v = float(r[vi].replace(',', ''))
    v = v / 1000 if r[ui] == 'ns' else (v * 1000 if r[ui] == 'ms' else v)
    agg[name][0] += 1; agg[name][1] += v; seq.append((name, round(v, 1)))
tot = sum(t for _, t in agg.values())
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f'{c:5d} {t:10.1f} us {100*t/tot:5.1f}%  {k}')
if len(sys.argv) > 2: print(seq[-int(sys.argv[2]):])
