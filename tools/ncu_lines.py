"""Top CUDA source lines by warp-stall samples from an ncu report (dev tool).
usage: ncu_lines.py report.ncu-rep kernel_regex [top]"""
import csv, subprocess, sys, io
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '-k', f'regex:{kern}',
                      '--print-source', 'cuda,sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file = ''
data = []
hdr = None
for r in rows:
    if not r: continue
    if r[0] == 'File Path': cur_file = r[1].split('/')[-1]; continue
    if r[0] == 'Line No': hdr = r; continue
    if hdr and r[0].isdigit():
        try:
            ws = int(r[4] or 0); ie = int(r[7] or 0)
        except ValueError:
            continue
        data.append((ws, ie, f'{cur_file}:{r[0]}', r[1].strip()[:90]))
tw = sum(d[0] for d in data) or 1; ti = sum(d[1] for d in data) or 1
for d in sorted(data, key=lambda x: -x[0])[:top]:
    print(f'{100*d[0]/tw:5.1f}% stall {100*d[1]/ti:5.1f}% inst  {d[2]}: {d[3]}')
