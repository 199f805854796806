"""Hottest SASS instructions (stall samples) of a `--page source --csv --print-source sass` export (dev tool).
usage: ncu_hot.py file.csv.gz [top]"""
import csv
import gzip
import sys

rows = list(csv.reader(gzip.open(sys.argv[1], 'rt')))
hdr = rows[1]
si, ni = hdr.index('Source'), hdr.index('Warp Stall Sampling (All Samples)')
lsb = hdr.index('stall_long_sb')
body = rows[2:]
tot = sum(int(r[ni] or 0) for r in body) or 1
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
idx = sorted(range(len(body)), key=lambda i: -int(body[i][ni] or 0))[:top]
for i in sorted(idx):
    r = body[i]
    print(f"{i:5d} {100*int(r[ni])/tot:5.1f}% lsb={r[lsb]:>5} {r[si].strip()[:90]}")
