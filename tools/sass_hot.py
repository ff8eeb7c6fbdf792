"""Summarise an `ncu --page source --csv` SASS dump: opcode mix and hot loop.
    python tools/sass_hot.py dump.csv [min_frac]"""
import csv, re, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.001
h = [r for r in rows if 'Source' in r and 'Instructions Executed' in r][0]
si, ii, wi = h.index('Source'), h.index('Instructions Executed'), h.index('Warp Stall Sampling (All Samples)')
data = []
for r in rows:
    if len(r) > ii and r[ii].isdigit():
        data.append((r[si], int(r[ii]), int(r[wi] or 0)))
tot = sum(d[1] for d in data); tw = sum(d[2] for d in data) or 1
print("total warp inst %.4e  stall samples %d" % (tot, tw))
op = defaultdict(int)
for d in data:
    m = re.match(r'\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)', d[0])
    if m: op[m.group(2)] += d[1]
print(" ".join(f"{k}:{100*v/tot:.1f}%" for k, v in sorted(op.items(), key=lambda x: -x[1])[:28]))
for i, d in enumerate(data):
    if d[1] > tot * thr or d[2] > tw * 0.01:
        print(f"{i:5d} {d[1]:11d} {100*d[2]/tw:4.1f}  {d[0][:95]}")
