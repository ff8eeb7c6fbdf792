# opcode mix of the forward / backward raster kernels (ncu source page, reduced on the box)
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --warm-iters 0"
$CMD > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --clock-control none --profile-from-start off -k "regex:fwd_kernel|bwd_kernel" -c 2 -o /tmp/rm -f $CMD > gpurun_out/ncu_rm.log 2>&1
ncu -i /tmp/rm.ncu-rep --page source --csv > /tmp/rm_src.csv 2>/dev/null
python - <<'PY'
import csv, collections
rows = list(csv.reader(open('/tmp/rm_src.csv')))
cur = None; hdr = None; data = collections.defaultdict(list)
for r in rows:
    if r and r[0] == 'Kernel Name': cur = r[1][:30]; continue
    if r and r[0] == 'Address': hdr = r; continue
    if cur and hdr and len(r) > 5: data[cur].append(r)
out = open('gpurun_out/raster_opmix.txt', 'w')
for k, v in data.items():
    ie = hdr.index('Instructions Executed'); src = hdr.index('Source')
    c = collections.Counter(); tot = 0
    for r in v:
        try: n = int(r[ie])
        except ValueError: continue
        op = r[src].split()
        if not op: continue
        o = op[1] if op[0].startswith('@') else op[0]
        c[o] += n; tot += n
    print(k, tot, file=out)
    for o, n in c.most_common(30): print(f"   {o:22s} {n:12d} {100*n/tot:5.1f}%", file=out)
PY
echo done
