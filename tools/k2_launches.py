"""Per-launch K2 durations (us) from an ncu launch-list csv: python tools/k2_launches.py TAG"""
import csv, sys
tag = sys.argv[1]
with open(f'gpurun_out/launches_{tag}.csv') as f:
    lines = [l for l in f if l.startswith('"')]
r = csv.reader(lines)
hdr = next(r)
ki, mi, vi, ii = (hdr.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'ID'))
d = {}
for row in r:
    if row[mi] == 'gpu__time_duration.sum':
        d[int(row[ii])] = (row[ki], float(row[vi].replace(',', '')))
for g in ('<0, 0>', '<1, 0>', '<2, 0>'):
    ts = [t for i, (n, t) in sorted(d.items()) if 'k_dp_step' in n and g in n]
    if ts:
        print(g, f'sum {sum(ts)/1e3:.2f} ms', [round(x / 1000) for x in ts])
