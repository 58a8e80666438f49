"""Per-CUDA-line stall samples and executed instructions from
`ncu -i REP --page source --csv --print-source cuda,sass`: python tools/ncu_lines.py CSV [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur = None
agg = {}
fname = None
for r in rows:
    if not r:
        continue
    if r[0] == 'File Path':
        fname = r[1].split('/')[-1]
        continue
    if r[0] in ('Function Name', 'Line No'):
        continue
    if r[0] != '':
        try:
            cur = (fname, int(r[0]), r[1].strip()[:70])
        except ValueError:
            cur = None
        continue
    if cur is None or len(r) < 8:
        continue
    try:
        s, ins = int(r[4]), int(r[7])
    except ValueError:
        continue
    a = agg.setdefault(cur, [0, 0])
    a[0] += s
    a[1] += ins
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f'samples {ts}  instructions {ti}')
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f'{100*v[0]/ts:5.1f}% smp {100*v[1]/ti:5.1f}% ins  {k[0]}:{k[1]}  {k[2]}')
