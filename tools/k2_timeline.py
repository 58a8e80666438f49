"""Summarise the GBMW_K2_HIST=1 K2 launch timeline (TL lines) of the last pass in a log."""
import collections, re, sys
lines = [l for l in open(sys.argv[1]) if l.startswith('TL')]
idx = [i for i, l in enumerate(lines) if l.startswith('TL u=1 g=0')]
last = lines[idx[-1]:] if idx else lines
by = collections.defaultdict(list)
for l in last:
    m = re.match(r'TL u=(\d+) g=(\d+) a=\[([\d.]+), ([\d.]+)\] b=\[([\d.]+), ([\d.]+)\]', l)
    u, g = int(m.group(1)), int(m.group(2))
    by[g].append((u,) + tuple(float(m.group(i)) for i in range(3, 7)))
for g, v in sorted(by.items()):
    v.sort()
    aa = sum(x[2] - x[1] for x in v); bb = sum(x[4] - x[3] for x in v); ab = sum(x[3] - x[2] for x in v)
    gaps = sum(v[i + 1][1] - v[i][4] for i in range(len(v) - 1))
    print(f'group {g}: steps {len(v)} span {v[0][1]:.0f} -> {v[-1][4]:.0f} us; sum classify {aa:.0f} rounds {bb:.0f} '
          f'a->b gaps {ab:.0f} step gaps {gaps:.0f}')
    for x in v[:4] + v[len(v) // 2:len(v) // 2 + 2] + v[-2:]:
        u, a0, a1, b0, b1 = x
        print(f'   u={u:3d} a [{a0:8.1f},{a1:8.1f}] ({a1 - a0:6.1f}) gap {b0 - a1:5.1f} b ({b1 - b0:6.1f})')
