"""Summarize a K2 TBN_TRACE timeline: per-GEMM phases of each group of CTA 0."""
import os
import sys

for fn in sys.argv[1:]:
    lines = open(fn).read().split('TRACE rows=')[-1].splitlines()[1:]
    d = {}
    for l in lines:
        p = l.split()
        if len(p) == 3 and p[0] == 'TRACE':
            d[int(p[1])] = int(p[2])
    t0 = min(v for v in d.values() if v > 0)
    print(fn)
    for g in range(int(os.environ.get("NGROUPS", "1"))):
        G = g * 4000
        for k in range(4):
            if d.get(G + 3000 + 8 * k) is None:
                continue
            a = [d.get(G + 3000 + 8 * k + i) for i in range(4)]
            print(f"g{g} tile{k}: start {a[0]-t0} xload {a[1]-a[0]} body {a[2]-a[1]} tail {a[3]-a[2]}")
        prev = None
        tot = dict(bar=0, issue=0, wait=0, epi=0)
        for j in range(200):
            v = [d.get(G + 4 * j + i) for i in range(4)]
            if v[0] is None or v[3] is None:
                continue
            bar, iss, wait = v[1] - v[0], v[2] - v[1], v[3] - v[2]
            epi = v[0] - prev if prev else 0
            tot['bar'] += bar; tot['issue'] += iss; tot['wait'] += wait; tot['epi'] += epi
            if os.environ.get("VERBOSE"):
                print(f"  j={j:3d} bar={bar:5d} issue={iss:5d} wait={wait:5d} epi={epi:5d}")
            prev = v[3]
        print(f"g{g} totals", tot)
        for s in range(1, 9):
            a, b = d.get(G + 3500 + 4 * s), d.get(G + 3501 + 4 * s)
            if a and b:
                print(f"  g{g} sparsemax s={s}: {b - a}")
