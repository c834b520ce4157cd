"""Summarize a TBN_TRACE timeline (gemm handoffs of group 0, tile 0)."""
import sys
for fn in sys.argv[1:]:
    lines = open(fn).read().split('TRACE rows=')[-1].splitlines()[1:]
    d = {}
    for l in lines:
        p = l.split()
        if len(p) == 3 and p[0] == 'TRACE':
            d[int(p[1])] = int(p[2])
    print(fn, 'end', d.get(2))
    prev_end = None
    G = int(__import__("os").environ.get("TG", "0")) * 5000
    for j in range(64):
        a0, a1, a2, a3, f0 = (d.get(G + 1000 + 4 * j), d.get(G + 1001 + 4 * j), d.get(G + 1002 + 4 * j),
                              d.get(G + 1003 + 4 * j), d.get(G + 2000 + 4 * j))
        if a0 is None or a1 is None:
            continue
        f0 = f0 or a0
        mw = d.get(G + 3500 + j)
        print(f"j={j:2d} at_bar issuer={a0} half1={f0} bar={a1 - max(a0, f0):5d} issue={a2 - a1:5d} "
              f"mma+wake={a3 - a2:5d} (mbar {mw - a2 if mw else -1:5d}) epi={a0 - prev_end if prev_end else 0:5d}")
        prev_end = a3
    g = lambda k: d.get(k)
    if g(3090) is not None:
        print("tile start: xwait", g(3091) - g(3090), "xn", g(3092) - g(3091))
    if g(3100) is not None:
        print("tail: head", g(3101) - g(3100), "claim", g(3102) - g(3101), "imp+flush", g(3103) - g(3102),
              "-> end", d.get(2) - g(3103), "| last gemm end -> agg done", g(3100) - prev_end)
    for s in range(1, 9):
        t = [d.get(3000 + 8 * s + k) for k in range(5)]
        if t[0] is None:
            continue
        print(f"att s={s}: z={t[1]-t[0]} tau={t[2]-t[1]} claim={t[3]-t[2]} masks+A={t[4]-t[3]}")
