"""Summarize the K3 timeline written by tools/k3_trace.sh (last forward)."""
import sys
txt = open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/k3_trace.txt").read().split("TRACE rows=")[-1]
d = {}
for l in txt.splitlines():
    p = l.split()
    if len(p) == 3 and p[0] == "TRACE" and p[1].lstrip("-").isdigit() and p[2].lstrip("-").isdigit():
        d[int(p[1])] = int(p[2])
for s in range(1, 9):
    t = [d.get(1000 + 10 * s + k) for k in range(7)]
    if t[0] and all(t[:6]):
        print(f"step {s}: zphase {t[1]-t[0]} michelot {t[2]-t[1]} mask {t[3]-t[2]} xm {t[4]-t[3]} "
              f"transform {t[5]-t[4]} eta {t[6]-t[5] if t[6] else None}")
g = [(d.get(100 + 2 * j), d.get(101 + 2 * j)) for j in range(60) if d.get(100 + 2 * j)]
for j, (a, b) in enumerate(g[:8]):
    e = d.get(100 + 2 * (j + 1))
    print(f"gemm {j}: issue {b - a if b else None} -> next {e - b if (e and b) else None}")
