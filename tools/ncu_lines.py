"""Per-source-line instruction/stall attribution from `ncu --page source --csv --print-source cuda,sass`."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
rowsper = float(sys.argv[2]) if len(sys.argv) > 2 else 65536
agg = collections.defaultdict(lambda: [0.0, 0.0, ''])
cur = None; hdr = None
for r in rows:
    if not r: continue
    if r[0] == 'File Path': cur = r[1].split('/')[-1]; hdr = None; continue
    if r[0] == 'Function Name': continue
    if r[0] == 'Line No': hdr = r; continue
    if hdr is None or not r[0]: continue
    try: ex = float(r[7] or 0); st = float(r[4] or 0)
    except ValueError: continue
    k = (cur, r[0]); agg[k][0] += ex; agg[k][1] += st; agg[k][2] = r[1]
tot = sum(v[0] for v in agg.values()); ts = sum(v[1] for v in agg.values())
print('total warp instr %.0f  per row %.0f' % (tot, tot * 32 / rowsper))
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[3]) if len(sys.argv) > 3 else 40]:
    print('%5.1f%% ex %5.1f%% st  %s:%s  %s' % (100 * v[0] / tot, 100 * v[1] / ts, k[0], k[1], v[2].strip()[:80]))
