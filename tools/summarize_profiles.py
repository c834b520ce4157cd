"""Distill gpurun_out/ ncu captures into tracked profiles/ summaries.

    python tools/summarize_profiles.py hr tf32x3 r1

Reads gpurun_out/launches_<cfg>_<prec>_<tag>.csv (launch list) and
gpurun_out/full_<cfg>_<prec>_<tag>.ncu-rep (one --set full capture) and writes
profiles/<tag>_<cfg>_<prec>.md plus an entry in profiles/ncu_summary.json
(bench.py reads `dram_bytes_per_launch` from it for roofline.traffic).
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
cfg, prec, tag = sys.argv[1], sys.argv[2], sys.argv[3]
out_dir = ROOT / "profiles"
out_dir.mkdir(exist_ok=True)

# ---- launch list ----
rows = []
txt = (ROOT / "gpurun_out" / f"launches_{cfg}_{prec}_{tag}.csv").read_text().splitlines()
hdr = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
for r in csv.DictReader(io.StringIO("\n".join(txt[hdr:]))):
    rows.append((r["Kernel Name"], float(r["Metric Value"])))
tot = sum(t for _, t in rows)
fused = [t for n, t in rows if ("tabnet_fused" in n or "tabnet_rowthread" in n or "tabnet_wide" in n)]
share = sum(fused) / tot if tot else 0.0

# ---- full capture ----
rep = ROOT / "gpurun_out" / f"full_{cfg}_{prec}_{tag}.ncu-rep"
raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
lines = raw.splitlines()
h = next(csv.reader([lines[0]]))
vals = next(csv.reader([lines[2]]))
d = dict(zip(h, vals))


def num(k):
    try:
        return float(d[k].replace(",", ""))
    except (KeyError, ValueError):
        return None


metrics = {
    "duration_ns": num("gpu__time_duration.sum"),
    "dram_bytes_read": num("dram__bytes_read.sum"),
    "dram_bytes_write": num("dram__bytes_write.sum"),
    "sm_clock_hz": num("smsp__cycles_elapsed.avg.per_second"),
    "issue_slots_busy_pct": num("sm__instruction_throughput.avg.pct_of_peak_sustained_active"),
    "tensor_pipe_active_pct": num("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
    "tc_pipe_active_pct": num("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active"),
    "xu_pipe_pct": num("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
    "fma_pipe_pct": num("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    "alu_pipe_pct": num("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
    "dram_throughput_pct": num("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    "registers_per_thread": num("launch__registers_per_thread"),
    "warps_active_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "inst_executed": num("smsp__inst_executed.sum"),
}
units = {k: d.get(k) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum")}
# ncu reports byte sums in the unit of its header row (second line)
u = dict(zip(h, next(csv.reader([lines[1]]))))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
for key, mk in (("dram_bytes_read", "dram__bytes_read.sum"), ("dram_bytes_write", "dram__bytes_write.sum")):
    if metrics[key] is not None:
        metrics[key] *= scale.get(u.get(mk, "byte"), 1)
dur_unit = u.get("gpu__time_duration.sum", "ns")
if metrics["duration_ns"] is not None and dur_unit in ("usecond", "us"):
    metrics["duration_ns"] *= 1e3
elif metrics["duration_ns"] is not None and dur_unit in ("msecond", "ms"):
    metrics["duration_ns"] *= 1e6
traffic = (metrics["dram_bytes_read"] or 0) + (metrics["dram_bytes_write"] or 0)

summ_path = out_dir / "ncu_summary.json"
summ = json.loads(summ_path.read_text()) if summ_path.exists() else {}
# merge: keep keys written by other captures (tools/update_traffic.py's
# steady-state traffic) for the same config/precision
summ.setdefault(f"{cfg}/{prec}", {}).update({
    "tag": tag, "dram_bytes_per_launch": traffic, "fused_kernel_share_of_launch_list": share,
    "launch_list_ns": [t for _, t in rows], **metrics,
})
summ_path.write_text(json.dumps(summ, indent=1, sort_keys=True))

md = [f"# ncu summary — {cfg} / {prec} ({tag})", "",
      f"Command: `tools/profile.sh {cfg} {prec} {tag}` under gpurun (1x B200, `--clock-control none`).", "",
      "## Launch list (bench.py --steps 5 --warmup 3; cold-cache, serialised)", "",
      "| kernel | launches | mean ns | share |", "|---|---|---|---|"]
names = {}
for n, t in rows:
    names.setdefault(n[:80], []).append(t)
for n, ts in names.items():
    md.append(f"| `{n}` | {len(ts)} | {sum(ts)/len(ts):.0f} | {sum(ts)/tot:.3f} |")
md += ["", "## Fused kernel, `--set full`", "", "| metric | value |", "|---|---|"]
for k, v in metrics.items():
    md.append(f"| {k} | {v if v is None else round(v, 3)} |")
md.append(f"| dram traffic per launch (read+write, bytes) | {traffic:.0f} |")
(out_dir / f"{tag}_{cfg}_{prec}.md").write_text("\n".join(md) + "\n")
print("\n".join(md))
