"""Fold steady-state DRAM captures (tools/profile_traffic.sh, ncu application
replay without cache control on launch 16 of a rotating > L2 sequence) into
profiles/ncu_summary.json as `dram_bytes_per_launch_steady` (+ per row);
bench.py reports that as roofline.traffic.
    python tools/update_traffic.py r2"""
import csv
import io
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2510_19689_b200 import workloads as W  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r2"
summ_p = ROOT / "profiles" / "ncu_summary.json"
summ = json.loads(summ_p.read_text()) if summ_p.exists() else {}
for f in sorted((ROOT / "gpurun_out").glob(f"traffic_*_{tag}.csv")):
    cfg, prec = f.stem.split("_")[1:3]
    txt = f.read_text().splitlines()
    hdr = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
    m = {r["Metric Name"]: float(r["Metric Value"]) for r in csv.DictReader(io.StringIO("\n".join(txt[hdr:])))}
    w = W.WORKLOADS[cfg]
    rows = min(w.batch, 262144)
    b = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
    e = summ.setdefault(f"{cfg}/{prec}", {})
    e.update({"dram_bytes_per_launch_steady": b, "dram_read_steady": m["dram__bytes_read.sum"],
              "dram_write_steady": m["dram__bytes_write.sum"], "steady_rows": rows,
              "dram_bytes_per_row_steady": b / rows,
              "algorithmic_bytes_per_row": W.algorithmic_counts(w)["bytes_per_row"],
              "steady_duration_ns": m["gpu__time_duration.sum"],
              "steady_how": f"ncu --replay-mode application --cache-control none, launch 16 of back-to-back "
                            f"forwards over rotating input/output sets > L2 (tools/profile_traffic.sh, {tag})"})
    print(f"{cfg}/{prec}: {b / rows:.0f} B/row DRAM (algorithmic {e['algorithmic_bytes_per_row']})")
summ_p.write_text(json.dumps(summ, indent=1, sort_keys=True))
