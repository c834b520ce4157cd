"""Cold start (PAPER.md:451's 3-5 s): model load + weight
packing + CUDA init + first forward, each in a FRESH process.

  python tools/cold_start.py            -> one JSON line
Arms (wide model, 8.2 MB .tbnt, and HR):
  * reference: the unmodified reference's load_model (pure-Python CRC-32C) +
    apply of one row on its CPU path (only when baseline/_ref is installed);
  * native: io.load_device_model (tbn_model_create_from_tbnt: parse, CRC,
    pack, upload in C++) + one forward through the C-ABI host call.
"""
import json
import os
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
CHILD = r'''
import sys, time, json
t0 = time.perf_counter()
sys.path.insert(0, {root!r})
import numpy as np
arm, path, prec = sys.argv[1], sys.argv[2], sys.argv[3]
data = open(path, "rb").read()
t1 = time.perf_counter()
if arm == "native":
    import paper_2510_19689_b200 as P
    from paper_2510_19689_b200 import io as PIO
    from paper_2510_19689_b200 import _native as N
    t2 = time.perf_counter()
    N.check(N.lib().tbn_device_init(0))
    tc = time.perf_counter()
    eng = PIO.load_device_model(data, precision=prec, device=0)
    t3 = time.perf_counter()
    x = np.zeros((1, eng.config.feature_count), np.float64)
    out = eng.forward_host_f64(x, 0)
    t4 = time.perf_counter()
else:
    sys.path.insert(0, {ref!r})
    from tabserve.model import io as RIO
    t2 = time.perf_counter()
    tc = time.perf_counter()
    m = RIO.load_model(data)
    t3 = time.perf_counter()
    x = np.zeros((1, m.config.feature_count))
    m.apply(x)
    t4 = time.perf_counter()
print(json.dumps(dict(startup_and_read_s=t1 - t0, import_s=t2 - t1, cuda_context_s=tc - t2,
                      load_parse_pack_upload_s=t3 - tc, first_forward_s=t4 - t3, total_s=t4 - t0)))
'''


def main():
    sys.path.insert(0, str(ROOT))
    import paper_2510_19689_b200 as P
    from paper_2510_19689_b200 import workloads as W
    ref = ROOT / "baseline" / "_ref"
    res = {}
    with tempfile.TemporaryDirectory() as td:
        for name, prec in (("wide", "bf16"), ("hr", "bf16")):
            path = Path(td) / f"{name}.tbnt"
            path.write_bytes(P.save_model(W.make_model(name, "trained")))
            child = CHILD.format(root=str(ROOT), ref=str(ref))
            for arm in ("native", "reference"):
                if arm == "reference" and not (ref / "tabserve").exists():
                    continue
                runs = []
                for _ in range(3):
                    r = subprocess.run([sys.executable, "-c", child, arm, str(path), prec], capture_output=True,
                                       text=True, timeout=300)
                    if r.returncode != 0:
                        runs.append({"error": r.stderr[-500:]})
                        break
                    runs.append(json.loads(r.stdout.strip().splitlines()[-1]))
                ok = [x for x in runs if "total_s" in x]
                res[f"{name}/{arm}"] = {"bytes": path.stat().st_size,
                                        "best": min(ok, key=lambda d: d["total_s"]) if ok else runs}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
