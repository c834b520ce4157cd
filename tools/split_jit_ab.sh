#!/bin/bash
# NVRTC shapes with the split instance: parity/bitwise tests, then the paper model's
# (F=35, n_d=n_a=8, S=3) one-tile latency with and without it (same box)
[ -n "$SKIP_TESTS" ] || timeout 1200 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "runtime_compiled or random_shapes or geometry" > gpurun_out/jit_split.log 2>&1; echo "rc=$?" >> gpurun_out/jit_split.log
[ -n "$SKIP_TESTS" ] || grep -q "rc=0" gpurun_out/jit_split.log || exit 1
cat > /tmp/jit_lat.py <<'PY'
import sys, json, torch
sys.path.insert(0, ".")
import numpy as np
import paper_2510_19689_b200 as P
from paper_2510_19689_b200 import workloads as W
from paper_2510_19689_b200.device import DeviceRunner
from paper_2510_19689_b200.config import ModelConfig
cfg = ModelConfig(feature_count=35, n_classes=2, n_d=8, n_a=8, n_steps=3, seed=0)
from paper_2510_19689_b200.network import init_parameters
p = init_parameters(cfg)
res = {}
for prec in ("bf16", "tf32x3"):
    m = P.TabNetModel(config=cfg, params=p, norm_mean=np.zeros(35), norm_var=np.ones(35), model_version="paper", precision=prec)
    for rows in (1, 1024, 8192):
        r = DeviceRunner(m, rows, device=0)
        x = torch.randn(rows, 35, device="cuda")
        for _ in range(20): r.run(x)
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            r.run(x, stream=s)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for _ in range(50): r.run(x, stream=s)
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(4): g.replay()
        e1.record(); torch.cuda.synchronize()
        res[f"{prec}/{rows}"] = round(e0.elapsed_time(e1) / 200 * 1e3, 2)
print(json.dumps(res))
PY
for v in split nosplit split nosplit; do
  if [ $v = nosplit ]; then export TBN_K2_NO_SPLIT=1; else unset TBN_K2_NO_SPLIT; fi
  echo "$v $(timeout 300 python /tmp/jit_lat.py 2>&1 | tail -1)"
done
