"""First use of each kernel family in a FRESH process through the host call
(tbn_forward_host_f64), which captures its copies and launch as a CUDA graph:
any one-time device setup a launcher does lazily (shared-memory attributes,
the K3 L2 persisting set-aside) must not run inside that capture."""
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent

CHILD = r'''
import sys
sys.path.insert(0, {root!r})
import numpy as np
import paper_2510_19689_b200 as P
from paper_2510_19689_b200 import io as PIO
from paper_2510_19689_b200 import workloads as W
name, prec = sys.argv[1], sys.argv[2]
eng = PIO.load_device_model(P.save_model(W.make_model(name, "trained")), precision=prec, device=0)
x = W.make_inputs(W.WORKLOADS[name], 5).astype(np.float64)
out = eng.forward_host_f64(x, 0)
assert np.all(np.isfinite(out["probabilities"])) and np.allclose(out["masks"].sum(-1), 1.0, atol=1e-3)
print("ok")
'''


@pytest.mark.gpu
@pytest.mark.parametrize("name,prec", [("wide", "bf16"), ("hr", "bf16"), ("hr", "tf32x3"), ("bls", "tf32x3"),
                                       ("wide", "fp32"), ("wide", "tf32x3")])
def test_first_forward_in_fresh_process(name, prec):
    r = subprocess.run([sys.executable, "-c", CHILD.format(root=str(ROOT)), name, prec],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]
