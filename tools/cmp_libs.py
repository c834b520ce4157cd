"""Bitwise A/B of two builds: the same forwards with the in-tree library and with
another one (argv[1]), compared array by array.  python tools/cmp_libs.py ALT.so"""
import sys, os, shutil, subprocess
sys.path.insert(0, ".")
import numpy as np
# run the same forwards with two libraries (subprocesses), compare bitwise
CHILD = r'''
import sys, numpy as np
sys.path.insert(0, ".")
import paper_2510_19689_b200 as P
from paper_2510_19689_b200 import workloads as W
out = {}
for name in ("hr", "adult", "bls"):
    for prec in ("bf16", "tf32", "tf32x3"):
        if name == "bls" and prec != "bf16": continue
        m = (P.TabNetRegressor if name == "bls" else P.TabNetModel).from_reference(W.make_model(name), precision=prec)
        x = W.make_inputs(W.WORKLOADS[name], 3000, seed=3).astype(np.float64)
        r = m.apply(x)
        out[f"{name}_{prec}"] = np.concatenate([r.logits.ravel(), r.masks.ravel(), r.importance.ravel()])
np.savez(sys.argv[1], **out)
'''
lib = "paper_2510_19689_b200/libtabnet_b200.so"
shutil.copy(lib, "/tmp/lib_cur.so")
subprocess.run([sys.executable, "-c", CHILD, "/tmp/a.npz"], check=True)
shutil.copy(sys.argv[1], lib)
subprocess.run([sys.executable, "-c", CHILD, "/tmp/b.npz"], check=True)
shutil.copy("/tmp/lib_cur.so", lib)
a, b = np.load("/tmp/a.npz"), np.load("/tmp/b.npz")
for k in a.files:
    print(k, "bitwise-equal" if np.array_equal(a[k], b[k]) else f"DIFF max {np.abs(a[k]-b[k]).max():.3e}")
