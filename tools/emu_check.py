"""Dev: K2 single-pass modes against the rounding-faithful emulation
(oracle/tabnet_emulate.py) and the float64 oracle; exact modes' exempt/flip
counts at several delta.  python tools/emu_check.py"""
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
import paper_2510_19689_b200 as P
from paper_2510_19689_b200 import workloads as W
from oracle import tabnet_oracle as O, tabnet_emulate as E
from parity import compare


def rowstats(a, b, mass):
    me = np.abs(a["masks"] - b["masks"]).max(-1) / np.maximum(mass, 1e-30)
    ie = np.abs(a["importance"] - b["importance"]).max(-1)
    return (f"mask/rowmass max {me.max():.2e} p99.9 {np.quantile(me, 0.999):.2e} p99 {np.quantile(me, 0.99):.2e} "
            f"med {np.median(me):.2e} | imp max {ie.max():.2e} | prob max "
            f"{np.abs(a['probabilities'] - b['probabilities']).max():.2e} | class diff "
            f"{int(np.sum(np.argmax(a['probabilities'], 1) != np.argmax(b['probabilities'], 1)))}")


for name, rows in (("hr", 65536), ("adult", 4096), ("bls", 16384)):
    w = W.WORKLOADS[name]
    for regime, bias in (("trained", False), ("trained", True), ("init", False)):
        base = W.make_model(name, regime)
        params = base.params
        if bias:
            rng = np.random.default_rng(11)
            params = {k: (v + rng.normal(0.0, 0.3, v.shape) if k.endswith("_b") else v) for k, v in params.items()}
        x = W.make_inputs(w, rows)
        ref = None
        for prec in ("bf16", "tf32"):
            m = P.TabNetModel(config=base.config, params=params, norm_mean=base.norm_mean,
                              norm_var=base.norm_var, model_version="e", precision=prec)
            r = m.apply(x.astype(np.float64))
            got = dict(logits=r.logits, probabilities=r.probabilities, masks=r.masks, importance=r.importance)
            emu = E.apply_model_emulated(m, x, mode=prec)
            if ref is None:
                ref = O.apply_model(m, x.astype(np.float64))
            mass = np.abs(emu["masks"]).sum(-1)
            print(f"{name} {regime}{'+bias' if bias else ''} {prec} kernel-vs-emu : {rowstats(got, emu, mass)}", flush=True)
            print(f"{name} {regime}{'+bias' if bias else ''} {prec} kernel-vs-f64 : {rowstats(got, ref, mass)}", flush=True)
            print(f"{name} {regime}{'+bias' if bias else ''} {prec} emu-vs-f64    : {rowstats(emu, ref, mass)}", flush=True)

# exact modes: exempt and flip counts against delta
for name, rows in (("hr", 65536),):
    for prec in ("tf32x3", "fp32"):
        m = P.TabNetModel.from_reference(W.make_model(name, "trained"), precision=prec)
        x = W.make_inputs(W.WORKLOADS[name], rows).astype(np.float64)
        ref = O.apply_model(m, x, diagnostics=True)
        zs, tau = ref["z_shift"], ref["tau"]
        ref["margin"] = np.abs(zs - tau[..., None]).min(axis=2) / np.maximum(np.abs(zs).max(axis=2), 1e-300)
        p = np.sort(ref["probabilities"], axis=1)
        ref["top2_gap"] = p[:, -1] - p[:, -2]
        r = m.apply(x)
        got = dict(logits=r.logits, probabilities=r.probabilities, masks=r.masks, importance=r.importance)
        sup_bad = np.any((ref["masks"] > 0) != (r.masks > 0), axis=(0, 2))
        worst = ref["margin"].min(axis=0)[sup_bad]
        print(f"{name} {prec}: support-flip rows {int(sup_bad.sum())} (worst margin of a flip row "
              f"{worst.max() if worst.size else 0:.2e}); class flips "
              f"{int(np.sum(np.argmax(r.probabilities, 1) != np.argmax(ref['probabilities'], 1)))}")
        for d in (1e-4, 2e-5, 1e-5):
            rep = compare(ref, got, delta=d)
            print(f"   delta={d:g}: exempt {len(rep.exempt_rows)} ok={rep.ok} {rep.summary()[:300]}", flush=True)
