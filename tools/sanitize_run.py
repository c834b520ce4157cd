"""One small forward of every kernel instance (K1/K2/K3/CUDA-core, the
standalone sparsemax, batch statistics, partition means, preprocessing) for
compute-sanitizer runs (tools/sanitize.sh).  Rows span a partial tile and a
CTA with warps without rows."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2510_19689_b200 as P
from paper_2510_19689_b200 import workloads as W
from paper_2510_19689_b200.device import DeviceRunner

which = sys.argv[1] if len(sys.argv) > 1 else "all"
cases = [("adult", "bf16"), ("adult", "tf32x3"), ("hr", "bf16"), ("hr", "tf32"), ("hr", "tf32x3"),
         ("bls", "bf16"), ("bls", "tf32x3"), ("bls", "tf32"), ("wide", "bf16"), ("wide", "tf32x3"), ("hr", "fp32"), ("wide", "fp32")]
for name, prec in cases:
    if which != "all" and which != f"{name}/{prec}":
        continue
    m = W.make_engine_model(name, "trained", precision=prec, device=0)
    rows = 300 if name != "wide" else 160
    r = DeviceRunner(m, rows, device=0)
    x = torch.from_numpy(W.make_inputs(W.WORKLOADS[name], rows)).cuda()
    r.run(x)
    torch.cuda.synchronize()
    r.check_finite()
    from paper_2510_19689_b200 import _native as N
    rp = DeviceRunner(m, 600 if name != "wide" else 160, device=0, flags=N.FLAG_PACKED)   # packed geometry
    rp.run(torch.from_numpy(W.make_inputs(W.WORKLOADS[name], 600 if name != "wide" else 160)).cuda())
    torch.cuda.synchronize()
    rp.check_finite()
    del rp
    m.apply(x[:37].double().cpu().numpy(), use_batch_stats=True)   # batch-stats kernel + host path
    # zero-copy host path: the kernel reads/writes the caller's page-locked buffers
    xp = x.cpu().pin_memory()
    op = {k: torch.empty(v.shape, dtype=v.dtype).pin_memory().numpy() for k, v in r.views(rows).items()}
    m.engine().forward_host_f32(xp.numpy(), 0, op)
    del xp, op
    print("ok", name, prec, flush=True)
    del r, m
if which in ("all", "jit"):
    # a runtime-compiled (NVRTC) K2 shape: the paper's own model (F=35, n_d=n_a=8, S=3),
    # its latency instance (300 rows) and throughput instance (packed, 1,200 rows)
    cfg = P.ModelConfig(feature_count=35, n_classes=2, n_d=8, n_a=8, n_steps=3, seed=0)
    rng = np.random.default_rng(3)
    for prec in ("bf16", "tf32x3"):
        mj = P.TabNetModel(config=cfg, params=P.init_parameters(cfg), norm_mean=rng.standard_normal(35),
                           norm_var=rng.uniform(0.5, 2.0, 35), model_version="jit35", precision=prec)
        from paper_2510_19689_b200 import _native as N
        for rows, fl in ((300, 0), (1200, N.FLAG_PACKED)):
            rj = DeviceRunner(mj, rows, device=0, flags=fl)
            rj.run(torch.from_numpy(np.random.default_rng(rows).standard_normal((rows, 35)).astype(np.float32)).cuda())
            torch.cuda.synchronize()
            rj.check_finite()
            del rj
        del mj
    print("ok jit", flush=True)
if which in ("all", "aux"):
    print(P.sparsemax(np.random.default_rng(0).standard_normal((100, 35))).shape)
    print(P.sparsemax(np.random.default_rng(0).standard_normal((10, 700))).shape)   # float64 kernel
    from paper_2510_19689_b200 import interpret
    m = W.make_engine_model("hr", "trained", precision="bf16", device=0)
    interpret.stability_score(m, W.make_inputs(W.WORKLOADS["hr"], 400).astype(np.float64), 4)
    # the same partition means over an importance buffer written with plain
    # stores (the CUDA-core fp32 kernel) instead of TMA bulk stores: initcheck
    # does not track cp.async.bulk writes, so only this one is meaningful to it
    mf = W.make_engine_model("hr", "trained", precision="fp32", device=0)
    interpret.stability_score(mf, W.make_inputs(W.WORKLOADS["hr"], 400).astype(np.float64), 4)
    print("ok aux", flush=True)
import gc
for k in list(globals()):
    if k in ("m", "r", "x", "xp", "op", "mf"):
        del globals()[k]
gc.collect()
torch.cuda.synchronize()
torch.cuda.empty_cache()
if hasattr(torch._C, "_host_emptyCache"):      # torch's pinned-memory cache (else reported as leaks)
    torch._C._host_emptyCache()
