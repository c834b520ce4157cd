"""(python tools/serving_order_probe.py [freeze])  Is the occasional ~0.5 s p99 of the 256-row GPU serving case caused by the
preceding reference-CPU arm?  Runs the GPU 256-row case 3x, then the reference
16-row case, then the GPU 256-row case 3x again."""
import json
import sys
sys.path.insert(0, "tools")
import serving_bench as sb  # noqa: E402
import paper_2510_19689_b200 as P  # noqa: E402
from paper_2510_19689_b200 import workloads as W  # noqa: E402

base = W.make_model("hr", "trained")
gpu = P.TabNetModel.from_reference(base, precision="bf16")
c = base.config
cpu = sb.RefModel(config=sb.ModelConfig(feature_count=c.feature_count, n_classes=c.n_classes, n_d=c.n_d,
                                        n_a=c.n_a, n_steps=c.n_steps, gamma=c.gamma),
                  params=base.params, norm_mean=base.norm_mean, norm_var=base.norm_var,
                  model_version=base.model_version)


if len(sys.argv) > 1 and sys.argv[1] == "freeze":
    import gc
    gc.collect()
    gc.freeze()      # long-lived objects (torch, the models) out of the collector's scans
    print("gc frozen", flush=True)


def show(tag, r):
    print(tag, json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)


for i in range(3):
    show("gpu256", sb.run(gpu, 256, 400, 8, 256))
show("cpu16", sb.run(cpu, 16, 200, 32, 256))
for i in range(3):
    show("gpu256", sb.run(gpu, 256, 400, 8, 256))
show("gpu16", sb.run(gpu, 16, 2000, 32, 256))
for i in range(2):
    show("gpu256", sb.run(gpu, 256, 400, 8, 256))
