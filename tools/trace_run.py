"""Dev aid: run one forward with TBN_TRACE=1 and print CTA 0's clock64 timeline.
    python tools/trace_run.py <precision> <rows> [config]"""
import os, sys
os.environ["TBN_TRACE"] = "1"
sys.path.insert(0, ".")
import torch
from paper_2510_19689_b200 import workloads as W
from paper_2510_19689_b200.device import DeviceRunner
prec = sys.argv[1] if len(sys.argv) > 1 else "tf32x3"
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 128
cfg = sys.argv[3] if len(sys.argv) > 3 else "hr"
m = W.make_engine_model(cfg, "trained", precision=prec, device=0)
outs = tuple(os.environ.get("TBN_OUTPUTS", "logits,probabilities,masks,importance,predicted_class").split(","))
r = DeviceRunner(m, rows, device=0, outputs=outs)
x = torch.from_numpy(W.make_inputs(W.WORKLOADS[cfg], rows)).cuda()
r.run(x); torch.cuda.synchronize()
r.run(x); torch.cuda.synchronize()
