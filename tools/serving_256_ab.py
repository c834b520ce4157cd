import sys, json
sys.path.insert(0, 'tools')
import serving_bench as sb
import paper_2510_19689_b200 as P
from paper_2510_19689_b200 import workloads as W
gpu = P.TabNetModel.from_reference(W.make_model("hr", "trained"), precision="bf16")
for rep in range(3):
    r = sb.run(gpu, 256, 400, 8, 256)
    print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in r.items()}))
