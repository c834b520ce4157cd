for c in adult/bf16 aux; do
compute-sanitizer --tool memcheck --leak-check full --print-limit 20 python tools/sanitize_run.py $c > gpurun_out/mc_${c//\//_}.log 2>&1
grep "ERROR SUMMARY" gpurun_out/mc_${c//\//_}.log
done
python - <<'PY'
import sys, gc
sys.path.insert(0, ".")
import paper_2510_19689_b200 as P
from paper_2510_19689_b200 import workloads as W
m = W.make_engine_model("adult", "trained", precision="bf16", device=0)
print("refs to model:", sys.getrefcount(m))
m.apply(W.make_inputs(W.WORKLOADS["adult"], 37).astype("float64"))
print("refs after apply:", sys.getrefcount(m), [type(r).__name__ for r in gc.get_referrers(m)])
PY
