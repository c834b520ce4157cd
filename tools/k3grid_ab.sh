# K3 / K3X grid-size A/B (TBN_K3_GRID): fewer CTAs = less row-state scratch in L2
for p in tf32x3 bf16; do for g in 148 128 112 96 74; do
  TBN_K3_GRID=$g timeout 300 python bench.py --config wide --precision $p --no-cpu-baseline --no-e2e --no-parity-mode --steps 5 --warmup 3 > gpurun_out/k3g.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/k3g.json')); print('$p grid=$g', round(d['ms_per_step'],3), 'ms')"
done; done
