#!/bin/bash
# same-box A/B of the latency sweep (device + e2e p50/p99) with and without the split instance
for v in split nosplit split nosplit; do
  if [ $v = nosplit ]; then export TBN_K2_NO_SPLIT=1; else unset TBN_K2_NO_SPLIT; fi
  timeout 600 python bench.py --config hr_latency --rows 1024 --latency-sweep --no-cpu-baseline --no-parity-mode --steps 20 2>/dev/null > gpurun_out/lat_$v.json
  python -c "
import json; l=json.load(open('gpurun_out/lat_$v.json'))['latency_sweep']
print('$v', ' '.join(f\"{k}:{l[k]['device_p50']*1e3:.1f}/{l[k]['e2e_p50']*1e3:.1f}\" for k in l))"
done
