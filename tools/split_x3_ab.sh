#!/bin/bash
# 3xTF32 (the Python default) split instance: bitwise geometry tests, then same-box A/B of
# one-tile batches (device, L2 flushed) and the float64 apply() call for small batches
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "geometry or random_shapes or runtime_compiled or parity" > gpurun_out/x3_geom.log 2>&1; echo "geom rc=$?" >> gpurun_out/x3_geom.log
grep -q "geom rc=0" gpurun_out/x3_geom.log || exit 1
for v in split nosplit split nosplit; do
  if [ $v = nosplit ]; then export TBN_K2_NO_SPLIT=1; else unset TBN_K2_NO_SPLIT; fi
  for r in 1 1024 8192; do
    timeout 300 python bench.py --config hr8 --precision tf32x3 --rows $r --no-cpu-baseline --no-e2e --no-parity-mode --steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', $r, 'flushed_us', round(d['ms_per_step']*1e3,2))"
  done
  echo "$v apply_f64_us $(timeout 300 python tools/apply_small.py tf32x3)"
done
