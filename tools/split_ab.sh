set -x
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "geometry" > gpurun_out/split_geom.log 2>&1; echo "geom rc=$?" >> gpurun_out/split_geom.log
for v in split nosplit split nosplit; do
  if [ $v = nosplit ]; then export TBN_K2_NO_SPLIT=1; else unset TBN_K2_NO_SPLIT; fi
  for r in 1 1024 8192; do
    timeout 300 python bench.py --config hr8 --rows $r --no-cpu-baseline --no-e2e --no-parity-mode --steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', $r, 'flushed_ms', round(d['ms_per_step']*1e3,2), 'p50', round(d['latency_ms']['p50']*1e3,2), 'steady', d.get('steady_state') and round(d['steady_state']['value']/1e9,3))"
  done
done > gpurun_out/split_ab.txt 2>&1
