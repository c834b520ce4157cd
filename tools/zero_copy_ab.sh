# e2e with zero-copy up to kZeroCopyMax rows: latency sweep (1..1,024 rows), larger batches, float64 apply
python bench.py --config hr_latency --rows 1024 --latency-sweep --no-cpu-baseline --no-parity-mode --no-e2e --steps 5 > gpurun_out/zc.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/zc.json'))
print('lat', {k: round(v['e2e_p50']*1000,1) for k,v in d['latency_sweep'].items()})"
for r in 2048 8192 32768 65536; do
  python bench.py --config hr --rows $r --no-cpu-baseline --no-parity-mode --inflight 0 --steps 10 > gpurun_out/zc.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/zc.json')); e=d['e2e']; print('rows=$r', round(e['ms_per_step']*1000,1), 'us; apply_f64', round(e['apply_f64']['ms_per_call']*1000,1), 'us')"
done
