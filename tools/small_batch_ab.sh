# host-path A/B: staged+graph small-batch path up to TBN_SMALL_BATCH rows, parallel copy-out above TBN_PAR_MIN values
run() {
env "$@" python bench.py --config hr_latency --rows 1024 --latency-sweep --no-cpu-baseline --no-parity-mode --no-e2e --steps 5 > gpurun_out/sb.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/sb.json'))
print('$*', {k: round(v['e2e_p50']*1000,1) for k,v in d['latency_sweep'].items()})"
}
run TBN_SMALL_BATCH=32
run TBN_SMALL_BATCH=1024 TBN_PAR_MIN=32768
run TBN_SMALL_BATCH=1024 TBN_PAR_MIN=65536
run TBN_SMALL_BATCH=1024 TBN_PAR_MIN=131072
