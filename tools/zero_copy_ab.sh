# e2e A/B: copy-engine chunks vs the kernel reading/writing the caller's pinned buffers (TBN_ZERO_COPY)
for c in hr bls adult; do for z in 0 1; do
  if [ $z = 1 ]; then export TBN_ZERO_COPY=1; else unset TBN_ZERO_COPY; fi
  python bench.py --config $c --no-cpu-baseline --no-parity-mode --steps 10 > gpurun_out/zc.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/zc.json')); e=d['e2e']; print('$c zc=$z', round(e['ms_per_step'],4), 'ms', '%.3g'%e['value'], 'device', round(d['ms_per_step']*1000,1), 'us')"
done; done
TBN_ZERO_COPY=1 python -m pytest tests/test_parity_gpu.py -q -m gpu -k "pinned_buffers" 2>&1 | tail -2
