#!/bin/bash
# (historical: the TBN_K2_SPLIT_SM variant was measured slower and removed)
# the split instance with and without the shared sparsemax/mask loop (TBN_K2_SPLIT_SM),
# same box: bitwise geometry test first, then 8,192-row batches back to back (bench
# north_star_share) and the e2e latency sweep
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "geometry or random_shapes or runtime_compiled" > gpurun_out/splitsm_geom.log 2>&1; echo "geom rc=$?" >> gpurun_out/splitsm_geom.log
grep -q "geom rc=0" gpurun_out/splitsm_geom.log || exit 1
cp paper_2510_19689_b200/libtabnet_b200.so /tmp/lib_sm1.so
TBN_EXTRA_FLAGS="-DTBN_K2_SPLIT_SM=0" python -m paper_2510_19689_b200.build --force > /dev/null 2>&1
cp paper_2510_19689_b200/libtabnet_b200.so /tmp/lib_sm0.so
for v in sm1 sm0 sm1 sm0; do
  cp /tmp/lib_$v.so paper_2510_19689_b200/libtabnet_b200.so
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-parity-mode --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v share_us', round(d['north_star_share']['one_batch']['us'],2), 'hr65536_us', round(d['ms_per_step']*1e3,2))"
  timeout 600 python bench.py --config hr_latency --rows 1024 --latency-sweep --no-cpu-baseline --no-parity-mode --steps 20 2>/dev/null > gpurun_out/lat_$v.json
  python -c "
import json; l=json.load(open('gpurun_out/lat_$v.json'))['latency_sweep']
print('$v', ' '.join(f\"{k}:{l[k]['device_p50']*1e3:.1f}/{l[k]['e2e_p50']*1e3:.1f}\" for k in l))"
done
cp /tmp/lib_sm1.so paper_2510_19689_b200/libtabnet_b200.so
