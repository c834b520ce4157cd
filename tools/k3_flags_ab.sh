#!/bin/bash
# A/B K3 build flags on wide bf16 @ 262,144 rows (device time per batch)
cp paper_2510_19689_b200/libtabnet_b200.so /tmp/lib_prod.so
for v in "$@"; do
  label=${v%%=*}; flags=${v#*=}
  TBN_EXTRA_FLAGS="$flags" python -m paper_2510_19689_b200.build --force > /dev/null 2>&1 || { echo "$label BUILD FAILED"; continue; }
  for rep in 1 2; do
    python bench.py --config wide --rows 262144 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity-mode 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$label', d['ms_per_step'], d['roofline']['frac'])"
  done
done
cp /tmp/lib_prod.so paper_2510_19689_b200/libtabnet_b200.so
