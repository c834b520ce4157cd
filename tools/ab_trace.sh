#!/bin/bash
# Timeline traces of kernel variants: bash tools/ab_trace.sh "label=flags" ...
set -e
cp paper_2510_19689_b200/libtabnet_b200.so /tmp/lib_prod.so
for v in "$@"; do
  label=${v%%=*}; flags=${v#*=}
  TBN_TRACE_BUILD=1 TBN_EXTRA_FLAGS="$flags" python -m paper_2510_19689_b200.build --force > /dev/null
  for p in ${PRECS:-tf32x3 tf32}; do
    python tools/trace_run.py $p ${ROWS:-128} 2> gpurun_out/trace_${label}_${p}.txt
  done
done
cp /tmp/lib_prod.so paper_2510_19689_b200/libtabnet_b200.so
