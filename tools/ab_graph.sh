#!/bin/bash
# A/B kernel variants with CUDA-graph timing: for each "label=flags" argument,
# rebuild with TBN_EXTRA_FLAGS=flags and run tools/scan_graph.py (+ a quick
# oracle check).  Usage (under gpurun): bash tools/ab_graph.sh hr "base=" "x=-DFOO"
set -e
CFG=$1; shift
cp paper_2510_19689_b200/libtabnet_b200.so /tmp/lib_prod.so
for v in "$@"; do
  label=${v%%=*}; flags=${v#*=}
  TBN_EXTRA_FLAGS="$flags" python -m paper_2510_19689_b200.build --force > /dev/null
  echo "== $label ($flags)"
  python tools/scan_graph.py $CFG ${PRECS:-bf16} 2>&1 | grep -v Warn | sed "s/^/$label /"
  if [ -n "$QUICK" ]; then python tools/tc_quick.py 2>&1 | grep -E "^$CFG" | sed "s/^/$label /"; fi
done
cp /tmp/lib_prod.so paper_2510_19689_b200/libtabnet_b200.so
