#!/bin/bash
# A/B kernel variants on the GPU box: for each "label=flags" argument, rebuild
# the library with TBN_EXTRA_FLAGS=flags and run tools/scan_rows.py.
# Usage (under gpurun): bash tools/ab.sh hr "base=" "notoken=-DTBN_NO_TOKEN"
set -e
CFG=$1; shift
cp paper_2510_19689_b200/libtabnet_b200.so /tmp/lib_prod.so
for v in "$@"; do
  label=${v%%=*}; flags=${v#*=}
  TBN_EXTRA_FLAGS="$flags" python -m paper_2510_19689_b200.build --force > /dev/null
  echo "== $label ($flags)"
  python tools/scan_rows.py $CFG ${PRECS:-tf32x3 tf32} 2>&1 | sed "s/^/$label /"
  if [ -n "$QUICK" ]; then python tools/tc_quick.py 2>&1 | tail -12 | sed "s/^/$label /"; fi
done
cp /tmp/lib_prod.so paper_2510_19689_b200/libtabnet_b200.so
