#!/bin/bash
# synccheck on one K2 instance for build variants: bash tools/sync_ab.sh case "label=flags" ...
CASE=$1; shift
B=paper_2510_19689_b200/_build
cp paper_2510_19689_b200/libtabnet_b200.so /tmp/lib_prod.so
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Iinclude -Ipaper_2510_19689_b200/csrc --expt-relaxed-constexpr"
for v in "$@"; do
  label=${v%%=*}; flags=${v#*=}
  $NV $flags -c paper_2510_19689_b200/csrc/kernel_k2.cu -o /tmp/ab_obj.o
  objs=$(ls $B/*.o | grep -v "/kernel_k2.cu.o")
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o paper_2510_19689_b200/libtabnet_b200.so $objs /tmp/ab_obj.o -ldl
  compute-sanitizer --tool synccheck --print-limit 3 python tools/sanitize_run.py $CASE > /tmp/sync_$label.log 2>&1
  echo "$label: $(grep -E 'ERROR SUMMARY' /tmp/sync_$label.log | tail -1)"
  grep -v "Host Frame" /tmp/sync_$label.log | grep -A4 "Barrier error" | head -6
done
cp /tmp/lib_prod.so paper_2510_19689_b200/libtabnet_b200.so
