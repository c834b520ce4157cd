#!/bin/bash
# A/B variants of ONE kernel file on the GPU box: for each "label=flags", rebuild
# that object with the extra flags, relink, and time it (tools/k2_time.py).
#   bash tools/k2ab.sh kernel_k2.cu hr bf16 "base=" "v1=-DFOO"
set -e
SRC=$1; CFG=$2; PREC=$3; shift 3
B=paper_2510_19689_b200/_build
cp paper_2510_19689_b200/libtabnet_b200.so /tmp/lib_prod.so
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Iinclude -Ipaper_2510_19689_b200/csrc --expt-relaxed-constexpr"
for v in "$@"; do
  label=${v%%=*}; flags=${v#*=}
  $NV $flags -c paper_2510_19689_b200/csrc/$SRC -o /tmp/ab_obj.o
  objs=$(ls $B/*.o | grep -v "/$SRC.o")
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o paper_2510_19689_b200/libtabnet_b200.so $objs /tmp/ab_obj.o -ldl
  LABEL=$label timeout ${K2AB_TIMEOUT:-180} python tools/k2_time.py $CFG $PREC || echo "$label: failed or timed out"
done
cp /tmp/lib_prod.so paper_2510_19689_b200/libtabnet_b200.so
