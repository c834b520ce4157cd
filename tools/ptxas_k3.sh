#!/bin/bash
# ptxas register/spill report for the K3 instance(s) (dev aid)
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xptxas -v -Iinclude -Ipaper_2510_19689_b200/csrc \
  $TBN_EXTRA_FLAGS -c paper_2510_19689_b200/csrc/kernel_k3.cu -o /tmp/k3.o 2>&1 | grep -A2 "tabnet_wide" | grep -E "registers|spill"
