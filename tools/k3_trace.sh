#!/bin/bash
# Build the traced library, run one wide bf16 forward with the mapped-memory
# timeline (shows progress even if the kernel hangs), restore the library.
cp paper_2510_19689_b200/libtabnet_b200.so /tmp/lib_prod.so
TBN_TRACE_BUILD=1 python -m paper_2510_19689_b200.build --force > /dev/null
TBN_TRACE=1 timeout 60 python tools/k3_check.py > gpurun_out/k3_trace.txt 2>&1
echo "rc=$?" >> gpurun_out/k3_trace.txt
cp /tmp/lib_prod.so paper_2510_19689_b200/libtabnet_b200.so
