#!/bin/bash
# Build the traced library, run one wide bf16 forward of ROWS rows with the
# clock64 timeline (TBN_TRACE), restore the library.
cp paper_2510_19689_b200/libtabnet_b200.so /tmp/lib_prod.so
TBN_TRACE_BUILD=1 python -m paper_2510_19689_b200.build --force > /dev/null
timeout 60 python tools/trace_run.py bf16 ${ROWS:-128} wide 2> gpurun_out/k3_trace.txt > /dev/null
echo "rc=$?" >> gpurun_out/k3_trace.txt
cp /tmp/lib_prod.so paper_2510_19689_b200/libtabnet_b200.so
