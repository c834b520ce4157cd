#!/bin/bash
# Build the timeline-instrumented library into a scratch copy, run one forward, restore.
set -e
cp paper_2510_19689_b200/libtabnet_b200.so /tmp/lib_prod.so
TBN_TRACE_BUILD=1 python -m paper_2510_19689_b200.build --force > /dev/null
python tools/trace_run.py "$@" 2> gpurun_out/trace_$1_$2.txt
cp /tmp/lib_prod.so paper_2510_19689_b200/libtabnet_b200.so
