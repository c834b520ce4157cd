#!/bin/bash
# What the driver runs at round end, in order: GPU tests, smoke, reference arm, our arm.
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/re_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/re_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/re_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/re_smoke.log
timeout 600 python bench.py --impl reference > gpurun_out/re_reference.json 2> gpurun_out/re_reference.err; echo "ref rc=$?" >> gpurun_out/re_reference.err
timeout 600 python bench.py > gpurun_out/re_bench.json 2> gpurun_out/re_bench.err; echo "bench rc=$?" >> gpurun_out/re_bench.err
