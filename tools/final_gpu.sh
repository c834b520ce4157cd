#!/bin/bash
# Round-end GPU evidence after the split instance: full GPU suite, sanitizers on
# the shapes with a split instance, latency sweep, default bench line.
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest3.log
timeout 300 python bench.py > gpurun_out/f_hr_bf16.json 2> gpurun_out/f_hr_bf16.err
timeout 600 python bench.py --config hr_latency --rows 1024 --latency-sweep --no-cpu-baseline --steps 20 > gpurun_out/f_lat.json 2> gpurun_out/f_lat.err
bash tools/sanitize.sh "hr/bf16 hr/tf32 adult/bf16 adult/tf32x3" > /dev/null 2>&1
