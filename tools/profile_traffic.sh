#!/bin/bash
# Steady-state DRAM bytes per launch of the fused kernel: ncu application
# replay without cache control on launch 16 of a rotating > L2 sequence
# (tools/prof_rot.py), i.e. the traffic the bench's timed graph sees.
#   bash tools/profile_traffic.sh <config> <precision> <tag>
CFG=${1:-hr}; PREC=${2:-bf16}; TAG=${3:-r2}
ncu --replay-mode application --cache-control none --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum \
    -k regex:"tabnet_(fused|rowthread|wide|forward)" -s 16 -c 1 --csv \
    --log-file gpurun_out/traffic_${CFG}_${PREC}_${TAG}.csv python tools/prof_rot.py --config $CFG --precision $PREC
