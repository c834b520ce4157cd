#!/bin/bash
# ncu evidence for profiles/: (1) the launch list of a short bench run (device
# time per launch, cold-cache, serialised) and (2) one --set full capture of the
# fused kernel.  Run under gpurun on ONE GPU; outputs land in gpurun_out/.
#   bash tools/profile.sh <config> <precision> <tag>     (ROWS=n overrides the batch)
set -e
CFG=${1:-hr}; PREC=${2:-tf32x3}; TAG=${3:-r1}
RARG=""; [ -n "$ROWS" ] && RARG="--rows $ROWS"
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
    --log-file gpurun_out/launches_${CFG}_${PREC}_${TAG}.csv \
    python bench.py --config $CFG --precision $PREC --steps 5 --warmup 3 --no-cpu-baseline --no-e2e $RARG > /dev/null
ncu --set full --import-source on --clock-control none -k regex:"tabnet_(fused|rowthread|wide)" -s 3 -c 1 \
    -o gpurun_out/full_${CFG}_${PREC}_${TAG} python tools/prof_run.py --config $CFG --precision $PREC $RARG > /dev/null
