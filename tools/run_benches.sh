#!/bin/bash
# Regenerate the round's evidence on ONE B200 (run under gpurun):
#   bench lines for every BASELINE config/mode -> gpurun_out/f_*.json,
#   then copy/summarize here with:  for f in gpurun_out/f_*.json ...; python tools/summarize_profiles.py
set -e
# bench lines only (tools/run_all.sh without the ncu captures)
python bench.py                                   > gpurun_out/f_hr_bf16.json
python bench.py --precision tf32   --no-cpu-baseline > gpurun_out/f_hr_tf32.json
python bench.py --precision tf32x3 --no-cpu-baseline > gpurun_out/f_hr_x3.json
python bench.py --config adult                    > gpurun_out/f_adult_bf16.json
python bench.py --config adult --precision tf32x3 --no-cpu-baseline > gpurun_out/f_adult_x3.json
python bench.py --config bls                      > gpurun_out/f_bls_bf16.json
python bench.py --config bls --precision tf32   --no-cpu-baseline > gpurun_out/f_bls_tf32.json
python bench.py --config bls --precision tf32x3 --no-cpu-baseline > gpurun_out/f_bls_x3.json
python bench.py --config bls --precision fp32   --no-cpu-baseline --steps 5 > gpurun_out/f_bls_fp32.json
python bench.py --config hr_latency --rows 1024 --latency-sweep --no-cpu-baseline --steps 20 > gpurun_out/f_lat.json
python bench.py --config wide --rows 262144 --steps 5 --warmup 3 > gpurun_out/f_wide_bf16.json
python bench.py --config wide --steps 3 --warmup 3 --no-e2e > gpurun_out/f_wide16m_bf16.json   # config 5: 2^24 rows streamed
python bench.py --config hr8 --rows 8192 --no-cpu-baseline > gpurun_out/f_hr8_share.json          # one GPU's share of 65,536 on 8
python bench.py --config wide --precision fp32 --rows 262144 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/f_wide_fp32.json
python bench.py --config wide --precision tf32x3 --rows 262144 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/f_wide_x3.json
python bench.py --config hr8 --rows 8192 --inflight 16 --no-cpu-baseline --no-e2e --no-parity-mode > gpurun_out/f_hr8_share16.json
python bench.py --impl reference                  > gpurun_out/f_reference.json
