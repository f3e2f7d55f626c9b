#!/bin/bash
# host/device stage traces (BDDC_B200_PROFILE=1) of one warm step per config
mkdir -p gpurun_out
for c in 3 4 5; do
BDDC_B200_PROFILE=1 BENCH_SETTLE=0 BENCH_CLOCK_MS=0 python bench.py --config $c --steps 2 --warmup 2 --no-cpu-baseline --apply-reps 2 > gpurun_out/r2_prof_cfg$c.json 2> gpurun_out/r2_prof_cfg$c.log
done
