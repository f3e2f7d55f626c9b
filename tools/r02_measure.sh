#!/bin/bash
# Round-2 measurement pass on one B200: bench lines for cfg3 (headline) and
# cfg4, then the cfg3 launch list (ncu, one timed step, no settle steps).
set -x
mkdir -p gpurun_out
python bench.py --config 3 > gpurun_out/r2_bench_cfg3.json 2> gpurun_out/r2_bench_cfg3.err
python bench.py --config 4 --no-cpu-baseline > gpurun_out/r2_bench_cfg4.json 2> gpurun_out/r2_bench_cfg4.err
BENCH_SETTLE=0 python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --apply-reps 1 > gpurun_out/r2_plain3.log 2>&1 && \
BENCH_SETTLE=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2_launches_cfg3.csv \
  python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --apply-reps 1 > gpurun_out/r2_ncu_launches3.log 2>&1
