#!/bin/bash
# primal-tree depth sweep on cfg3 / cfg4 (BDDC_B200_ROOT_DEPTH), short benches
mkdir -p gpurun_out
for c in 3 4; do for d in 0 1 2 3; do
BDDC_B200_ROOT_DEPTH=$d python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --apply-reps 5 > gpurun_out/r2_depth_cfg${c}_d$d.json 2>/dev/null
done; done
