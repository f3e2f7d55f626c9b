#!/bin/bash
# kernel durations inside one preconditioner + Schur application (ncu launch
# list of the profiled region) vs the event-timed application: launch gaps
mkdir -p gpurun_out
for c in 3 4; do
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r2_apply_launches_cfg$c.csv python tools/prof_driver.py --config $c --what apply > gpurun_out/r2_apply_launches_cfg$c.log 2>&1
done
