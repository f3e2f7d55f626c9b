#!/bin/bash
# Closing pass of round 2 on one B200, at the final commit: the whole GPU suite
# and smoke() (they also absorb the start of the call, when the box is still
# busy with the push), the bench lines of every config and the reference arm,
# then the evidence taken under ncu (never a bench value): the cfg3 launch list,
# DRAM traffic of the leaf factorization and of one operator application
# (cfg3, cfg4), full captures of the fused coarse stage and the prolongation.
set -x
mkdir -p gpurun_out
P=r02k
python -m pytest tests -m gpu -x -q > gpurun_out/${P}_gputests_full.log 2>&1
tail -3 gpurun_out/${P}_gputests_full.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.log 2>&1
tail -1 gpurun_out/${P}_smoke.log
python bench.py > gpurun_out/${P}_bench_cfg3_run1.json 2> gpurun_out/${P}_bench_cfg3.err
for c in 1 2 4 5; do python bench.py --config $c > gpurun_out/${P}_bench_cfg$c.json 2> gpurun_out/${P}_bench_cfg$c.err; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${P}_bench_reference_cfg3.json 2> gpurun_out/${P}_bench_reference_cfg3.err
python bench.py > gpurun_out/${P}_bench_cfg3.json 2> /dev/null
BENCH_SETTLE=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${P}_launches_cfg3.csv \
  python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --apply-reps 1 > gpurun_out/${P}_ncu_launches3.log 2>&1
for spec in "3 leaf" "3 apply" "4 leaf" "4 apply"; do
  set -- $spec
  python tools/ncu_traffic.py --config $1 --phase $2 > /dev/null
  cnt=$(python tools/ncu_traffic.py --config $1 --phase $2 --count)
  skip=$(echo $cnt | python -c "import json,sys; print(json.load(sys.stdin)['skip'])")
  c=$(echo $cnt | python -c "import json,sys; print(json.load(sys.stdin)['count'])")
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -s $skip -c $c --csv --log-file gpurun_out/${P}_traffic_$2_cfg$1.csv python tools/ncu_traffic.py --config $1 --phase $2 > gpurun_out/${P}_traffic_$2_cfg$1.log 2>&1
done
NCU="ncu --set full --clock-control none --import-source on --profile-from-start off"
$NCU -k regex:k_coarse_explicit -c 1 -o gpurun_out/${P}_coarse_cfg3 -f python tools/prof_driver.py --config 3 --what apply > gpurun_out/${P}_ncu_coarse3.log 2>&1
$NCU -k regex:k_prolong_fused -c 1 -o gpurun_out/${P}_prolong_cfg3 -f python tools/prof_driver.py --config 3 --what apply > gpurun_out/${P}_ncu_prolong3.log 2>&1
ls gpurun_out | grep ${P} | wc -l
