#!/bin/bash
# Round-2 closing measurement pass on one B200 (after the GPU tests are green):
# bench lines of every config (cpu_baseline included), the reference arm, the
# cfg3 launch list, DRAM traffic of the leaf factorization and of one operator
# application (cfg3, cfg4), and full ncu captures of the kernels changed since
# tools/r02_final.sh (fused coarse stage, leaf k_chol_dag with the front-major
# trailing tasks, copy sums).
set -x
mkdir -p gpurun_out
P=r02f
python bench.py > gpurun_out/${P}_bench_cfg3.json 2> gpurun_out/${P}_bench_cfg3.err
for c in 1 2 4 5; do python bench.py --config $c > gpurun_out/${P}_bench_cfg$c.json 2> gpurun_out/${P}_bench_cfg$c.err; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${P}_bench_reference_cfg3.json 2> gpurun_out/${P}_bench_reference_cfg3.err
BENCH_SETTLE=0 python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --apply-reps 1 > gpurun_out/${P}_plain3.log 2>&1 && \
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
$NCU -k regex:k_sum_copies -c 2 -o gpurun_out/${P}_sumcopies_cfg3 -f python tools/prof_driver.py --config 3 --what apply > gpurun_out/${P}_ncu_sumcopies3.log 2>&1
$NCU -k regex:k_chol_dag -c 1 -o gpurun_out/${P}_chol_cfg3 -f python tools/prof_driver.py --config 3 --what step > gpurun_out/${P}_ncu_chol3.log 2>&1
$NCU -k regex:k_sweep -c 2 -o gpurun_out/${P}_sweep_cfg3 -f python tools/prof_driver.py --config 3 --what apply > gpurun_out/${P}_ncu_sweep3.log 2>&1
ls -la gpurun_out | tail -30
