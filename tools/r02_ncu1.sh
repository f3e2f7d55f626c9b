#!/bin/bash
# targeted ncu --set full captures (one GPU): dataflow sweeps (cfg3, cfg4),
# leaf k_chol_dag (cfg3), k_syevx (cfg4)
set -x
mkdir -p gpurun_out
python tools/prof_driver.py --config 3 --what apply > gpurun_out/r2_pd3.log 2>&1 || exit 1
NCU="ncu --set full --clock-control none --import-source on --profile-from-start off"
$NCU -k regex:k_sweep -c 2 -o gpurun_out/r2_sweep_cfg3 -f python tools/prof_driver.py --config 3 --what apply > gpurun_out/r2_ncu_sweep3.log 2>&1
$NCU -k regex:k_sweep -c 2 -o gpurun_out/r2_sweep_cfg4 -f python tools/prof_driver.py --config 4 --what apply > gpurun_out/r2_ncu_sweep4.log 2>&1
$NCU -k regex:k_chol_dag -c 1 -o gpurun_out/r2_chol_cfg3 -f python tools/prof_driver.py --config 3 --what step > gpurun_out/r2_ncu_chol3.log 2>&1
$NCU -k regex:k_syevx -c 1 -o gpurun_out/r2_syevx_cfg4 -f python tools/prof_driver.py --config 4 --what step > gpurun_out/r2_ncu_syevx4.log 2>&1
ls -la gpurun_out
