# Round bench lines (one B200): default workload (cfg2) with the CPU baseline,
# the other BASELINE configs, the reference arm, and the cfg2 launch list.
set -x
python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
for c in 1 3 4 5; do python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference_cfg2.json 2> gpurun_out/bench_reference_cfg2.err
python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/launches_cfg2.csv \
  python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
