set -x
for c in 2 3 4; do
  cnt=$(python tools/ncu_traffic.py --config $c --phase leaf --count)
  skip=$(echo $cnt | python -c "import json,sys; print(json.load(sys.stdin)['skip'])")
  n=$(echo $cnt | python -c "import json,sys; print(json.load(sys.stdin)['count'])")
  echo "$c leaf $skip $n" >> gpurun_out/traffic_counts.txt
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -s $skip -c $n --csv --log-file gpurun_out/traffic_leaf_cfg$c.csv python tools/ncu_traffic.py --config $c --phase leaf > gpurun_out/traffic_leaf_cfg$c.log 2>&1
done
cnt=$(python tools/ncu_traffic.py --config 2 --phase leaf --count)
skip=$(echo $cnt | python -c "import json,sys; print(json.load(sys.stdin)['skip'])")
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_chol_dag -s 0 -c 2 -o gpurun_out/chol_dag_cfg2 python tools/ncu_traffic.py --config 2 --phase leaf > gpurun_out/ncu_full.log 2>&1
