set -e
for spec in "2 leaf" "2 apply" "3 leaf" "3 apply" "4 leaf" "4 apply"; do
  set -- $spec
  python tools/ncu_traffic.py --config $1 --phase $2 > /dev/null
  cnt=$(python tools/ncu_traffic.py --config $1 --phase $2 --count)
  skip=$(echo $cnt | python -c "import json,sys; print(json.load(sys.stdin)['skip'])")
  c=$(echo $cnt | python -c "import json,sys; print(json.load(sys.stdin)['count'])")
  echo "$1 $2 $skip $c" >> gpurun_out/traffic_counts.txt
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -s $skip -c $c --csv --log-file gpurun_out/traffic_$2_cfg$1.csv python tools/ncu_traffic.py --config $1 --phase $2 > gpurun_out/traffic_$2_cfg$1.log 2>&1
done
