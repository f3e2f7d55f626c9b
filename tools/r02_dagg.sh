#!/bin/bash
# Group size of k_chol_dag's plain task order (BDDC_B200_DAGG): time per call and
# DRAM bytes per launch on the cfg3 (512 x 1408, p 768) and cfg4 (216 x 1856, p 1216) leaf batches.
mkdir -p gpurun_out
for shape in "512 1408 768" "216 1856 1216"; do
  for G in 100000 96 64 48 32 24 16 12 8; do
    echo "== shape $shape G $G"
    BDDC_B200_DAGG=$G tools/chol_bench $shape 0 5 | head -1
  done
done > gpurun_out/dagg_times.log 2>&1
cat gpurun_out/dagg_times.log
for G in 100000 48 24 12; do
  BDDC_B200_DAGG=$G ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_chol_dag -s 1 -c 1 --csv --log-file gpurun_out/dagg_traffic_$G.csv tools/chol_bench 512 1408 768 0 1 > /dev/null 2>&1
  grep -h "k_chol_dag" gpurun_out/dagg_traffic_$G.csv | awk -F'","' -v g=$G '{print g, $(NF-3), $(NF-1), $NF}'
done
