#!/bin/bash
# compute-sanitizer passes over the persistent/dataflow kernels (one tool per run)
mkdir -p gpurun_out
python tools/sanitize_cases.py > gpurun_out/r2_sanitize_plain.log 2>&1 || exit 1
for tool in racecheck synccheck memcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py > gpurun_out/r2_sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r2_sanitize_$tool.log
done
