#!/bin/bash
# Closing check on one B200: the whole GPU suite and smoke() first (they also
# absorb the start of the call, when the box is still busy with the push), then
# the bench lines of every config and the reference arm.
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r02h_gputests_full.log 2>&1
tail -3 gpurun_out/r02h_gputests_full.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02h_smoke.log 2>&1
tail -1 gpurun_out/r02h_smoke.log
python bench.py > gpurun_out/r02h_bench_cfg3.json 2> gpurun_out/r02h_bench_cfg3.err
for c in 1 2 4 5; do python bench.py --config $c > gpurun_out/r02h_bench_cfg$c.json 2> gpurun_out/r02h_bench_cfg$c.err; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02h_bench_reference_cfg3.json 2> gpurun_out/r02h_bench_reference_cfg3.err
python bench.py > gpurun_out/r02h_bench_cfg3_again.json 2> /dev/null
