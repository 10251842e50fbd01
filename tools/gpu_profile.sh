#!/bin/bash
# Run on the GPU box (under gpurun): launch list of a short bench run and one
# full ncu capture of the persistent MIS-2 kernel.  Outputs in gpurun_out/.
set -x
TAG=${1:-r01}
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_under_ncu_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:mis2_persistent -s 2 -c 1 \
    -o gpurun_out/prof_${TAG} python tools/ncu_mis2.py 1 > gpurun_out/ncu_full_${TAG}.log 2>&1
