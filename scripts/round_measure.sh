#!/bin/bash
# One GPU call: bench line (default run), ncu launch list of the bench command,
# ncu --set full captures of the top kernels at config-4 size (dev aid).
# usage: bash scripts/round_measure.sh TAG
TAG=${1:-run}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --quick > /dev/null 2>&1
for k in tc_fold_i8 tc_walk_i8 tc_wgrad fold_up; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/full_${TAG}_$k python scripts/kbench.py c4b1024 > /dev/null 2>&1
done
ls -la gpurun_out | tail -8
