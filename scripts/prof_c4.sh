#!/bin/bash
# ncu launch list + full capture of the named kernels on the C4 kbench (dev aid)
set -x
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_kb.csv python scripts/kbench.py c4 > /dev/null 2>&1
for k in "$@"; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_$k python scripts/kbench.py c4 > /dev/null 2>&1
done
