#!/bin/bash
# One GPU call at a milestone: full -m gpu suite, smoke(), then round_measure.sh
# (bench line, ncu launch list, full captures).  usage: bash scripts/final_measure.sh TAG
TAG=${1:-run}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$TAG.log 2>&1
bash scripts/round_measure.sh $TAG
