mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r01o.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r01o.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r01o.log 2>&1
bash scripts/round_measure.sh r01o
