set -x
BPPSA_NVCC_EXTRA="-DBPPSA_F8_TRACE" python paper_1907_10134_b200/build.py --force > gpurun_out/r8_build.log 2>&1
python scripts/r8_trace.py 2>&1 | tee gpurun_out/r8_trace.txt
