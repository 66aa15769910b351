# usage: bash scripts/ab_wgrad.sh v1 v2 ... (scripts/<v>.cu.txt variants of tc_wgrad.cu)
for v in "$@"; do
  cp scripts/$v.cu.txt paper_1907_10134_b200/csrc/tc_wgrad.cu
  python paper_1907_10134_b200/build.py --force > /dev/null || echo "build failed $v"
  echo $v $(python scripts/wg_time.py)
done
