# usage: bash scripts/ab_levels.sh v1 v2 ... (scripts/<v>.cu.txt variants of levels.cu), kbench c4b512 each
for v in "$@"; do
  cp scripts/$v.cu.txt paper_1907_10134_b200/csrc/levels.cu
  python paper_1907_10134_b200/build.py --force > /dev/null || echo "build failed $v"
  echo $v $(python scripts/kbench.py c4b512 | grep -o "kernels \[[0-9.]*, [0-9.]*, [0-9.]*, [0-9.]*")
done
