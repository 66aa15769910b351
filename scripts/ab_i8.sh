# usage: bash scripts/ab_i8.sh "<nvcc defines>" ... : builds each variant of the library in a
# scratch copy and prints the C4 (block0 1024) kernel times (dev aid for fold A/B on one box)
ROOT=$(pwd)
for v in "$@"; do
  D=/tmp/abv; rm -rf $D; mkdir -p $D
  cp -r $ROOT/bppsa_workloads $ROOT/oracle $ROOT/paper_1907_10134_b200 $ROOT/include $ROOT/scripts $D/
  (cd $D && BPPSA_NVCC_EXTRA="$v" python paper_1907_10134_b200/build.py --force > /dev/null 2>&1 || echo "build failed: $v")
  [ -z "$NOPREC" ] && (cd $D && python scripts/prec_ab.py 4096 | sed "s/^/[$v] /")
  for rep in 1 2; do
    echo "[$v]" $(cd $D && python scripts/kbench.py c4b1024 | grep -o 'kernels \[[0-9., ]*\]\|wgrad [0-9.]*')
  done
done
