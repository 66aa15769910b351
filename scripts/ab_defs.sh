# usage: bash scripts/ab_defs.sh "<script args>" "<nvcc defines>" ... : builds each variant of the
# library in a scratch copy and runs `python scripts/<script args>` twice in it (dev aid for A/B on one box)
ROOT=$(pwd)
CMD="$1"; shift
for v in "$@"; do
  D=/tmp/abv; rm -rf $D; mkdir -p $D
  cp -r $ROOT/bppsa_workloads $ROOT/oracle $ROOT/paper_1907_10134_b200 $ROOT/include $ROOT/scripts $D/
  (cd $D && BPPSA_NVCC_EXTRA="$v" python paper_1907_10134_b200/build.py --force > /dev/null 2>&1 || echo "build failed: $v")
  for rep in 1 2; do
    echo "[$v]" $(cd $D && python scripts/$CMD 2>&1 | tail -1)
  done
done
