#!/bin/bash
# Build the engine with extra -D flags into tools/_exp/lib<name>.so (A/B timing):
#   bash tools/build_variant.sh <name> "-DLIN_CTX_SMEM=0 ..."
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; FLAGS=$2
W=/tmp/gwg_variant_$NAME
rm -rf $W; mkdir -p $W/paper_1210_7683_b200 $W/include
cp -r $ROOT/paper_1210_7683_b200/csrc $W/paper_1210_7683_b200/
cp $ROOT/include/*.h $W/include/
rm -rf $W/paper_1210_7683_b200/csrc/_build
make -s -j8 -C $W/paper_1210_7683_b200/csrc EXTRA="$FLAGS" LIB=$ROOT/tools/_exp/lib$NAME.so > $W/build.log 2>&1 || { tail -30 $W/build.log; exit 1; }
grep -A3 "Compiling entry function '_ZN3gwg19linear_solve_kernelILi4ELi2E" $W/paper_1210_7683_b200/csrc/_build/kernels_lin_a.ptxas.log | grep -i "spill" | head -1
echo "built tools/_exp/lib$NAME.so"
