#!/bin/bash
# Build a libfrr variant with extra -D flags on one source file, for A/B timing
# with FRR_LIBRARY=tools/variants/libfrr_<name>.so.
# Usage: [REV=<git rev>] tools/build_variant.sh <name> <source.cu> [nvcc flags...]
# (REV: compile the file as of that revision, e.g. REV=HEAD for the baseline)
set -e
name=$1; src=$2; shift 2
cd "$(dirname "$0")/../paper_2501_07642_b200/csrc"
make -s >/dev/null
mkdir -p ../../tools/variants build/variants
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -Xptxas -v"
base=${src%.cu}
if [ -n "$REV" ]; then
  git show "$REV:./$src" > build/variants/rev_$src
  cp build/variants/rev_$src ./.rev_$src
  srcf=./.rev_$src
else
  srcf=$src
fi
nvcc $FLAGS "$@" -c $srcf -o build/variants/${base}_$name.o 2> build/variants/${base}_$name.log || { cat build/variants/${base}_$name.log; exit 1; }
objs=""
for f in frr_abi frr_gen frr_select frr_mma frr_mma_nt frr_rev; do
  [ "$f" = "$base" ] && objs="$objs build/variants/${base}_$name.o" || objs="$objs build/$f.o"
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../../tools/variants/libfrr_$name.so $objs
[ -n "$REV" ] && rm -f ./.rev_$src
echo "built tools/variants/libfrr_$name.so $(grep -o 'Used [0-9]* registers' build/variants/${base}_$name.log | tr '\n' ' ')"
