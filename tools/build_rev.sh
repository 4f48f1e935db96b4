#!/bin/bash
# Build libmst.so from a git revision into paper_2407_15892_b200/lib/libmst_<name>.so (for A/B).
# usage: tools/build_rev.sh <rev> <name> [extra nvcc -D flags]
set -e
rev=$1; name=$2; shift 2
tmp=$(mktemp -d)
mkdir -p $tmp/csrc $tmp/include/mst
for f in $(git ls-tree --name-only $rev paper_2407_15892_b200/csrc/); do git show $rev:$f > $tmp/csrc/$(basename $f); done
for f in $(git ls-tree --name-only $rev include/mst/); do git show $rev:$f > $tmp/include/mst/$(basename $f); done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
  --expt-relaxed-constexpr -I $tmp/include -I $tmp/csrc "$@" -o paper_2407_15892_b200/lib/libmst_$name.so $tmp/csrc/*.cu
rm -rf $tmp
echo paper_2407_15892_b200/lib/libmst_$name.so
