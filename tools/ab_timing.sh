#!/bin/bash
# A/B the kernel variants in paper_2407_15892_b200/lib/libmst*.so with op_timing.py
for lib in paper_2407_15892_b200/lib/libmst*.so; do
  echo "=== $lib"
  MST_LIB=$PWD/$lib timeout 300 python tools/op_timing.py 2>&1 | grep -v "launch [1-9]"
done
