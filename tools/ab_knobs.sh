#!/bin/bash
# A/B tuning knobs of the current build: tools/ab_knobs.sh "k=v[:k=v]" "k=v" ...  (first is the baseline)
L=paper_2407_15892_b200/lib/libmst.so
base=$1; shift
for v in "$@"; do timeout 300 python tools/ab_block.py "$L:$base" "$L:$v" 8 | tail -3; done
