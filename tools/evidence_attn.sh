#!/bin/bash
# Attention evidence (GPU box): throughput next to flash_attn / cuDNN SDPA at
# four shapes, and ncu --set full of the forward / backward kernels with the
# raw page exported.  usage: bash tools/evidence_attn.sh
O=gpurun_out
rm -f $O/r02_attn_bench.jsonl
for a in "8192 32 8 128" "16384 32 8 128" "4096 32 8 128 2" "8192 16 16 64"; do
  timeout 300 python tools/attn_bench.py $a >> $O/r02_attn_bench.jsonl 2>> $O/r02_attn_bench.err
done
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:attn_ \
  -o $O/r02_attn python tools/prof_op.py attn > $O/r02_ncu_attn.log 2>&1
ncu -i $O/r02_attn.ncu-rep --page raw --csv > $O/r02_attn_raw.csv 2>/dev/null
ncu -i $O/r02_attn.ncu-rep --page details --csv > $O/r02_attn_details.csv 2>/dev/null
rm -f $O/r02_attn.ncu-rep
