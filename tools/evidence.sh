#!/bin/bash
# Round-end evidence refresh on the GPU box (dev tool): bench line, ncu launch
# list of one block step + full captures of one chunk's five GEMM launches,
# M sweep / long context / max-seq, per-launch timing.  Writes gpurun_out/ev_*.
# usage (from the repo root, through gpurun): bash tools/evidence.sh
set -x
O=gpurun_out
timeout 900 python bench.py > $O/ev_bench.json 2> $O/ev_bench.err
timeout 300 python tools/step_timing.py > $O/ev_step_timing.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file $O/ev_launches.csv python tools/prof_op.py step > $O/ev_ncu_list.log 2>&1
timeout 1800 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:mst_grouped \
  --launch-skip 6 --launch-count 5 -o $O/ev_full python tools/prof_op.py step > $O/ev_ncu_full.log 2>&1
ncu -i $O/ev_full.ncu-rep --page raw --csv > $O/ev_full_raw.csv 2>/dev/null
rm -f $O/ev_full.ncu-rep
timeout 900 python tools/sweep.py sweep-m > $O/ev_sweeps.jsonl 2> $O/ev_sweeps.err
timeout 900 python tools/sweep.py long >> $O/ev_sweeps.jsonl 2>> $O/ev_sweeps.err
timeout 900 python tools/sweep.py sweep-m2 > $O/ev_config2_msweep.jsonl 2>> $O/ev_sweeps.err
timeout 900 python tools/sweep.py max-seq >> $O/ev_sweeps.jsonl 2>> $O/ev_sweeps.err
