#!/bin/bash
# Round-2 evidence on the GPU box: GPU test suite, bench line, ncu launch list
# of the bench command and of one block step, full ncu captures of one chunk's
# five GEMM launches and of the attention kernels, attention throughput.
# usage (repo root, through gpurun): bash tools/evidence_r02.sh
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r02_gpu_tests.log 2>&1
timeout 900 python bench.py > $O/r02_bench.json 2> $O/r02_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file $O/r02_launches.csv python tools/prof_op.py step > $O/r02_ncu_list.log 2>&1
timeout 1800 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:mst_grouped \
  --launch-skip 6 --launch-count 5 -o $O/r02_full python tools/prof_op.py step > $O/r02_ncu_full.log 2>&1
ncu -i $O/r02_full.ncu-rep --page raw --csv > $O/r02_full_raw.csv 2>/dev/null
rm -f $O/r02_full.ncu-rep
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:attn_ \
  -o $O/r02_attn python tools/prof_op.py attn > $O/r02_ncu_attn.log 2>&1
ncu -i $O/r02_attn.ncu-rep --page raw --csv > $O/r02_attn_raw.csv 2>/dev/null
rm -f $O/r02_attn.ncu-rep
for a in "8192 32 8 128" "16384 32 8 128" "4096 32 8 128 2" "8192 16 16 64"; do
  timeout 300 python tools/attn_bench.py $a >> $O/r02_attn_bench.jsonl 2>> $O/r02_attn_bench.err
done
