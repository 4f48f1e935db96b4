#!/bin/bash
# Round-2 final evidence (GPU box): full GPU suite, bench line + reference arm,
# ncu launch list of the bench command and of one block step (DRAM bytes per
# launch), ncu --set full of one chunk's GEMM launches, attention bench at four
# shapes, whole-decoder bench.  usage: bash tools/evidence_r02c.sh
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r02c_gpu_tests.log 2>&1
timeout 900 python bench.py > $O/r02c_bench.json 2> $O/r02c_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/r02c_bench_ref.json 2> $O/r02c_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 400 --csv --log-file $O/r02c_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-max-seq --no-e2e > $O/r02c_ncu_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file $O/r02c_launches.csv python tools/prof_op.py step > $O/r02c_ncu_list.log 2>&1
timeout 1800 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:mst_grouped \
  --launch-skip 6 --launch-count 5 -o $O/r02c_full python tools/prof_op.py step > $O/r02c_ncu_full.log 2>&1
ncu -i $O/r02c_full.ncu-rep --page raw --csv > $O/r02c_full_raw.csv 2>/dev/null
rm -f $O/r02c_full.ncu-rep
rm -f $O/r02c_attn_bench.jsonl
for a in "8192 32 8 128" "16384 32 8 128" "4096 32 8 128 2" "8192 16 16 64"; do
  timeout 300 python tools/attn_bench.py $a >> $O/r02c_attn_bench.jsonl 2>> $O/r02c_attn_bench.err
done
timeout 1200 python tools/model_bench.py 2 8192 32768 > $O/r02c_model_bench.jsonl 2> $O/r02c_model_bench.err
