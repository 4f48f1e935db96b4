#!/bin/bash
# Round-2 evidence after the paired-dW / row-scaled-head changes (GPU box):
# full GPU suite (+ the r02 parity file with its printed errors), bench line,
# ncu launch list of the bench command and of one block step, ncu --set full
# of one chunk's GEMM launches.  usage: bash tools/evidence_r02b.sh
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r02b_gpu_tests.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity_r02.py -q -s -p no:cacheprovider > $O/r02b_parity_r02_prints.log 2>&1
timeout 900 python bench.py > $O/r02b_bench.json 2> $O/r02b_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 400 --csv --log-file $O/r02b_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-max-seq --no-e2e > $O/r02b_ncu_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file $O/r02b_launches.csv python tools/prof_op.py step > $O/r02b_ncu_list.log 2>&1
timeout 1800 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:mst_grouped \
  --launch-skip 6 --launch-count 5 -o $O/r02b_full python tools/prof_op.py step > $O/r02b_ncu_full.log 2>&1
ncu -i $O/r02b_full.ncu-rep --page raw --csv > $O/r02b_full_raw.csv 2>/dev/null
rm -f $O/r02b_full.ncu-rep
