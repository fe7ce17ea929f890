#!/bin/bash
set -x
F=gpurun_out/psab
mkdir -p $F
timeout 900 python -m pytest tests/test_per_step_gpu.py tests/test_agg_staged_gpu.py tests/test_train_gpu.py -q -x 2>&1 | tail -3 > $F/tests.txt
for v in A B; do
  for w in llama_block ffnn; do
    FLOWPLACE_B200_LIB=$PWD/paper_2505_23131_b200/_flowplace_b200_$v.so timeout 600 python bench.py --workload $w --mp-mode per_step --steps 3 --warmup 2 --no-cpu 2>/dev/null | tail -1 > $F/${v}_${w}.json
  done
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ps_step -s 20 -c 3 --csv --log-file $F/ps_B.csv python bench.py --workload llama_block --mp-mode per_step --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
cat $F/tests.txt
python tools/ncu_csv.py $F/ps_B.csv | tail -3
