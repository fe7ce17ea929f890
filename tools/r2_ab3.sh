#!/bin/bash
set -x
F=gpurun_out/ab3
mkdir -p $F
for rep in 1 2 3; do
for v in A B; do
  for w in llama_block ffnn; do
    FLOWPLACE_B200_LIB=$PWD/paper_2505_23131_b200/_flowplace_b200_$v.so timeout 300 python bench.py --steps 30 --warmup 5 --workload $w --no-cpu 2>/dev/null | tail -1 > $F/${v}_${w}_$rep.json
  done
done
done
timeout 600 python bench.py --workload ffnn --mode train --steps 10 > $F/bench_ffnn_train.json 2>/dev/null
timeout 600 python -m pytest tests/test_policy_gpu.py tests/test_train_gpu.py -q -x 2>&1 | tail -2 > $F/tests.txt
cat $F/tests.txt
