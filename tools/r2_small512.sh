#!/bin/bash
set -x
F=gpurun_out/s512
mkdir -p $F
FP_SMALL_THREADS=512 timeout 900 python -m pytest tests/test_policy_gpu.py tests/test_train_gpu.py tests/test_heuristics_gpu.py -q -x 2>&1 | tail -3 > $F/tests.txt
for rep in 1 2; do
for V in 512 256; do
  for w in ffnn chainmm; do
  FP_SMALL_THREADS=$V timeout 300 python bench.py --workload $w --no-cpu --steps 30 > $F/bench_${w}_${V}_$rep.json 2>/dev/null
  done
done
done
for V in 512 256; do
FP_SMALL_THREADS=$V timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gnn_small -c 4 --csv --log-file $F/launches_$V.csv python bench.py --workload ffnn --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
done
cat $F/tests.txt
for V in 512 256; do python tools/ncu_csv.py $F/launches_$V.csv | tail -2; done
