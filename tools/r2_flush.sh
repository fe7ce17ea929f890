#!/bin/bash
set -x
F=gpurun_out/flush
mkdir -p $F
timeout 900 python -m pytest tests/test_agg_staged_gpu.py -q -x 2>&1 | tail -15 > $F/tests.txt
for rep in 1 2; do
for V in sm ce; do
  for w in ffnn llama_block; do
  FP_E2E_FLUSH=$V timeout 300 python bench.py --workload $w --no-cpu --steps 30 > $F/bench_${w}_${V}_$rep.json 2>/dev/null
  done
done
done
FP_E2E_FLUSH=ce timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -c 30 --csv --log-file $F/launches_ce.csv python bench.py --workload ffnn --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
cat $F/tests.txt
python tools/ncu_csv.py $F/launches_ce.csv | tail -8
