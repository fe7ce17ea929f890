#!/bin/bash
# small-graph encoder: shared-memory-resident tables vs global (FP_SMALL_RESIDENT=0)
set -x
F=gpurun_out/smallres
mkdir -p $F
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > $F/tests.txt
for rep in 1 2; do
for R in 1 0; do
  for w in ffnn chainmm; do
  FP_SMALL_RESIDENT=$R timeout 300 python bench.py --workload $w --no-cpu --steps 30 > $F/bench_${w}_R${R}_$rep.json 2>/dev/null
  done
done
done
for R in 1 0; do
FP_SMALL_RESIDENT=$R timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gnn_small -c 6 --csv --log-file $F/launches_R$R.csv python bench.py --workload ffnn --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
done
cat $F/tests.txt
for R in 1 0; do python tools/ncu_csv.py $F/launches_R$R.csv | tail -3; done
