#!/bin/bash
set -x
F=gpurun_out/e2e
mkdir -p $F
for rep in 1 2; do
for w in ffnn llama_block chainmm; do
  timeout 300 python bench.py --workload $w --no-cpu --steps 30 > $F/bench_${w}_$rep.json 2>/dev/null
done
timeout 300 python bench.py --workload ffnn --mode train --no-cpu --steps 10 > $F/bench_ffnn_train_$rep.json 2>/dev/null
done
