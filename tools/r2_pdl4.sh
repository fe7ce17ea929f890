#!/bin/bash
set -x
F=gpurun_out/pdl4
mkdir -p $F
timeout 900 python -m pytest tests/test_train_gpu.py tests/test_per_step_gpu.py tests/test_dist_gpu.py -q -x 2>&1 | tail -3 > $F/tests.txt
for rep in 1 2; do
for V in 1 0; do
  for w in ffnn llama_layer; do
  FP_PDL=$V timeout 300 python bench.py --workload $w --mode train --no-cpu --steps 10 > $F/bench_${w}_P${V}_$rep.json 2>/dev/null
  done
done
done
cat $F/tests.txt
