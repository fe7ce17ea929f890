#!/bin/bash
set -x
F=gpurun_out/pdl5
mkdir -p $F
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $F/tests.txt
for V in 1 0; do
  for w in ffnn llama_layer; do
  FP_PDL=$V timeout 300 python bench.py --workload $w --mode train --no-cpu --steps 10 > $F/bench_train_${w}_P${V}.json 2>/dev/null
  done
  for w in ffnn llama_block; do
  FP_PDL=$V timeout 300 python bench.py --workload $w --mp-mode per_step --no-cpu --steps 3 --warmup 2 > $F/bench_ps_${w}_P${V}.json 2>/dev/null
  done
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $F/smoke.txt 2>&1
cat $F/tests.txt $F/smoke.txt
