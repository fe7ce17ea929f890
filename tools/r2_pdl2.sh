#!/bin/bash
set -x
F=gpurun_out/pdl2
mkdir -p $F
for rep in 1 2; do
for V in 1 0; do
  for w in ffnn llama_block; do
  FP_PDL=$V timeout 300 python bench.py --workload $w --no-cpu --steps 30 > $F/bench_${w}_P${V}_$rep.json 2>/dev/null
  done
done
done
