#!/bin/bash
# PDL A/B (FP_PDL=0 turns programmatic dependent launch off) + GPU tests
set -x
F=gpurun_out/pdl
mkdir -p $F
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > $F/tests.txt
for rep in 1 2; do
for V in 1 0; do
  for w in llama_block ffnn; do
  FP_PDL=$V timeout 300 python bench.py --workload $w --no-cpu --steps 30 > $F/bench_${w}_P${V}_$rep.json 2>/dev/null
  done
done
done
FP_PDL=1 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $F/smoke.txt 2>&1
cat $F/tests.txt $F/smoke.txt
