#!/bin/bash
set -x
F=gpurun_out/close2
mkdir -p $F
B="timeout 900 python bench.py"
$B > $F/bench_llama_block.json 2>/dev/null
$B --workload ffnn > $F/bench_ffnn.json 2>/dev/null
$B --workload chainmm --batch 1024 > $F/bench_chainmm_b1024.json 2>/dev/null
$B --workload chainmm --batch 1 --steps 20 > $F/bench_chainmm_b1.json 2>/dev/null
$B --workload ffnn --mode train --steps 10 > $F/bench_ffnn_train.json 2>/dev/null
$B --workload llama_layer --mode train --steps 10 > $F/bench_llama_layer_train.json 2>/dev/null
$B --workload llama_block --mp-mode per_step --steps 3 --warmup 3 --no-cpu > $F/bench_llama_block_per_step.json 2>/dev/null
$B --workload ffnn --mp-mode per_step --steps 5 --no-cpu > $F/bench_ffnn_per_step.json 2>/dev/null
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $F/gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $F/smoke.txt 2>&1
cat $F/gputest.txt $F/smoke.txt
