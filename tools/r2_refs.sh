#!/bin/bash
set -x
F=gpurun_out/refs
mkdir -p $F
B="timeout 900 python bench.py"
$B --impl reference --steps 3 --warmup 1 > $F/ref_llama_block.json 2>/dev/null
$B --workload ffnn --impl reference --steps 3 --warmup 1 > $F/ref_ffnn.json 2>/dev/null
$B --workload chainmm --batch 1024 --impl reference --steps 3 --warmup 1 > $F/ref_chainmm.json 2>/dev/null
$B --workload llama_layer --mode train --impl reference --steps 3 --warmup 1 > $F/ref_llama_layer_train.json 2>/dev/null
$B --workload llama_layer --mode train --steps 10 > $F/bench_llama_layer_train.json 2>/dev/null
$B --workload ffnn --mode train --steps 10 > $F/bench_ffnn_train.json 2>/dev/null
