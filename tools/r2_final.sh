#!/bin/bash
# Round-2 final refresh: bench lines (ours + the reference arm) for every
# workload, launch lists and ncu summaries -> gpurun_out/final2/ (copied into
# profiles/r2/final/ afterwards).  Run on the GPU box.
set -x
F=gpurun_out/final2
mkdir -p $F
B="timeout 900 python bench.py"
$B > $F/bench_llama_block.json 2> $F/bench_llama_block.err
$B --impl reference --steps 3 --warmup 1 > $F/ref_llama_block.json 2>/dev/null
$B --workload ffnn > $F/bench_ffnn.json 2>/dev/null
$B --workload ffnn --impl reference --steps 3 --warmup 1 > $F/ref_ffnn.json 2>/dev/null
$B --workload chainmm --batch 1024 > $F/bench_chainmm_b1024.json 2>/dev/null
$B --workload chainmm --batch 1024 --impl reference --steps 3 --warmup 1 > $F/ref_chainmm.json 2>/dev/null
$B --workload chainmm --batch 1 --steps 20 > $F/bench_chainmm_b1.json 2>/dev/null
$B --workload llama_layer --mode train --steps 10 > $F/bench_llama_layer_train.json 2>/dev/null
$B --workload llama_layer --mode train --impl reference --steps 3 --warmup 1 > $F/ref_llama_layer_train.json 2>/dev/null
$B --workload ffnn --mode train --steps 10 > $F/bench_ffnn_train.json 2>/dev/null
$B --workload ffnn --mp-mode per_step --steps 5 --no-cpu > $F/bench_ffnn_per_step.json 2>/dev/null
$B --workload ffnn --mp-mode per_step --steps 5 --no-cpu --encoder tc > $F/bench_ffnn_per_step_tc.json 2>/dev/null
$B --workload ffnn --mp-mode per_step --impl reference --steps 2 --warmup 1 > $F/ref_ffnn_per_step.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $F/launches_bench_llama_block.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $F/launches_bench_llama_layer_train.csv python bench.py --workload llama_layer --mode train --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rollout_kernel -s 3 -c 1 -o $F/prof_rollout_llama_block python bench.py --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:plc_replay -s 2 -c 1 -o $F/prof_replay_llama_layer python bench.py --workload llama_layer --mode train --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
ls -la $F
