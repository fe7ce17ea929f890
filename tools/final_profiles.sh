#!/bin/bash
# Round-end refresh of the bench lines, launch list and ncu captures under gpurun_out/final/
# (copied into profiles/ afterwards).  Run on the GPU box: gpurun -- bash tools/final_profiles.sh
mkdir -p gpurun_out/final
python bench.py > gpurun_out/final/bench_ffnn.json 2> gpurun_out/final/bench_ffnn.err
python bench.py --workload llama_block > gpurun_out/final/bench_llama_block.json 2>/dev/null
python bench.py --workload llama_layer --mode train --steps 10 > gpurun_out/final/bench_llama_layer_train.json 2>/dev/null
python bench.py --mode train --steps 10 > gpurun_out/final/bench_ffnn_train.json 2>/dev/null
python bench.py --mp-mode per_step --steps 5 > gpurun_out/final/bench_ffnn_per_step.json 2>/dev/null
python bench.py --workload llama_block --mp-mode per_step --steps 3 --warmup 3 > gpurun_out/final/bench_llama_block_per_step.json 2>/dev/null
python bench.py --workload chainmm --batch 1 --steps 20 > gpurun_out/final/bench_chainmm_b1.json 2>/dev/null
python bench.py --workload chainmm --batch 1024 --steps 20 > gpurun_out/final/bench_chainmm_b1024.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches_bench_ffnn.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:rollout_kernel -s 3 -c 1 -o gpurun_out/final/prof_rollout_ffnn python tools/profile_step.py --workload ffnn --steps 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:plc_grad -s 2 -c 1 -o gpurun_out/final/prof_plc_grad python bench.py --workload llama_layer --mode train --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
ls -la gpurun_out/final
