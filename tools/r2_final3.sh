#!/bin/bash
# Round-2 closing refresh (after the FULLD rollout specialisations and the
# staged per_step aggregation): roofline capture first (bench.py reads the
# fresh profiles/r2/rollout_ncu.json it writes), then bench lines (ours + the
# reference arm), launch lists and ncu summaries -> gpurun_out/final3/.
set -x
bash tools/roofline_capture.sh
F=gpurun_out/final3
mkdir -p $F
cp profiles/r2/rollout_ncu.json $F/rollout_ncu.json
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
$B --workload llama_block --batch 8192 --steps 5 --no-cpu > $F/bench_llama_block_b8192.json 2>/dev/null
$B --workload llama_block --full-outputs --no-cpu > $F/bench_llama_block_full_outputs.json 2>/dev/null
$B --workload ffnn --full-outputs --no-cpu > $F/bench_ffnn_full_outputs.json 2>/dev/null
$B --workload llama_block --mp-mode per_step --steps 3 --warmup 3 --no-cpu > $F/bench_llama_block_per_step.json 2>/dev/null
$B --workload llama_block --mp-mode per_step --encoder tc --steps 3 --warmup 3 --no-cpu > $F/bench_llama_block_per_step_tc.json 2>/dev/null
$B --workload ffnn --mp-mode per_step --steps 5 --no-cpu > $F/bench_ffnn_per_step.json 2>/dev/null
$B --workload ffnn --mp-mode per_step --steps 5 --no-cpu --encoder tc > $F/bench_ffnn_per_step_tc.json 2>/dev/null
$B --workload ffnn --mp-mode per_step --impl reference --steps 2 --warmup 1 > $F/ref_ffnn_per_step.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $F/launches_bench_llama_block.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $F/launches_bench_ffnn.csv python bench.py --workload ffnn --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $F/launches_bench_llama_layer_train.csv python bench.py --workload llama_layer --mode train --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $F/launches_per_step_llama_block.csv python bench.py --workload llama_block --mp-mode per_step --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rollout_kernel -s 3 -c 1 -o $F/prof_rollout_llama_block python bench.py --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:plc_replay -s 2 -c 1 -o $F/prof_replay_llama_layer python bench.py --workload llama_layer --mode train --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gnn_agg_staged -s 8 -c 1 -o $F/prof_agg_staged_llama_per_step python bench.py --workload llama_block --mp-mode per_step --steps 1 --warmup 2 --no-cpu > /dev/null 2>&1
for r in prof_rollout_llama_block prof_replay_llama_layer prof_agg_staged_llama_per_step; do
  python tools/ncu_summary.py $F/$r.ncu-rep > $F/${r}_summary.txt 2>&1
done
python tools/ncu_lines.py $F/prof_rollout_llama_block.ncu-rep --top 40 > $F/prof_rollout_llama_block_lines.txt 2>&1
python tools/ncu_lines.py $F/prof_agg_staged_llama_per_step.ncu-rep --top 30 > $F/prof_agg_staged_lines.txt 2>&1
rm -f $F/*.ncu-rep   # (gpurun copies back at most 64 MiB)
ls -la $F gpurun_out/roof
