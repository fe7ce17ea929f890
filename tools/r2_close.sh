#!/bin/bash
# closing check at HEAD: GPU tests, smoke, the headline bench lines, a torchrun N=2 smoke
set -x
F=gpurun_out/close
mkdir -p $F
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > $F/gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $F/smoke.txt 2>&1
B="timeout 900 python bench.py"
$B > $F/bench_llama_block.json 2>/dev/null
$B --workload ffnn > $F/bench_ffnn.json 2>/dev/null
$B --workload chainmm --batch 1024 > $F/bench_chainmm_b1024.json 2>/dev/null
$B --workload chainmm --batch 1 --steps 20 > $F/bench_chainmm_b1.json 2>/dev/null
$B --workload ffnn --full-outputs --no-cpu > $F/bench_ffnn_full_outputs.json 2>/dev/null
$B --workload ffnn --mode train --steps 10 > $F/bench_ffnn_train.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $F/launches_bench_ffnn.csv python bench.py --workload ffnn --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
bash tools/r2_dist.sh > $F/dist.txt 2>&1
cat $F/gputest.txt $F/smoke.txt $F/dist.txt
