#!/bin/bash
# HEAD check on the GPU box: gpu tests, smoke, default + FFNN bench lines.
set -x
F=gpurun_out/head
mkdir -p $F
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > $F/gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $F/smoke.txt 2>&1
timeout 600 python bench.py > $F/bench_llama_block.json 2> $F/bench_llama_block.err
timeout 600 python bench.py --workload ffnn > $F/bench_ffnn.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $F/launches_ffnn.csv python bench.py --workload ffnn --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
cat $F/gputest.txt $F/smoke.txt
python tools/ncu_csv.py $F/launches_ffnn.csv 2>/dev/null | tail -20
