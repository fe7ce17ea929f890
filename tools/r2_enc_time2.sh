#!/bin/bash
set -x
F=gpurun_out/enc2
mkdir -p $F
timeout 300 python tools/small_timing.py ffnn > $F/small_ffnn.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $F/launches_llama.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
for w in llama_block ffnn; do timeout 300 python bench.py --workload $w --no-cpu --steps 30 > $F/bench_$w.json 2>/dev/null; done
python tools/ncu_csv.py $F/launches_llama.csv | tail -9
tail -4 $F/small_ffnn.txt
