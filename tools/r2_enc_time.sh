#!/bin/bash
set -x
F=gpurun_out/enc
mkdir -p $F
timeout 300 python tools/small_timing.py ffnn > $F/small_ffnn.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $F/launches_llama.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
python tools/ncu_csv.py $F/launches_llama.csv | tail -24
tail -12 $F/small_ffnn.txt
