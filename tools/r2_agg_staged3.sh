#!/bin/bash
set -x
F=gpurun_out/aggs3
mkdir -p $F
timeout 900 python -m pytest tests/test_per_step_gpu.py tests/test_tc_encoder_gpu.py tests/test_train_gpu.py -q -x 2>&1 | tail -5 > $F/tests.txt
for w in llama_block ffnn; do
for enc in dmma tc; do
  timeout 600 python bench.py --workload $w --mp-mode per_step --encoder $enc --steps 3 --warmup 2 --no-cpu > $F/bench_${w}_${enc}.json 2>/dev/null
done
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:gnn_agg -s 8 -c 2 --csv --log-file $F/ncu_staged.csv python bench.py --workload llama_block --mp-mode per_step --steps 1 --warmup 2 --no-cpu > /dev/null 2>&1
cat $F/tests.txt
