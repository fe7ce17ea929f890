#!/bin/bash
# staged aggregation: 1024 (default) vs 512 threads (FP_AGG_VARIANT=5)
set -x
F=gpurun_out/aggs2
mkdir -p $F
for V in 0 5; do
  for w in llama_block ffnn; do
  for enc in dmma tc; do
  FP_AGG_VARIANT=$V timeout 600 python bench.py --workload $w --mp-mode per_step --encoder $enc --steps 3 --warmup 2 --no-cpu > $F/bench_${w}_${enc}_V$V.json 2>/dev/null
  done
  done
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:gnn_agg -s 8 -c 2 --csv --log-file $F/ncu_staged.csv python bench.py --workload llama_block --mp-mode per_step --steps 1 --warmup 2 --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:gnn_agg -s 8 -c 2 --csv --log-file $F/ncu_staged_tc.csv python bench.py --workload llama_block --mp-mode per_step --encoder tc --steps 1 --warmup 2 --no-cpu > /dev/null 2>&1
