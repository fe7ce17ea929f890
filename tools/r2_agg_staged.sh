#!/bin/bash
# staged (TMA bulk) per_step aggregation vs the gather kernel (FP_AGG_VARIANT=9)
set -x
F=gpurun_out/aggs
mkdir -p $F
timeout 900 python -m pytest tests/test_per_step_gpu.py tests/test_tc_gpu.py -q -x 2>&1 | tail -5 > $F/tests.txt
for V in 0 9; do
  FP_AGG_VARIANT=$V timeout 600 python bench.py --workload llama_block --mp-mode per_step --steps 3 --warmup 2 --no-cpu > $F/bench_llama_V$V.json 2>$F/err_llama_V$V.txt
  FP_AGG_VARIANT=$V timeout 600 python bench.py --workload ffnn --mp-mode per_step --steps 3 --warmup 2 --no-cpu > $F/bench_ffnn_V$V.json 2>/dev/null
  FP_AGG_VARIANT=$V timeout 600 python bench.py --workload ffnn --mp-mode per_step --encoder tc --steps 3 --warmup 2 --no-cpu > $F/bench_ffnn_tc_V$V.json 2>/dev/null
  FP_AGG_VARIANT=$V timeout 600 python bench.py --workload llama_block --mp-mode per_step --encoder tc --steps 3 --warmup 2 --no-cpu > $F/bench_llama_tc_V$V.json 2>/dev/null
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size --clock-control none -k regex:gnn_agg -s 8 -c 4 --csv --log-file $F/ncu_staged.csv python bench.py --workload llama_block --mp-mode per_step --steps 1 --warmup 2 --no-cpu > /dev/null 2>&1
cat $F/tests.txt
