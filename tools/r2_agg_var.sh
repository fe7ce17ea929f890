#!/bin/bash
# per_step aggregation kernel variants (FP_AGG_VARIANT): occupancy / messages in flight
set -x
F=gpurun_out/aggv
mkdir -p $F
for rep in 1 2; do
for V in 0 1 2 3; do
  FP_AGG_VARIANT=$V timeout 600 python bench.py --workload llama_block --mp-mode per_step --steps 3 --warmup 2 --no-cpu > $F/bench_V${V}_$rep.json 2>/dev/null
done
done
for V in 0 2 3; do
FP_AGG_VARIANT=$V timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem,launch__occupancy_limit_warps,launch__grid_size --clock-control none -k regex:gnn_agg -s 8 -c 2 --csv --log-file $F/ncu_V$V.csv python bench.py --workload llama_block --mp-mode per_step --steps 1 --warmup 2 --no-cpu > /dev/null 2>&1
done
