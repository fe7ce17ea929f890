timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gnn_agg -s 8 -c 4 --csv --log-file gpurun_out/agg_ab.csv python bench.py --workload llama_block --mp-mode per_step --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 python bench.py --workload llama_block --mp-mode per_step --steps 3 --warmup 3 --no-cpu > gpurun_out/agg_ab_bench.json 2>&1
python tools/ncu_csv.py gpurun_out/agg_ab.csv; tail -1 gpurun_out/agg_ab_bench.json | cut -c1-200
