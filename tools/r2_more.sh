set -x
mkdir -p gpurun_out/more
timeout 600 python bench.py --steps 20 --warmup 5 --full-outputs --no-cpu > gpurun_out/more/bench_llama_full.json 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --workload ffnn --full-outputs --no-cpu > gpurun_out/more/bench_ffnn_full.json 2>&1
timeout 900 ncu --set full --clock-control none -k regex:gnn_agg -s 8 -c 2 -o gpurun_out/more/ps_agg_llama python bench.py --workload llama_block --mp-mode per_step --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:gnn_agg -s 8 -c 6 --csv --log-file gpurun_out/more/ps_agg_llama.csv python bench.py --workload llama_block --mp-mode per_step --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
tail -1 gpurun_out/more/bench_llama_full.json | cut -c1-200
tail -1 gpurun_out/more/bench_ffnn_full.json | cut -c1-200
