#!/bin/bash
# ncu capture of the rollout kernel inside the exact bench commands (traffic
# and executed instructions for bench.py's roofline / latency objects) ->
# gpurun_out/roof/*.csv, summarised into profiles/r2/rollout_ncu.json by
# tools/roofline_json.py.  Run on the GPU box.
mkdir -p gpurun_out/roof
M=dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__inst_executed.avg.per_cycle_active,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
for w in llama_block ffnn chainmm; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:rollout_kernel -s 3 -c 1 --csv \
    --log-file gpurun_out/roof/${w}_rollout.csv python bench.py --workload $w --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
done
timeout 600 ncu --metrics $M --clock-control none -k regex:rollout_kernel -s 3 -c 1 --csv \
  --log-file gpurun_out/roof/llama_layer_train.csv python bench.py --workload llama_layer --mode train --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:rollout_kernel -s 3 -c 1 --csv \
  --log-file gpurun_out/roof/ffnn_train.csv python bench.py --workload ffnn --mode train --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
python tools/roofline_json.py
