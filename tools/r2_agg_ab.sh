#!/bin/bash
# per_step aggregation: rows-per-unit A/B (FP_AGG_ROWS 1/2/4), parity tests,
# ncu DRAM bytes of the batched kernel.  Run on the GPU box.
set -x
F=gpurun_out/agg
mkdir -p $F
timeout 900 python -m pytest tests/test_per_step_gpu.py -q -x 2>&1 | tail -5 > $F/tests.txt
for R in 1 2 4; do
  FP_AGG_ROWS=$R timeout 600 python bench.py --workload llama_block --mp-mode per_step --steps 3 --warmup 3 --no-cpu > $F/bench_R$R.json 2>$F/bench_R$R.err
  FP_AGG_ROWS=$R timeout 600 python bench.py --workload ffnn --mp-mode per_step --steps 3 --warmup 3 --no-cpu > $F/bench_ffnn_R$R.json 2>/dev/null
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gnn_agg -s 8 -c 4 --csv --log-file $F/agg_ncu.csv python bench.py --workload llama_block --mp-mode per_step --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
cat $F/tests.txt
for f in $F/bench_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('$f', round(d['value']), r.get('kernel'), r.get('kernel_ms'), round(r.get('frac',0),3), r.get('achieved'))"; done
python tools/ncu_csv.py $F/agg_ncu.csv 2>/dev/null | tail -12
