#!/bin/bash
set -x
F=gpurun_out/psprof
mkdir -p $F
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ps_step_kernel -s 20 -c 1 -o $F/ps python bench.py --workload llama_block --mp-mode per_step --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
python tools/ncu_summary.py $F/ps.ncu-rep > $F/ps_summary.txt 2>&1
python tools/ncu_lines.py $F/ps.ncu-rep --top 45 > $F/ps_lines.txt 2>&1
rm -f $F/ps.ncu-rep
