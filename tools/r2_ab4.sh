#!/bin/bash
# same-box A/B (A = HEAD, B = split-K SEL head in the small encoder) + GPU tests on B
set -x
F=gpurun_out/ab4
mkdir -p $F
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > $F/tests.txt
for rep in 1 2 3; do
for v in A B; do
  for w in ffnn chainmm; do
    FLOWPLACE_B200_LIB=$PWD/paper_2505_23131_b200/_flowplace_b200_$v.so timeout 300 python bench.py --steps 30 --warmup 5 --workload $w --no-cpu 2>/dev/null | tail -1 > $F/${v}_${w}_$rep.json
  done
done
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gnn_small -c 4 --csv --log-file $F/small_B.csv python bench.py --workload ffnn --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
cat $F/tests.txt
python tools/ncu_csv.py $F/small_B.csv | tail -2
