#!/bin/bash
# same-box A/B of two library builds (A = HEAD, B = working tree) + GPU tests
set -x
F=gpurun_out/ab2
mkdir -p $F
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > $F/tests.txt
for rep in 1 2 3; do
for v in A B; do
  for w in llama_block ffnn; do
    FLOWPLACE_B200_LIB=$PWD/paper_2505_23131_b200/_flowplace_b200_$v.so timeout 300 python bench.py --steps 30 --warmup 5 --workload $w --no-cpu 2>/dev/null | tail -1 > $F/${v}_${w}_$rep.json
  done
done
done
FLOWPLACE_B200_LIB=$PWD/paper_2505_23131_b200/_flowplace_b200_B.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file $F/launches_B.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
cat $F/tests.txt
python tools/ncu_csv.py $F/launches_B.csv | tail -9
