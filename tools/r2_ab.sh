# A/B of two library builds on one box: FLOWPLACE_B200_LIB selects the .so
for rep in 1 2; do
for v in A B; do
  for w in llama_block ffnn; do
    FLOWPLACE_B200_LIB=$PWD/paper_2505_23131_b200/_flowplace_b200_$v.so timeout 300 python bench.py --steps 30 --warmup 5 --workload $w --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', '$w', round(d['value']), round(d['roofline']['kernel_ms'],4))"
  done
done
done
