for v in A B A B; do
  FLOWPLACE_B200_LIB=$PWD/paper_2505_23131_b200/_flowplace_b200_$v.so timeout 600 python tools/sweep.py --sizes 1000,10000 --batch 1024 --reps 2 --out gpurun_out/ab_wide_$v.jsonl > /dev/null 2>&1
  python -c "
import json
for l in open('gpurun_out/ab_wide_$v.jsonl'): d=json.loads(l); print('$v', d['n'], round(d['episodes_per_s']))"
done
