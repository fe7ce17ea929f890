set -x
mkdir -p gpurun_out/ps
timeout 600 python -m pytest tests/test_train_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
for enc in dmma tc; do
timeout 600 python bench.py --workload ffnn --mp-mode per_step --steps 5 --warmup 3 --no-cpu --encoder $enc > gpurun_out/ps/ps_ffnn_$enc.json 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ps/ps_launches.csv python bench.py --workload ffnn --mp-mode per_step --steps 1 --warmup 3 --no-cpu --encoder tc > /dev/null 2>&1
for f in gpurun_out/ps/*.json; do tail -1 $f | cut -c1-200; done
