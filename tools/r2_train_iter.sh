set -x
mkdir -p gpurun_out/tr
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/tr/gputest.txt
timeout 300 python bench.py --steps 10 --warmup 3 --workload llama_layer --mode train --no-cpu > gpurun_out/tr/bench_train.json 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --workload ffnn --mode train --no-cpu > gpurun_out/tr/bench_train_ffnn.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/tr/train_launches.csv python bench.py --workload llama_layer --mode train --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
cat gpurun_out/tr/gputest.txt
tail -1 gpurun_out/tr/bench_train.json | cut -c1-400
tail -1 gpurun_out/tr/bench_train_ffnn.json | cut -c1-300
