set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2_gputest.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_ffnn.json 2> gpurun_out/r2_bench_ffnn.err
timeout 600 python bench.py --steps 20 --warmup 5 --workload llama_block --no-cpu > gpurun_out/r2_bench_llama.json 2>&1
cat gpurun_out/r2_gputest.txt gpurun_out/r2_bench_ffnn.json gpurun_out/r2_bench_llama.json
