set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/s_gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s_smoke.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/s_bench.json 2> gpurun_out/s_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/s_bench_ref.json 2> gpurun_out/s_bench_ref.err
timeout 600 python bench.py --steps 20 --warmup 5 --workload ffnn --no-cpu > gpurun_out/s_bench_ffnn.json 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --workload llama_layer --mode train --no-cpu > gpurun_out/s_bench_train.json 2>&1
cat gpurun_out/s_gputest.txt gpurun_out/s_smoke.txt gpurun_out/s_bench.json gpurun_out/s_bench_ref.json gpurun_out/s_bench_ffnn.json gpurun_out/s_bench_train.json
