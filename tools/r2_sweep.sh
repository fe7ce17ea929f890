mkdir -p gpurun_out/sw
timeout 900 python tools/sweep.py --sizes 1000,10000 --batch 256,1024,4096,16384,65536 --reps 2 --out gpurun_out/sw/sweep_1k_10k.jsonl > gpurun_out/sw/a.log 2>&1
timeout 900 python tools/sweep.py --sizes 100000 --batch 256,1024,4096 --reps 2 --out gpurun_out/sw/sweep_100k.jsonl > gpurun_out/sw/b.log 2>&1
timeout 600 python bench.py --workload llama_block --batch 8192 --steps 10 --warmup 3 --no-cpu > gpurun_out/sw/bench_llama_8192.json 2>&1
tail -2 gpurun_out/sw/*.log; cat gpurun_out/sw/*.jsonl | cut -c1-200; tail -1 gpurun_out/sw/bench_llama_8192.json | cut -c1-300
