export FP_BENCH_DIST_BACKEND=gloo
for mode in rollout train; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --mode $mode --no-cpu 2>&1 | grep -E '^\{|Error|error' | cut -c1-300
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 2 --warmup 1 --impl reference 2>&1 | grep -E '^\{|Error|error' | cut -c1-300
