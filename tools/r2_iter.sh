# quick iteration: GPU tests, benches of the main workloads, phase profiles
set -x
mkdir -p gpurun_out/it
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/it/gputest.txt
for w in llama_block ffnn; do
  timeout 300 python bench.py --steps 20 --warmup 5 --workload $w --no-cpu > gpurun_out/it/bench_$w.json 2>&1
done
timeout 300 python bench.py --steps 10 --warmup 3 --workload llama_layer --mode train --no-cpu > gpurun_out/it/bench_train.json 2>&1
timeout 300 python tools/phase_profile.py --workload llama_block > gpurun_out/it/phase_llama.txt 2>&1
timeout 300 python tools/phase_profile.py --workload ffnn > gpurun_out/it/phase_ffnn.txt 2>&1
cat gpurun_out/it/gputest.txt
python - <<'P'
import json
for w in ("llama_block", "ffnn", "train"):
    try:
        d = json.loads(open(f"gpurun_out/it/bench_{w}.json").read().strip().splitlines()[-1])
        print(w, round(d["value"]), "e2e", round(d["e2e"]["value"]), "kernel_ms", d["roofline"].get("kernel_ms"), "ms/step", d["ms_per_step"])
    except Exception as e:
        print(w, "ERR", e)
P
tail -8 gpurun_out/it/phase_llama.txt
