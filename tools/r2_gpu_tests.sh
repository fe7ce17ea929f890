set -x
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/r2_gputest_all.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:sim_batch -c 40 --csv --log-file gpurun_out/r2_abi_launches.csv python tools/ref_abi_latency.py --calls 10 > /dev/null 2>&1
cat gpurun_out/r2_gputest_all.txt
python tools/ncu_csv.py gpurun_out/r2_abi_launches.csv 2>/dev/null | tail -20 || tail -20 gpurun_out/r2_abi_launches.csv
