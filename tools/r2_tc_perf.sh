set -x
timeout 600 python -m pytest tests/test_tc_encoder_gpu.py tests/test_tc_gpu.py -q -x 2>&1 | tail -3
for enc in tc; do
  timeout 600 python bench.py --workload ffnn --mp-mode per_step --steps 5 --warmup 3 --no-cpu --encoder $enc > gpurun_out/r2_ps_ffnn_$enc.json 2>&1
  timeout 600 python tools/encode_profile.py --n 1000000 --encoder $enc --shuffle > gpurun_out/r2_enc1m_$enc.json 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_enc1m_tc_launches.csv python tools/encode_profile.py --n 1000000 --encoder tc --shuffle --reps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_node -s 2 -c 2 -o gpurun_out/r2_tc_node_1m python tools/encode_profile.py --n 1000000 --encoder tc --shuffle --reps 1 > /dev/null 2>&1
cat gpurun_out/r2_ps_ffnn_tc.json gpurun_out/r2_enc1m_tc.json
python tools/ncu_csv.py gpurun_out/r2_enc1m_tc_launches.csv | head -8
