mkdir -p gpurun_out/san; rm -f gpurun_out/san/summary.txt
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 30 --log-file gpurun_out/san/$tool.log python tools/sanitize.py > gpurun_out/san/$tool.out 2>&1
  echo "$tool rc=$?" >> gpurun_out/san/summary.txt
  tail -3 gpurun_out/san/$tool.log >> gpurun_out/san/summary.txt
done
cat gpurun_out/san/summary.txt
