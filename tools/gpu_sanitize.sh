CS=/usr/local/cuda/bin/compute-sanitizer
python tools/sanitize_cases.py > gpurun_out/san_plain.log 2>&1 || { echo plain failed; tail -5 gpurun_out/san_plain.log; exit 1; }
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool --print-limit 20 python tools/sanitize_cases.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Invalid|Race|hazard" gpurun_out/san_$tool.log | head -5
done
echo done
