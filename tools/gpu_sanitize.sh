# compute-sanitizer over the sanitize driver; summaries under gpurun_out/
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 --target-processes all python tools/sanitize_driver.py > gpurun_out/san_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/san_$tool.txt
done
