for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_driver.py > gpurun_out/r2s53_sanitizer_$tool.log 2>&1
  echo "exit=$?" >> gpurun_out/r2s53_sanitizer_$tool.log
done
