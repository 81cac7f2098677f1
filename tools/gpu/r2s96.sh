# compute-sanitizer over the final device code (memo forced on so its probes / inserts are covered)
for tool in memcheck racecheck synccheck initcheck; do
  TV_FITMEMO=1 timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_driver.py > gpurun_out/r2s96_sanitizer_$tool.log 2>&1
  echo "exit=$?" >> gpurun_out/r2s96_sanitizer_$tool.log
done
