# GA layout-switch tests; compute-sanitizer over the staged GA kernel (and every other device path)
python -m pytest tests/test_ga.py -m gpu -q > gpurun_out/r2s66_gatest.log 2>&1; echo rc=$? >> gpurun_out/r2s66_gatest.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_driver.py > gpurun_out/r2s66_sanitizer_$tool.log 2>&1
  echo "exit=$?" >> gpurun_out/r2s66_sanitizer_$tool.log
done
