# full bench (new roofline / ceilings fields), then compute-sanitizer over the small driver
python bench.py > gpurun_out/r2s7_bench.json 2> gpurun_out/r2s7_bench.err
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_driver.py > gpurun_out/r2s7_sanitizer_$tool.log 2>&1
  echo "exit=$?" >> gpurun_out/r2s7_sanitizer_$tool.log
done
