# export staging process-wide: tests + export timing + bench e2e
python -m pytest tests/test_gpu_api.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r2s90_test.log 2>&1; echo rc=$? >> gpurun_out/r2s90_test.log
for rep in 1 2; do python tools/time_export.py >> gpurun_out/r2s90_ab.log 2>&1; done
python bench.py --no-ga --no-s32 --no-cpu-baseline > gpurun_out/r2s90_bench.json 2>/dev/null
