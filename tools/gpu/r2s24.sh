for i in 1 2; do
python tools/time_enum.py | sed "s/^/ring /"
TV_LIB_PATH=variants/prev.so python tools/time_enum.py | sed "s/^/prev /"
done > gpurun_out/r2s24_time.log 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_api.py tests/test_ga.py -x -q -m gpu > gpurun_out/r2s24_parity.log 2>&1; echo rc=$? >> gpurun_out/r2s24_parity.log
