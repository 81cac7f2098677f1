python tools/time_enum.py > gpurun_out/r2s17_time.log 2>&1
TV_LIB_PATH=variants/prev.so python tools/time_enum.py >> gpurun_out/r2s17_time.log 2>&1
python tools/time_enum.py >> gpurun_out/r2s17_time.log 2>&1
TV_LIB_PATH=variants/prev.so python tools/time_enum.py >> gpurun_out/r2s17_time.log 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_ga.py -x -q -m gpu > gpurun_out/r2s17_parity.log 2>&1; echo rc=$? >> gpurun_out/r2s17_parity.log
