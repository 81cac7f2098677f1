for i in 1 2; do
python tools/time_enum.py | sed "s/^/ring12 /"
TV_LIB_PATH=variants/prev.so python tools/time_enum.py | sed "s/^/ring8 /"
done > gpurun_out/r2s52_time.log 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_ga.py -x -q -m gpu > gpurun_out/r2s52_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s52_tests.log
