python -m pytest tests/test_gpu_parity.py tests/test_ga.py -x -q -m gpu > gpurun_out/r2s48_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s48_tests.log
python tools/fit_sweep.py > gpurun_out/r2s48_fit.log 2>&1
python tools/time_enum.py > gpurun_out/r2s48_time.log 2>&1
python tools/size_sweep.py >> gpurun_out/r2s48_time.log 2>&1
python tools/prof_jatam.py >> gpurun_out/r2s48_time.log 2>&1
