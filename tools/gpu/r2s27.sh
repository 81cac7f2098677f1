python -m pytest tests/test_ga.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r2s27_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s27_tests.log
python tools/prof_jatam.py > gpurun_out/r2s27_jatam.log 2>&1
TV_ONEMER=0 python tools/prof_jatam.py >> gpurun_out/r2s27_jatam.log 2>&1
