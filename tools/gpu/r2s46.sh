python -m pytest tests/test_ga.py -x -q -m gpu > gpurun_out/r2s46_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s46_tests.log
python tools/prof_jatam.py > gpurun_out/r2s46_jatam.log 2>&1
TV_LIB_PATH=variants/prev.so python tools/prof_jatam.py >> gpurun_out/r2s46_jatam.log 2>&1
