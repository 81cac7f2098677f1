python -m pytest tests/test_ga.py -x -q -m gpu > gpurun_out/r2s37_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s37_tests.log
python tools/prof_jatam.py > gpurun_out/r2s37_jatam.log 2>&1
TV_FITCACHE=0 python tools/prof_jatam.py >> gpurun_out/r2s37_jatam.log 2>&1
python tools/prof_ga.py >> gpurun_out/r2s37_jatam.log 2>&1
