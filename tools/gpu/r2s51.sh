python -m pytest tests/test_ga.py -x -q -m gpu > gpurun_out/r2s51_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s51_tests.log
python bench.py --no-cpu-baseline --no-s32 > gpurun_out/r2s51_bench.json 2>&1
