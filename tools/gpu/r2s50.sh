python tools/ga_placement.py > gpurun_out/r2s50_ga.log 2>&1
TV_GA_CALIB=0 python tools/ga_placement.py | sed "s/^/nocalib /" >> gpurun_out/r2s50_ga.log 2>&1
python -m pytest tests/test_ga.py -x -q -m gpu > gpurun_out/r2s50_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s50_tests.log
python bench.py --no-cpu-baseline --no-s32 > gpurun_out/r2s50_bench.json 2>&1
