# GA placement: K-arena calibration over a random population, in bench order
TV_GA_CALIB_LOG=1 python tools/ga_bench_order.py > gpurun_out/r2s63_order.log 2>&1
echo "-- K=1" >> gpurun_out/r2s63_order.log
TV_GA_CALIB=1 python tools/ga_bench_order.py >> gpurun_out/r2s63_order.log 2>&1
TV_GA_CALIB_LOG=1 python bench.py --no-s32 > gpurun_out/r2s63_bench.json 2> gpurun_out/r2s63_bench.err
python -m pytest tests/test_ga.py -m gpu -q -x > gpurun_out/r2s63_gatest.log 2>&1; echo rc=$? >> gpurun_out/r2s63_gatest.log
