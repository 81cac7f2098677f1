python -m pytest tests -m gpu -x -q > gpurun_out/r2s11_gputest.log 2>&1; echo rc=$? >> gpurun_out/r2s11_gputest.log
python bench.py > gpurun_out/r2s11_bench.json 2> gpurun_out/r2s11_bench.err
python tools/time_enum.py > gpurun_out/r2s11_time.log 2>&1
TV_FORCED=0 python tools/time_enum.py >> gpurun_out/r2s11_time.log 2>&1
