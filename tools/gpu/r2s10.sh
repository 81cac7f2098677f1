python -m pytest tests -m gpu -x -q > gpurun_out/r2s10_gputest.log 2>&1; echo rc=$? >> gpurun_out/r2s10_gputest.log
python bench.py > gpurun_out/r2s10_bench.json 2> gpurun_out/r2s10_bench.err
