python -m pytest tests -m gpu -q > gpurun_out/r2s49_gputest.log 2>&1; echo rc=$? >> gpurun_out/r2s49_gputest.log
python bench.py > gpurun_out/r2s49_bench.json 2> gpurun_out/r2s49_bench.err
python tools/scaling_projection.py gpurun_out/r2s49_scaling.json > gpurun_out/r2s49_scaling.log 2>&1
