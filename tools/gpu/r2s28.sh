python bench.py > gpurun_out/r2s28_bench.json 2> gpurun_out/r2s28_bench.err
