python bench.py > gpurun_out/r2s19_bench.json 2> gpurun_out/r2s19_bench.err
