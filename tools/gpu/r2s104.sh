# reproducibility: three default bench runs back to back (fresh processes)
for i in 1 2 3; do python bench.py > gpurun_out/r2s104_bench_$i.json 2> gpurun_out/r2s104_bench_$i.err; done
