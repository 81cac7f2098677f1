for i in 1 2; do
python tools/time_enum.py | sed "s/^/base /"
TV_LIB_PATH=variants/a3t352.so TV_FAST_THREADS=352 python tools/time_enum.py | sed "s/^/a3t352 /"
done > gpurun_out/r2s29_time.log 2>&1
python bench.py --no-s32 --no-cpu-baseline > gpurun_out/r2s29_bench_nos32.json 2>&1
python tools/prof_ga.py >> gpurun_out/r2s29_time.log 2>&1
