# histogram export through one packed pinned copy: tests + A/B of export time and the bench e2e
python -m pytest tests/test_gpu_api.py tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_multirank.py -m gpu -q -x > gpurun_out/r2s89_test.log 2>&1; echo rc=$? >> gpurun_out/r2s89_test.log
for lib in paper_2205_15311_b200/libtv_old.so paper_2205_15311_b200/libtilevolve_b200.so; do
  for rep in 1 2; do TV_LIB_PATH=$lib python tools/time_export.py >> gpurun_out/r2s89_ab.log 2>&1; done
  TV_LIB_PATH=$lib python bench.py --no-ga --no-s32 --no-cpu-baseline > gpurun_out/r2s89_bench_$(basename $lib .so).json 2>/dev/null
done
