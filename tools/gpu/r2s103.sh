# A/B: dense-board neighbour reads as word rotates (TV_DENSE_FUNNEL build, a = 3 / S32) + parity
for rep in 1 2; do
  for lib in paper_2205_15311_b200/libtilevolve_b200.so paper_2205_15311_b200/libtv_df.so; do
    TV_LIB_PATH=$lib python tools/time_enum.py >> gpurun_out/r2s103_ab.log 2>&1
  done
done
TV_LIB_PATH=paper_2205_15311_b200/libtv_df.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -q -x > gpurun_out/r2s103_test.log 2>&1; echo rc=$? >> gpurun_out/r2s103_test.log
