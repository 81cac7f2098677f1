# A/B: branchless frontier packing (TV_NBP_BRANCHLESS build) + parity
for rep in 1 2 3; do
  for lib in paper_2205_15311_b200/libtilevolve_b200.so paper_2205_15311_b200/libtv_nbp.so; do
    TV_LIB_PATH=$lib python tools/time_enum.py >> gpurun_out/r2s112_ab.log 2>&1
  done
done
TV_LIB_PATH=paper_2205_15311_b200/libtv_nbp.so python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r2s112_test.log 2>&1; echo rc=$? >> gpurun_out/r2s112_test.log
