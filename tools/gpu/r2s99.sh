# A/B: ptxas / nvcc optimisation flags
for rep in 1 2; do
  for lib in libtilevolve_b200 libtv_v1 libtv_v2 libtv_v3; do
    echo -n "$lib " >> gpurun_out/r2s99_ab.log
    TV_LIB_PATH=paper_2205_15311_b200/$lib.so python tools/time_enum.py >> gpurun_out/r2s99_ab.log 2>&1
  done
done
