# A/B: second Fisher-Yates draw only for m == 3 (TV_H2_LAZY build)
for rep in 1 2; do
  for lib in paper_2205_15311_b200/libtilevolve_b200.so paper_2205_15311_b200/libtv_h2.so; do
    TV_LIB_PATH=$lib python tools/time_enum.py >> gpurun_out/r2s91_ab.log 2>&1
  done
done
