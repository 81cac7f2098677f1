# drain tail of the fast kernel (TV_TAIL_PROF) + A/B that the instrumentation costs nothing when off
for rep in 1 2; do
  for lib in paper_2205_15311_b200/libtv_old.so paper_2205_15311_b200/libtilevolve_b200.so; do
    TV_LIB_PATH=$lib python tools/time_enum.py >> gpurun_out/r2s106_ab.log 2>&1
  done
done
TV_TAIL_PROF=1 python tools/time_enum.py > gpurun_out/r2s106_tail.log 2>&1
TV_TAIL_PROF=1 python tools/size_sweep.py >> gpurun_out/r2s106_tail.log 2>&1
