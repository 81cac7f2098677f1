# GA pair guide entries: phase times (TV_GA_PROF) old vs new, calibration on/off
for lib in paper_2205_15311_b200/libtv_old.so paper_2205_15311_b200/libtilevolve_b200.so; do
  for cal in 1 0; do
    echo "-- $lib calib=$cal" >> gpurun_out/r2s56_ab.log
    TV_GA_CALIB=$cal TV_GA_PROF=1 TV_LIB_PATH=$lib python tools/prof_ga.py >> gpurun_out/r2s56_ab.log 2>&1
    TV_GA_CALIB=$cal TV_LIB_PATH=$lib python tools/ga_placement.py >> gpurun_out/r2s56_ab.log 2>&1
  done
done
