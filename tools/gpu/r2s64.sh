# GA placement structure: 8 calibration arenas, with and without spacer allocations
for gap in 0 2 64; do
  echo "-- gap $gap" >> gpurun_out/r2s64.log
  TV_GA_CALIB=8 TV_GA_CALIB_GAP=$gap TV_GA_CALIB_LOG=1 python tools/ga_bench_order.py >> gpurun_out/r2s64.log 2>&1
done
