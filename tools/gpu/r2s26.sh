timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_classify_fast" \
  -c 1 -o gpurun_out/r2s26_enum python tools/enum_once.py s28 > gpurun_out/r2s26_ncu.log 2>&1
for t in 12 16 20; do TV_SERVICE_THRESH=$t python tools/time_enum.py | sed "s/^/thresh=$t /"; done > gpurun_out/r2s26_time.log 2>&1
python tools/time_enum.py | sed "s/^/default /" >> gpurun_out/r2s26_time.log 2>&1
