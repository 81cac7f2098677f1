timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_classify_fast|k_prepass" \
  -c 2 -o gpurun_out/r2s20_enum python tools/enum_once.py s28 > gpurun_out/r2s20_ncu.log 2>&1
python tools/prof_ga.py > gpurun_out/r2s20_ga.log 2>&1
python tools/prof_ga.py >> gpurun_out/r2s20_ga.log 2>&1
TV_GA_PROF=1 python tools/prof_ga.py >> gpurun_out/r2s20_ga.log 2>&1
