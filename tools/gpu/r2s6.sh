# ncu full captures of the enumeration kernels after the work-elimination change
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_classify_fast|k_prepass" \
  -c 2 -o gpurun_out/r2s6_enum python tools/enum_once.py s28 > gpurun_out/r2s6_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_classify_fast|k_prepass" -c 2 \
  -o gpurun_out/r2s6_enum32 python tools/enum_once.py s32 >> gpurun_out/r2s6_ncu.log 2>&1
