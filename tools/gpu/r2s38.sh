timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_classify_fast|k_prepass" \
  -c 2 -o gpurun_out/r2s38_enum32 python tools/enum_once.py s32 > gpurun_out/r2s38_ncu.log 2>&1
