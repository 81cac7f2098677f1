# final ncu --set full of the S_{2,8} kernels (pre-pass, scatter, fast kernel) and the S32 kernels
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_classify_fast|k_prepass|k_key_scatter" \
  -c 3 -o gpurun_out/r2s94_enum python tools/enum_once.py s28 > gpurun_out/r2s94_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_classify_fast|k_prepass" -c 2 \
  -o gpurun_out/r2s94_enum32 python tools/enum_once.py s32 >> gpurun_out/r2s94_ncu.log 2>&1
