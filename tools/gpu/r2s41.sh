# final-state captures (2/3): ncu full of the S_{2,8} kernels
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_classify_fast|k_prepass|k_key_scatter" \
  -c 3 -o gpurun_out/r2s41_enum python tools/enum_once.py s28 > gpurun_out/r2s41_ncu.log 2>&1
