# final-state captures (3/3): ncu full of the S32 kernels and the GA kernel
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_classify_fast|k_prepass" -c 2 \
  -o gpurun_out/r2s42_enum32 python tools/enum_once.py s32 > gpurun_out/r2s42_ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k k_ga_run -c 1 \
  -o gpurun_out/r2s42_ga python tools/prof_ga.py --gens 200 >> gpurun_out/r2s42_ncu.log 2>&1
