# parity under all switches (a = 3 forced default changed), then profiles of the final kernels
python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r2s14_parity.log 2>&1; echo rc=$? >> gpurun_out/r2s14_parity.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_classify_fast|k_prepass" \
  -c 2 -o gpurun_out/r2s14_enum python tools/enum_once.py s28 > gpurun_out/r2s14_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_classify_fast|k_prepass" -c 2 \
  -o gpurun_out/r2s14_enum32 python tools/enum_once.py s32 >> gpurun_out/r2s14_ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k k_ga_run -c 1 \
  -o gpurun_out/r2s14_ga python tools/prof_ga.py --gens 200 >> gpurun_out/r2s14_ncu.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r2s14_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-ga --no-s32 \
  > /dev/null 2>&1
python tools/scaling_projection.py gpurun_out/r2s14_scaling.json > gpurun_out/r2s14_scaling.log 2>&1
