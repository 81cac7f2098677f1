#!/bin/bash
# Profiling captures for profiles/ (run on the GPU box from the repo root; outputs in gpurun_out/).
set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-ga --no-s32 \
  > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_classify_fast|k_prepass|k_shape_labels" \
  -c 4 -o gpurun_out/enum_full python tools/enum_once.py s28 > gpurun_out/ncu_enum.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_classify_fast|k_prepass" -c 2 \
  -o gpurun_out/enum32_full python tools/enum_once.py s32 > gpurun_out/ncu_enum32.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k k_ga_run -c 1 \
  -o gpurun_out/ga_full python tools/prof_ga.py --gens 200 > gpurun_out/ncu_ga.log 2>&1
tail -n 2 gpurun_out/ncu_enum.log; tail -n 2 gpurun_out/ncu_ga.log
