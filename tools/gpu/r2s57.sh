# ncu full of k_ga_run (first launch: 50 generations at 2^20) with source/SASS, current build
timeout 600 ncu --set full --import-source on --clock-control none -k k_ga_run -c 1 \
  -o gpurun_out/r2s57_ga python tools/prof_ga.py --gens 200 > gpurun_out/r2s57_ncu.log 2>&1
