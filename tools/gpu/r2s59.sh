# ncu full of k_ga_run (first launch: 50 generations at 2^20) with source/SASS, staged chunk + pair entries
timeout 600 ncu --set full --import-source on --clock-control none -k k_ga_run -c 1 \
  -o gpurun_out/r2s59_ga python tools/prof_ga.py --gens 200 > gpurun_out/r2s59_ncu.log 2>&1
