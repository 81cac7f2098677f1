python tools/ga_placement.py > gpurun_out/r2s32_ga.log 2>&1
