python tools/ga_offsets.py > gpurun_out/r2s34_ga.log 2>&1
