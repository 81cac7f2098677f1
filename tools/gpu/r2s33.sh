for pad in 0 1048576 2097152 3145728; do TV_GA_PAD=$pad python tools/ga_placement.py | sed "s/^/pad=$pad /"; done > gpurun_out/r2s33_ga.log 2>&1
