for fz in 1 2 0; do TV_FORCED=$fz python tools/time_enum.py | sed "s/^/FZ=$fz /"; done > gpurun_out/r2s12_time.log 2>&1
python tools/scaling_projection.py gpurun_out/r2s12_scaling.json > gpurun_out/r2s12_scaling.log 2>&1
