python tools/fit_sweep.py > gpurun_out/r2s47_fit.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s47_launches.csv python tools/fit_sweep.py > /dev/null 2>&1
