python tools/prof_jatam.py > gpurun_out/r2s22_jatam.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s22_launches.csv python tools/prof_jatam.py > /dev/null 2>&1
