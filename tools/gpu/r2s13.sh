python tools/size_sweep.py > gpurun_out/r2s13_sizes.log 2>&1
python tools/share_balance.py >> gpurun_out/r2s13_sizes.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s13_launches.csv python tools/size_sweep.py > /dev/null 2>&1
