python -m pytest tests/test_gpu_parity.py tests/test_ga.py -x -q -m gpu > gpurun_out/r2s44_parity.log 2>&1; echo rc=$? >> gpurun_out/r2s44_parity.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s44_launches.csv -k regex:k_key python tools/enum_once.py s28 > /dev/null 2>&1
