python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r2s43_parity.log 2>&1; echo rc=$? >> gpurun_out/r2s43_parity.log
python tools/time_enum.py > gpurun_out/r2s43_time.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s43_launches.csv -k regex:k_key python tools/enum_once.py s28 > /dev/null 2>&1
