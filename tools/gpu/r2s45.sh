python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r2s45_parity.log 2>&1; echo rc=$? >> gpurun_out/r2s45_parity.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s45_launches.csv -k regex:"k_key|k_prepass" python tools/enum_once.py s28 > /dev/null 2>&1
python tools/time_enum.py > gpurun_out/r2s45_time.log 2>&1
