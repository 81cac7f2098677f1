python tools/time_enum.py > gpurun_out/r2s16_time.log 2>&1
TV_LIB_PATH=variants/prev.so python tools/time_enum.py >> gpurun_out/r2s16_time.log 2>&1
python tools/time_enum.py >> gpurun_out/r2s16_time.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s16_launches.csv -k regex:k_prepass python tools/time_enum.py > /dev/null 2>&1
python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "early_unbound or full_s28 or s32" > gpurun_out/r2s16_parity.log 2>&1; echo rc=$? >> gpurun_out/r2s16_parity.log
