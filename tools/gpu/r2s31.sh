python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_api.py tests/test_ga.py tests/test_cli.py -x -q -m gpu > gpurun_out/r2s31_parity.log 2>&1; echo rc=$? >> gpurun_out/r2s31_parity.log
for i in 1 2; do
python tools/time_enum.py | sed "s/^/csort /"
TV_LIB_PATH=variants/prev.so python tools/time_enum.py | sed "s/^/cub /"
done > gpurun_out/r2s31_time.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s31_launches.csv python tools/enum_once.py s28 > /dev/null 2>&1
