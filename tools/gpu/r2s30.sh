for i in 1 2; do
python tools/time_enum.py | sed "s/^/t352 /"
TV_LIB_PATH=variants/a3t384.so python tools/time_enum.py | sed "s/^/a3t384 /"
done > gpurun_out/r2s30_time.log 2>&1
python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r2s30_parity.log 2>&1; echo rc=$? >> gpurun_out/r2s30_parity.log
