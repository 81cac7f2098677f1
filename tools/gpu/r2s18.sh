for i in 1 2; do
python tools/time_enum.py | sed "s/^/D19 /"
TV_GENERIC_D=1 python tools/time_enum.py | sed "s/^/Drt /"
done > gpurun_out/r2s18_time.log 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -x -q -m gpu > gpurun_out/r2s18_parity.log 2>&1; echo rc=$? >> gpurun_out/r2s18_parity.log
