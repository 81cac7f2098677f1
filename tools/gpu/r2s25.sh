for i in 1 2; do
python tools/time_enum.py | sed "s/^/ring /"
TV_STACK_S=4 python tools/time_enum.py | sed "s/^/ring4 /"
TV_LIB_PATH=variants/t416.so TV_FAST_THREADS=416 TV_STACK_S=4 TV_CTA_SLOTS=128 python tools/time_enum.py | sed "s/^/t416 /"
TV_LIB_PATH=variants/prev.so python tools/time_enum.py | sed "s/^/prev /"
done > gpurun_out/r2s25_time.log 2>&1
python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r2s25_parity.log 2>&1; echo rc=$? >> gpurun_out/r2s25_parity.log
