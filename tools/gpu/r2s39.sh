for i in 1 2; do
python tools/time_enum.py | sed "s/^/base /"
TV_LIB_PATH=variants/a3rows384.so python tools/time_enum.py | sed "s/^/rows384 /"
TV_LIB_PATH=variants/a3rows352.so python tools/time_enum.py | sed "s/^/rows352 /"
done > gpurun_out/r2s39_time.log 2>&1
