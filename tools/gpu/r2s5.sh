python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r2s5_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s5_tests.log
for sw in "0 1 1" "1 1 1" "1 1 0"; do set -- $sw
  TV_EARLY_UNBOUND=$1 TV_ONEMER=$2 TV_FORCED=$3 python tools/time_enum.py | sed "s/^/EU=$1 OM=$2 FZ=$3 /"
done > gpurun_out/r2s5_time.log 2>&1
TV_EARLY_UNBOUND=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s5_launches.csv python tools/time_enum.py > /dev/null 2>&1
