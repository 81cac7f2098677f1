# round 2 session 3: parity under the work-elimination switches + timings + per-kernel times
python -m pytest tests/test_gpu_parity.py tests/test_cli.py -x -q -m gpu > gpurun_out/r2s3_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s3_tests.log
for sw in "0 0 0" "1 1 0" "1 1 1" "0 1 1" "1 0 1"; do set -- $sw
  TV_EARLY_UNBOUND=$1 TV_ONEMER=$2 TV_FORCED=$3 python tools/time_enum.py | sed "s/^/EU=$1 OM=$2 FZ=$3 /"
done > gpurun_out/r2s3_time.log 2>&1
TV_EARLY_UNBOUND=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s3_launches_eu1.csv python tools/time_enum.py > /dev/null 2>&1
TV_EARLY_UNBOUND=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s3_launches_eu0.csv python tools/time_enum.py > /dev/null 2>&1
