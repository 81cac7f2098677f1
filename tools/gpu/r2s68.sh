# fix: lanes past the chunk end draw r = 0 (was an uninitialised draw); GA tests + memcheck of the switch cases
python -m pytest tests/test_ga.py -m gpu -q > gpurun_out/r2s68_gatest.log 2>&1; echo rc=$? >> gpurun_out/r2s68_gatest.log
for sw in "0 1" "0 0" "1 0"; do set -- $sw
  TV_GA_STG=$1 TV_GA_PAIR=$2 timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python tools/ga_case.py 4099 32 1 1.0 0 >> gpurun_out/r2s68.log 2>&1
  echo "exit=$? stg=$1 pair=$2" >> gpurun_out/r2s68.log
done
