set -x
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_cli.py tests/test_gpu_api.py -x -q -m gpu > gpurun_out/r2s2_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s2_tests.log
for eu in 0 1; do for om in 0 1; do TV_EARLY_UNBOUND=$eu TV_ONEMER=$om python tools/time_enum.py; done; done > gpurun_out/r2s2_time.log 2>&1
