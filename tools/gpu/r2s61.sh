# replica GA with 32-bit draws: GA tests, sweep A/B
python -m pytest tests/test_ga.py -m gpu -q -x > gpurun_out/r2s61_gatest.log 2>&1; echo rc=$? >> gpurun_out/r2s61_gatest.log
for lib in paper_2205_15311_b200/libtv_old.so paper_2205_15311_b200/libtilevolve_b200.so; do
  echo "-- $lib" >> gpurun_out/r2s61_ab.log
  TV_LIB_PATH=$lib python tools/sweep_bench.py >> gpurun_out/r2s61_ab.log 2>&1
done
