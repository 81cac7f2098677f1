# GA pair guide entries (genomes j, j+1): A/B against the previous build, GA tests
for lib in paper_2205_15311_b200/libtv_old.so paper_2205_15311_b200/libtilevolve_b200.so; do
  for rep in 1 2; do
    TV_LIB_PATH=$lib python tools/prof_ga.py >> gpurun_out/r2s55_ab.log 2>&1
    TV_LIB_PATH=$lib python tools/prof_ga.py --mode uniform >> gpurun_out/r2s55_ab.log 2>&1
    TV_LIB_PATH=$lib python tools/prof_ga.py --n 512 --gens 20000 >> gpurun_out/r2s55_ab.log 2>&1
  done
  echo "-- $lib" >> gpurun_out/r2s55_ab.log
done
python -m pytest tests/test_ga.py -m gpu -q > gpurun_out/r2s55_gatest.log 2>&1; echo rc=$? >> gpurun_out/r2s55_gatest.log
