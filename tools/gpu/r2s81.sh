# same-word E/W movelist marks folded into the placement XOR: parity tests + A/B (time_enum)
python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -q -x > gpurun_out/r2s81_test.log 2>&1; echo rc=$? >> gpurun_out/r2s81_test.log
for rep in 1 2; do
  for lib in paper_2205_15311_b200/libtv_old.so paper_2205_15311_b200/libtilevolve_b200.so; do
    TV_LIB_PATH=$lib python tools/time_enum.py >> gpurun_out/r2s81_ab.log 2>&1
  done
done
