# final-state pass (end of round 2): GPU tests, smoke, bench, reference arm, launch list, scaling projection
python -m pytest tests -m gpu -q > gpurun_out/r2s108_gputest.log 2>&1; echo rc=$? >> gpurun_out/r2s108_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s108_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2s108_smoke.log
python bench.py > gpurun_out/r2s108_bench.json 2> gpurun_out/r2s108_bench.err
python bench.py --impl reference > gpurun_out/r2s108_reference.json 2> gpurun_out/r2s108_reference.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r2s108_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-ga --no-s32 \
  > /dev/null 2>&1
python tools/scaling_projection.py gpurun_out/r2s108_scaling.json > gpurun_out/r2s108_scaling.log 2>&1
