# state after the GA staging work: GPU tests, smoke, bench, launch list, ncu full of k_ga_run
python -m pytest tests -m gpu -q > gpurun_out/r2s62_gputest.log 2>&1; echo rc=$? >> gpurun_out/r2s62_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s62_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2s62_smoke.log
python bench.py > gpurun_out/r2s62_bench.json 2> gpurun_out/r2s62_bench.err
timeout 600 ncu --set full --import-source on --clock-control none -k k_ga_run -c 1 \
  -o gpurun_out/r2s62_ga python tools/prof_ga.py --gens 200 > gpurun_out/r2s62_ncu.log 2>&1
