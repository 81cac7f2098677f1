# JaTAM generation launch breakdown (ncu launch list) + bench with the ga_jatam e2e leg
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2s70_launches_jatam.csv python tools/prof_jatam.py > gpurun_out/r2s70_jatam.log 2>&1
python bench.py --no-s32 > gpurun_out/r2s70_bench.json 2> gpurun_out/r2s70_bench.err
