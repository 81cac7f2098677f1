# lone-lane per-pop latency: kernel durations of single-genome launches, and one ncu full capture
for eu in 1 0; do
  TV_EARLY_UNBOUND=$eu timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv \
    --log-file gpurun_out/r2s78_launches_eu$eu.csv python tools/lone_lane.py > gpurun_out/r2s78_eu$eu.log 2>&1
done
TV_EARLY_UNBOUND=0 timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_classify_fast -c 1 \
  -o gpurun_out/r2s78_lone python tools/lone_lane.py > gpurun_out/r2s78_ncu.log 2>&1
