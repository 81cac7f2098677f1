python tools/time_enum.py | sed "s/^/default /" > gpurun_out/r2s36_tune.log 2>&1
for t in 14 16 24; do TV_SERVICE_THRESH=$t python tools/time_enum.py | sed "s/^/thresh=$t /"; done >> gpurun_out/r2s36_tune.log 2>&1
for c in 128 512; do TV_CTA_SLOTS=$c python tools/time_enum.py | sed "s/^/slots=$c /"; done >> gpurun_out/r2s36_tune.log 2>&1
TV_FORCED=1 python tools/time_enum.py | sed "s/^/forced1 /" >> gpurun_out/r2s36_tune.log 2>&1
