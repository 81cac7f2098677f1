for sl in 26 28 30 24; do TV_SLICE_LOG2=$sl python tools/time_s32.py; done > gpurun_out/r2s35_s32.log 2>&1
