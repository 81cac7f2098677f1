python bench.py --no-ga --no-cpu-baseline (s32 clocks sampled over its pass)
