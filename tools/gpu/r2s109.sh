bench.py x2 (--no-ga --no-cpu-baseline); nvidia-smi -q
