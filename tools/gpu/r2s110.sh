bench.py x2 (full)
