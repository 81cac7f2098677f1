python -m pytest tests/test_ga.py -m gpu -q; python tools/prof_ga.py (per-device smem attribute, calibration under memory pressure)
