python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_api.py -m gpu -q; python tools/time_enum.py (TV_H2_LAZY default)
