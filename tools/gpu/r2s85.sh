python -m pytest tests/test_gpu_multirank.py -m gpu -q -k sweep
