python -m pytest tests/test_gpu_api.py tests/test_gpu_parity.py -m gpu -q (classify_batch on the tensors' device)
