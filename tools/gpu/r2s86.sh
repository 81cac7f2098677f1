python -m pytest tests/test_gpu_multirank.py tests/test_cli.py -m gpu -q (CLI and GA sweeps under torchrun, two ranks on one GPU)
