python -m pytest tests/test_ga.py -m gpu -q -k generic_kernel_with_memo
