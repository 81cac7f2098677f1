python -m pytest tests/test_ga.py -m gpu -q -k zero_generations (staged-loop edge cases)
