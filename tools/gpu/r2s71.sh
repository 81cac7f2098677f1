python -m pytest tests/test_ga.py -m gpu -q -k 's38 or jatam' (JaTAM fitness / generations in S_{3,8}, L = 36)
