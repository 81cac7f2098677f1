python -m pytest tests/test_ga.py -m gpu -q; bench.ga_jatam_bench twice (memo default off below 2^21)
