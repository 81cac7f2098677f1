"""One device-vs-restatement GA case (development aid for compute-sanitizer runs).
usage: python tools/ga_case.py n L mode lam stop"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import test_ga
n, L, mode, lam, stop = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4]), int(sys.argv[5])
test_ga.test_device_ga_equals_restatement(n, L, mode, lam, stop)
print("ok", os.environ.get("TV_GA_STG"), os.environ.get("TV_GA_PAIR"))
