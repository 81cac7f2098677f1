# GA staged phase C with 32-bit draws (loop-free Poisson head, gkey in shared): GA tests, A/B
python -m pytest tests/test_ga.py -m gpu -q -x > gpurun_out/r2s60_gatest.log 2>&1; echo rc=$? >> gpurun_out/r2s60_gatest.log
run() { echo "-- $*" >> gpurun_out/r2s60_ab.log; env "$@" python tools/prof_ga.py >> gpurun_out/r2s60_ab.log 2>&1;
        env "$@" python tools/prof_ga.py --mode uniform >> gpurun_out/r2s60_ab.log 2>&1;
        env "$@" python tools/prof_ga.py --mode uniform --mu 4 >> gpurun_out/r2s60_ab.log 2>&1;
        env "$@" python tools/prof_ga.py --n 512 --gens 20000 >> gpurun_out/r2s60_ab.log 2>&1; }
run TV_LIB_PATH=paper_2205_15311_b200/libtv_old.so
run TV_GA_PROF=1
run TV_LIB_PATH=paper_2205_15311_b200/libtv_old.so
run TV_GA_PROF=1
