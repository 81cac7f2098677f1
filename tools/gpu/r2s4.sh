# ncu of the a = 3 pre-pass with the trivial-freedom proof (why 26 ms?)
TV_EARLY_UNBOUND=1 ncu --set full --import-source on -k regex:k_prepass -c 2 -o gpurun_out/r2s4_prepass python tools/time_enum.py > gpurun_out/r2s4.log 2>&1
