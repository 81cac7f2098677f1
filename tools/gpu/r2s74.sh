# JaTAM: f_known tied to the fitness signature, memo cleared per run; tests; generation time vs n, memo on/off
python -m pytest tests/test_ga.py -m gpu -q > gpurun_out/r2s74_gatest.log 2>&1; echo rc=$? >> gpurun_out/r2s74_gatest.log
TV_FITMEMO=1 python tools/jatam_scale.py > gpurun_out/r2s74_scale.log 2>&1
TV_FITMEMO=0 python tools/jatam_scale.py >> gpurun_out/r2s74_scale.log 2>&1
