python -m pytest tests -m gpu -q > gpurun_out/r2s23_gputest.log 2>&1; echo rc=$? >> gpurun_out/r2s23_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s23_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2s23_smoke.log
