# SPEC acceptance results regenerated on the final code
python tools/acceptance_s28.py > gpurun_out/r2s111_acc28.log 2>&1; echo rc=$? >> gpurun_out/r2s111_acc28.log
python tools/acceptance_s32.py > gpurun_out/r2s111_acc32.log 2>&1; echo rc=$? >> gpurun_out/r2s111_acc32.log
python tools/hash_integrity.py > gpurun_out/r2s111_hash.log 2>&1; echo rc=$? >> gpurun_out/r2s111_hash.log
mkdir -p gpurun_out/r2s111_results && cp results/*.json gpurun_out/r2s111_results/
