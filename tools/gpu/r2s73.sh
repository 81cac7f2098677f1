# JaTAM fitness memo: GA tests (memo exactness), A/B of the bench ga_jatam workload
python -m pytest tests/test_ga.py -m gpu -q > gpurun_out/r2s73_gatest.log 2>&1; echo rc=$? >> gpurun_out/r2s73_gatest.log
for memo in 1 0 1 0; do
  TV_FITMEMO=$memo python -c "
import bench, json
r = bench.ga_jatam_bench(cpu_leg=False)
print('memo $memo', round(r['value'], 1), 'gens/s', round(r['ms_per_generation'], 4), 'ms/gen', 'e2e', round(r['e2e']['value'], 1))
" >> gpurun_out/r2s73_ab.log 2>&1
done
