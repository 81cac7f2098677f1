# GA launch-geometry variants (TV_GA_THREADS x TV_GA_ILP)
for v in "" variants/ga_t512_i1.so variants/ga_t512_i2.so variants/ga_t512_i4.so variants/ga_t1024_i2.so; do
  for mode in asexual uniform; do
    TV_LIB_PATH=${v:-paper_2205_15311_b200/libtilevolve_b200.so} python tools/prof_ga.py --mode $mode | sed "s|^|${v:-base} |"
  done
  TV_LIB_PATH=${v:-paper_2205_15311_b200/libtilevolve_b200.so} python tools/prof_ga.py --n 512 --gens 20000 | sed "s|^|${v:-base} |"
done > gpurun_out/r2s8_ga.log 2>&1
