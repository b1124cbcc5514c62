# A/B of library variants on C2 and C3 (KAFMM_LIB selects the .so)
for v in "" m64 nt3 nt6; do
  lib=paper_2010_15155_b200/libkafmm${v:+_$v}.so
  for c in 2 3; do
    KAFMM_LIB=$PWD/$lib timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/ab_c${c}_${v:-base}.json 2>gpurun_out/ab_c${c}_${v:-base}.err
  done
done
