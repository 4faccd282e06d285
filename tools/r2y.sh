# K2 variants (rounds/blocks-per-SM/warps) through SYMPHONY_B200_LIB
for f in build/lib_*.so; do
  echo "== $f" >> gpurun_out/r2y.log
  SYMPHONY_B200_LIB=$PWD/$f python tools/bench_step.py 2 sub ktimes 2>&1 | grep -E "k_nxt_tma|ms_total" >> gpurun_out/r2y.log
  SYMPHONY_B200_LIB=$PWD/$f python tools/bench_step.py 2 full ktimes 2>&1 | grep -E "k_nxt_tma|ms_total" >> gpurun_out/r2y.log
done
