timeout 1200 python -m pytest tests -x -q -m gpu -k "not fullsize and not multigpu" > gpurun_out/r2s_tests.log 2>&1; echo "rc $?" >> gpurun_out/r2s_tests.log
python tools/bench_step.py 3 sub ktimes > gpurun_out/r2s_sub.log 2>&1
python tools/bench_step.py 3 full ktimes > gpurun_out/r2s_full.log 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/r2s_bench.json 2> gpurun_out/r2s_bench.err
SYM_WIDE_D2H=1 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2s_bench_wide.json 2> gpurun_out/r2s_bench_wide.err
