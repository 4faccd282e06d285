# confirm the reverted build: sanitizer (one tool), GPU tests, step timings, bench
bash tools/r2_san.sh ${1:-memcheck}
timeout 1200 python -m pytest tests -x -q -m gpu -k "not fullsize and not multigpu" > gpurun_out/r2t_tests.log 2>&1; echo "rc $?" >> gpurun_out/r2t_tests.log
python tools/bench_step.py 3 sub ktimes > gpurun_out/r2t_sub.log 2>&1
python tools/bench_step.py 3 full ktimes > gpurun_out/r2t_full.log 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/r2t_bench.json 2> gpurun_out/r2t_bench.err
