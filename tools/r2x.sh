# perf iteration: GPU tests + C4 full-size parity, step timings, one ncu capture
timeout 1500 python -m pytest tests -x -q -m gpu -k "(not fullsize and not multigpu and not guard) or c4_full or c3_full or C3" > gpurun_out/r2x_tests.log 2>&1; echo "rc $?" >> gpurun_out/r2x_tests.log
python tools/bench_step.py 3 sub ktimes > gpurun_out/r2x_sub.log 2>&1
python tools/bench_step.py 3 full ktimes > gpurun_out/r2x_full.log 2>&1
SYM_DEBUG_TIMING=1 python tools/bench_step.py 1 full > gpurun_out/r2x_phases.log 2>&1

