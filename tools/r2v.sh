# perf iteration: GPU tests (no full-size), step timings
timeout 1200 python -m pytest tests -x -q -m gpu -k "not fullsize and not multigpu and not guard" > gpurun_out/r2v_tests.log 2>&1; echo "rc $?" >> gpurun_out/r2v_tests.log
python tools/bench_step.py 3 sub ktimes > gpurun_out/r2v_sub.log 2>&1
python tools/bench_step.py 3 full ktimes > gpurun_out/r2v_full.log 2>&1
