timeout 1200 python -m pytest tests -x -q -m gpu -k "not fullsize and not multigpu" > gpurun_out/r2r_tests.log 2>&1; echo "rc $?" >> gpurun_out/r2r_tests.log
python tools/bench_step.py 3 sub ktimes > gpurun_out/r2r_sub.log 2>&1
python tools/bench_step.py 3 full ktimes > gpurun_out/r2r_full.log 2>&1
