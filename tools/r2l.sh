timeout 1200 python -m pytest tests -x -q -m gpu -k "not fullsize and not multigpu" > gpurun_out/r2l_tests.log 2>&1; echo "rc $?" >> gpurun_out/r2l_tests.log
python tools/bench_step.py 3 sub ktimes > gpurun_out/r2l_sub.log 2>&1
python tools/bench_step.py 3 full ktimes > gpurun_out/r2l_full.log 2>&1
timeout 600 python -m pytest tests/test_fullsize_gpu.py -x -q -k "C4 and not eager" > gpurun_out/r2l_c4.log 2>&1; echo "rc $?" >> gpurun_out/r2l_c4.log
