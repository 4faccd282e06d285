timeout 1200 python -m pytest tests -x -q -m gpu -k "not fullsize and not multigpu" > gpurun_out/r2q_tests.log 2>&1; echo "rc $?" >> gpurun_out/r2q_tests.log
python tools/bench_step.py 3 sub ktimes > gpurun_out/r2q_sub.log 2>&1
python tools/bench_step.py 3 full ktimes > gpurun_out/r2q_full.log 2>&1
python tools/sanitize_case.py > gpurun_out/r2q_sanplain.log 2>&1; echo "rc $?" >> gpurun_out/r2q_sanplain.log
