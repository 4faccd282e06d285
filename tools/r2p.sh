timeout 1200 python -m pytest tests -x -q -m gpu -k "not fullsize and not multigpu" > gpurun_out/r2p_tests.log 2>&1; echo "rc $?" >> gpurun_out/r2p_tests.log
timeout 600 python tools/chain_prof.py > gpurun_out/r2p_chainprof.log 2>&1
timeout 600 python tools/variant_probe.py 3 > gpurun_out/r2p_variants.log 2>&1
python tools/bench_step.py 3 sub ktimes > gpurun_out/r2p_sub.log 2>&1
