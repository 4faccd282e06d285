nvidia-smi -L
timeout 600 python -m pytest tests/test_multigpu_gpu.py -x -q > gpurun_out/r2d_multi.log 2>&1; echo "rc $?" >> gpurun_out/r2d_multi.log
timeout 600 python tools/chain_prof.py > gpurun_out/r2d_chainprof.log 2>&1
timeout 900 python -m pytest tests/test_fullsize_gpu.py -x -q -k "not eager" --durations=20 > gpurun_out/r2d_full.log 2>&1; echo "rc $?" >> gpurun_out/r2d_full.log
