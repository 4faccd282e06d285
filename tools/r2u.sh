# guard-mode tests, the reference arm (C port + Python reference), multi-GPU-free
timeout 1500 python -m pytest tests/test_guard_gpu.py -x -q > gpurun_out/guard.log 2>&1; echo "rc $?" >> gpurun_out/guard.log
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2u_ref.json 2> gpurun_out/r2u_ref.err
