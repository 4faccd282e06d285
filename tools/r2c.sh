timeout 900 python -m pytest tests/test_step_gpu.py -x -q > gpurun_out/r2c_step.log 2>&1; echo "rc $?" >> gpurun_out/r2c_step.log
timeout 600 python tools/variant_probe.py 3 > gpurun_out/r2c_variants.log 2>&1
