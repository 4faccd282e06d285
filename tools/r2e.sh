timeout 900 python -m pytest tests -x -q -m gpu -k "not eager and not fullsize" > gpurun_out/r2e_tests.log 2>&1; echo "rc $?" >> gpurun_out/r2e_tests.log
SYM_DEBUG_TIMING=2 python tools/probe.py C4:60 C4:7.5 > gpurun_out/r2e_probe.log 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err
