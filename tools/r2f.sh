python tools/dbg_case.py 'fig4b_timeout_zoo/*' 'table2_resnet50/*' 'stress/1*' 'C2/*' 'C4s0/*' > gpurun_out/r2f_dbg.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x 2>&1 | tail -30 > gpurun_out/r2f_parity.log
