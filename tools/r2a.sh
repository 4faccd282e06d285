set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python tools/probe.py C4:60 C3:60 C2:60 C5:60 C1:60 > gpurun_out/r2a_probe.log 2>&1
SYM_DEBUG_TIMING=2 python tools/probe.py C4:60 > gpurun_out/r2a_probe_c4_phases.log 2>&1
SYM_DEBUG_TIMING=2 python tools/probe.py C4:7.5 C3:60 > gpurun_out/r2a_probe_c3_phases.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_gputests.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2a_gputests.log
