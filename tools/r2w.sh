python tools/bench_step.py 1 sub > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_nxt|k_match" -c 3 -o gpurun_out/r2w python tools/bench_step.py 1 sub > gpurun_out/r2w_ncu.log 2>&1
echo rc $? >> gpurun_out/r2w_ncu.log
