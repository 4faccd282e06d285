python tools/bench_step.py 1 full > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_part$|k_part<|k_out|k_chain_recs" -c 4 -o gpurun_out/r2z python tools/bench_step.py 1 full > gpurun_out/r2z_ncu.log 2>&1
echo rc $? >> gpurun_out/r2z_ncu.log
