python tools/bench_step.py 1 full > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_fast_emit|k_walk_expand|k_token_keys|k_bkt_scatter|k_bkt_sort" -s 7 -c 7 -o gpurun_out/r2w2 python tools/bench_step.py 2 full > gpurun_out/r2w2_ncu.log 2>&1
echo rc $? >> gpurun_out/r2w2_ncu.log
