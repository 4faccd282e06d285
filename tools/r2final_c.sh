# final round-2 measurements, part C: ncu --set full of the step's top kernels (second step)
python tools/bench_step.py 2 full > gpurun_out/r2f_plain_c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_part$|k_part<|k_out|k_nxt_tma|k_match_coop|k_tie_fix|k_match_iter|k_chain_recs|k_bid|k_jump4|k_walk_expand|k_fast_emit" -s 15 -c 15 -o gpurun_out/r2f_full python tools/bench_step.py 2 full > gpurun_out/r2f_ncu2.log 2>&1
echo "rc $?" >> gpurun_out/r2f_ncu2.log
