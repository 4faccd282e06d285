timeout 900 python -m pytest tests -x -q -m gpu -k "not eager and not fullsize and not multigpu" > gpurun_out/r2h_tests.log 2>&1; echo "rc $?" >> gpurun_out/r2h_tests.log
python tools/bench_step.py 3 sub ktimes > gpurun_out/r2h_sub.log 2>&1
python tools/bench_step.py 3 full ktimes > gpurun_out/r2h_full.log 2>&1
python tools/bench_step.py 2 sub > /dev/null 2>&1 && ncu --set full --clock-control none -k regex:"k_ing_scatter|k_ing_count|k_nxt$|k_match_coop|k_out" -s 5 -c 5 -o gpurun_out/r2h_sub python tools/bench_step.py 2 sub > gpurun_out/r2h_ncu_sub.log 2>&1
