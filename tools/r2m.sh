python bench.py --steps 10 --warmup 3 > gpurun_out/r2m_bench.json 2> gpurun_out/r2m_bench.err
python tools/bench_step.py 2 full > gpurun_out/r2m_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 42 -c 42 --csv --log-file gpurun_out/r2m_launches_full.csv python tools/bench_step.py 2 full > gpurun_out/r2m_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_part$|k_part<|k_out|k_nxt|k_match_coop" -s 6 -c 6 -o gpurun_out/r2m_full python tools/bench_step.py 2 full > gpurun_out/r2m_ncu2.log 2>&1
