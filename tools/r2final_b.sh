# final round-2 measurements, part B: the launch list of one full-C4 step (ncu, one tool)
python tools/bench_step.py 2 full > gpurun_out/r2f_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 45 -c 45 --csv --log-file gpurun_out/r2f_launches_full.csv python tools/bench_step.py 2 full > gpurun_out/r2f_ncu1.log 2>&1
echo "rc $?" >> gpurun_out/r2f_ncu1.log
