# final round-2 measurements, part A: every GPU test, smoke, the N=1 bench and the reference arm
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2f_tests.log 2>&1; echo "rc $?" >> gpurun_out/r2f_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2f_smoke.log 2>&1
python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err
python bench.py --impl reference > gpurun_out/r2f_ref.json 2> gpurun_out/r2f_ref.err
