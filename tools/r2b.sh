set -x
python tools/variant_probe.py 3 > gpurun_out/r2b_variants.log 2>&1
python bench.py --steps 5 --warmup 3 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2b_ref.json 2> gpurun_out/r2b_ref.err
nproc >> gpurun_out/r2b_variants.log
