# 2 or 4 GPUs: the single-call multi-device tests, then bench.py under torchrun
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_multigpu_gpu.py -q > gpurun_out/r2_multi_tests_$N.log 2>&1; echo "rc $?" >> gpurun_out/r2_multi_tests_$N.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/r2_bench_${N}gpu.json 2> gpurun_out/r2_bench_${N}gpu.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus $N --steps 3 --warmup 3 > gpurun_out/r2_bench_${N}gpu_ref.json 2> gpurun_out/r2_bench_${N}gpu_ref.err
