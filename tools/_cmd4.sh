timeout 1200 python -m pytest tests/test_multigpu_gpu.py -q > gpurun_out/pytest_mgpu4.log 2>&1; echo pytest=$? >> gpurun_out/pytest_mgpu4.log
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2963$n bench.py --gpus $n --steps 100 --warmup 5 > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err
done
