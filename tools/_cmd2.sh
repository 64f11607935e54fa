nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
timeout 900 python -m pytest tests/test_multigpu_gpu.py -q -x > gpurun_out/pytest_mgpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_mgpu.log
timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 100 --warmup 5 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo rc=$? >> gpurun_out/bench_n2.err
